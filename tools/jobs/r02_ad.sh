timeout 600 python -m pytest tests/test_gpu_rowblock.py -q -x -p no:cacheprovider 2>&1 | tail -2
for nt in 512 256; do
HBP_ROWSTAGE_THREADS=$nt timeout 600 python tools/ab_sched.py --config cfg1 --flush --runs rowblock,rowstage --rounds 5 --iters 20 2>&1 | tail -2 | sed "s/^/nt=$nt /"
done
