timeout 900 python -m pytest tests/test_gpu_rowblock.py -q -x -p no:cacheprovider > gpurun_out/rowstage_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rowstage_tests.log
grep -E "^E " gpurun_out/rowstage_tests.log | head -10
for v in "1 256" "0 256" "1 512" "0 512"; do set -- $v
HBP_ROWSTAGE_PREFETCH=$1 HBP_ROWSTAGE_THREADS=$2 timeout 600 python tools/ab_sched.py --config cfg1 --flush --runs rowblock,rowstage --rounds 5 --iters 20 2>&1 | tail -1 | sed "s/^/pf=$1 nt=$2 /"
done
