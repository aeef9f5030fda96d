export PATH=/usr/local/cuda/bin:$PATH
for t in 1 0; do HBP_HASH_THREAD=$t timeout 900 python -m pytest tests/test_reorder_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/form=$t /"; done
for c in cfg3 cfg2 H; do
HBP_HASH_THREAD=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hash_perm" --csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 1 --warmup 3 2>/dev/null | grep k_hash | awk -F'","' '{print substr($5,1,40), $NF}' | head -1 | sed "s/^/$c /"
done
