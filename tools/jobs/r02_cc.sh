export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_reorder_kernels.py tests/test_gpu_parity.py -q -p no:cacheprovider 2>&1 | tail -1
HBP_HASH_THREAD=1 timeout 900 python -m pytest tests/test_reorder_kernels.py -q -p no:cacheprovider 2>&1 | tail -1
for c in H cfg4 cfg1; do
for t in 0 1; do
HBP_HASH_THREAD=$t timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hash_perm" --csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 1 --warmup 3 2>/dev/null | grep k_hash | awk -F'","' '{print substr($5,1,40), $NF}' | head -1 | sed "s/^/thread=$t $c /"
done
done
