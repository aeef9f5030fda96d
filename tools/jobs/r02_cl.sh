export PATH=/usr/local/cuda/bin:$PATH
for t in 0 1; do HBP_HASH_THREAD=$t timeout 900 python -m pytest tests/test_reorder_kernels.py tests/test_gpu_parity.py tests/test_oracle_golden.py -q -x -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/form=$t /"; done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "cfg1" 2>&1 | tail -1
for c in cfg1 H; do
HBP_HASH_THREAD=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hash_perm" --csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 1 --warmup 3 2>/dev/null | grep k_hash | awk -F'","' '{print substr($5,1,45), $NF}' | head -1 | sed "s/^/$c /"
done
