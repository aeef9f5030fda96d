export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_oracle_golden.py tests/test_reorder_kernels.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -1
for c in cfg3 cfg2; do
echo "== $c"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_count_runs|k_emit_runs" -c 4 --csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 1 --warmup 1 2>/dev/null | grep -v "==" | awk -F'","' 'NR>1{print substr($5,1,40), $NF}'
done
