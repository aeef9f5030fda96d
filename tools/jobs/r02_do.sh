export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_rowblock.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "rowstage or cfg1" 2>&1 | tail -2
HBP_ROWSTAGE_META=0 timeout 900 python -m pytest tests/test_gpu_rowblock.py -q -x -p no:cacheprovider -k "rowstage" 2>&1 | tail -1
for r in 1 2; do for m in 0 1; do
HBP_ROWSTAGE_META=$m timeout 600 python tools/ab_sched.py --config cfg1 --flush --runs rowstage --rounds 5 --iters 20 2>&1 | tail -1 | sed "s/^/meta=$m /"
done; done
for m in 0 1; do
HBP_ROWSTAGE_META=$m timeout 600 python bench.py --config cfg1 --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('bench meta=$m',d['ms_per_step'],d['roofline']['kernel_ms'],d['check'])"
HBP_ROWSTAGE_META=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmv_rowstage" -c 4 --csv python bench.py --config cfg1 --no-cpu-baseline --no-baselines --steps 3 --warmup 3 2>/dev/null | grep -v "==" | awk -F'","' 'NR>1{print "ncu meta='$m'", $(NF)}'
done
