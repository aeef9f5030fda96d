export PATH=/usr/local/cuda/bin:$PATH
for r in 1 2; do for v in 0 3; do for c in H cfg4 cfg2; do
HBP_STREAM_VARIANT=$v timeout 600 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('v$v $c',d['ms_per_step'],d['roofline']['kernel_ms'],d['config'].get('hot_columns'),d['check']['max_componentwise_err_vs_cusparse_f64'])"
done; done; done
