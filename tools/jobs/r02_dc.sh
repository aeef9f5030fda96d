export PATH=/usr/local/cuda/bin:$PATH
for r in 1 2 3; do for v in old new; do for c in cfg2 H cfg5; do
HBP_LIB_PATH=_prev/libhbp_$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('$v $c',d['ms_per_step'],d['roofline']['kernel_ms'],d['check']['max_componentwise_err_vs_cusparse_f64'])"
done; done; done
