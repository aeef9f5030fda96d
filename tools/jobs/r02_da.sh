export PATH=/usr/local/cuda/bin:$PATH
for r in 1 2; do for kb in 185 195 205 213 220; do
HBP_HOT_BUDGET_KB=$kb timeout 600 python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('budget $kb',d['ms_per_step'],d['roofline']['kernel_ms'],d['config'].get('hot_columns'),d['check']['max_componentwise_err_vs_cusparse_f64'])"
done; done
