export PATH=/usr/local/cuda/bin:$PATH
for r in 1 2 3; do for bw in 0 8192 16384 32768 65536; do for c in cfg2; do
HBP_L1_BAND=$bw timeout 600 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('band $bw $c',d['ms_per_step'],d['roofline']['kernel_ms'],d['check']['max_componentwise_err_vs_cusparse_f64'])"
done; done; done
for bw in 0 16384 32768; do for kb in 165 175; do
HBP_HOT_BUDGET_KB=$kb HBP_L1_BAND=$bw timeout 600 python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('band $bw budget $kb',d['ms_per_step'],d['roofline']['kernel_ms'],d['check']['max_componentwise_err_vs_cusparse_f64'])"
done; done
