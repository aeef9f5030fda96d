export PATH=/usr/local/cuda/bin:$PATH
for r in 1 2; do for wb in 48 64 80 96; do
HBP_WARM_BYTES=$((wb<<20)) timeout 600 python bench.py --config cfg5 --no-cpu-baseline --no-baselines --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('warm ${wb}MB',d['ms_per_step'],d['roofline']['kernel_ms'],d['check'])"
done; done
