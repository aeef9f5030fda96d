export PATH=/usr/local/cuda/bin:$PATH
for r in 1 2; do for ch in 1 2 4 8 16; do
HBP_PIPE_CHUNKS=$ch timeout 600 python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('chunks $ch',d['ms_per_step'],d['e2e']['value'],d['check']['e2e_y_equals_device_y'])"
done; done
for dp in 2 4; do
HBP_PIPE_DEPTH=$dp HBP_PIPE_CHUNKS=4 timeout 600 python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('depth $dp chunks 4',d['ms_per_step'],d['e2e']['value'],d['check']['e2e_y_equals_device_y'])"
done
