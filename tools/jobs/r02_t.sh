timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_t.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error" gpurun_out/gpu_tests_t.log | head -20; tail -3 gpurun_out/gpu_tests_t.log
for c in cfg2 cfg5; do timeout 600 python tools/warp_cost.py --config $c 2>&1 | tail -22; done
for c in cfg2 H cfg4 cfg5; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['schedule'],d['config']['slice_cost'],d['e2e']['value'],d['gpu_launches'],d.get('gather_roofline'))" || tail -5 gpurun_out/b_$c.err
done
