nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_ag.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error" gpurun_out/gpu_tests_ag.log | head -20; tail -2 gpurun_out/gpu_tests_ag.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in cfg2 H cfg4 cfg3 cfg5 cfg1 cfg2d; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],(d.get('gather_roofline') or {}).get('frac'),d['config']['schedule'],d['e2e']['value'],d['gpu_launches'],d['clocks']['reasons'],d['baselines_same_gpu'])" || tail -5 gpurun_out/b_$c.err
done
