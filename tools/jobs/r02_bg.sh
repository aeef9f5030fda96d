timeout 900 python -m pytest tests/test_gpu_hub.py tests/test_gpu_balanced.py -q -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
timeout 400 python bench.py --config cfg2d --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_cfg2d.json 2>gpurun_out/b_cfg2d.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg2d.json').read().splitlines()[-1]);print('cfg2d',d['ms_per_step'],d['value'],d['roofline']['frac'],(d.get('gather_roofline') or {}).get('frac'),d['config']['slice_cost'],d['check'])" || tail -5 gpurun_out/b_cfg2d.err
