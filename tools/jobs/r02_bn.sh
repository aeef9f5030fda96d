timeout 900 python -m pytest tests/test_gpu_hot.py tests/test_gpu_scale.py tests/test_gpu_stripes.py -q -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
for c in cfg2 cfg5 cfg2d; do
timeout 400 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],(d.get('gather_roofline') or {}).get('frac'),d['config']['hot_columns'],d['config']['hot_share'],d['e2e']['value'],d['check'])" || tail -5 gpurun_out/b_$c.err
done
