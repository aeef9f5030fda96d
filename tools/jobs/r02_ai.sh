timeout 900 python -m pytest tests/test_gpu_hot.py tests/test_gpu_balanced.py tests/test_gpu_scale.py tests/test_gpu_stripes.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/px/eq" --rounds 3 --iters 10 2>&1 | tail -4
for c in cfg2; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline'],(d.get('gather_roofline') or {}).get('frac'),d['config']['schedule'],d['e2e']['value'],d['gpu_launches'],d['clocks']['reasons'],d['baselines_same_gpu'],d['config']['hot_share'],d['config']['warm_columns'])" || tail -5 gpurun_out/b_$c.err
done
