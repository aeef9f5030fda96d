timeout 900 python -m pytest tests/test_gpu_hot.py -q -x -p no:cacheprovider 2>&1 | tail -1
for px in 0 wide; do
for c in cfg5 cfg2d; do
HBP_PACKED_X=$px timeout 400 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$px $c',d['ms_per_step'],d['value'],d['roofline']['frac'],(d.get('gather_roofline') or {}).get('frac'),d['config']['hot_columns'],d['config']['warm_columns'],d['config']['workers'],d['check']['max_componentwise_err_vs_cusparse_f64'])" || tail -5 gpurun_out/b_$c.err
done
done
