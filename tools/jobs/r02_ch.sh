timeout 900 python -m pytest tests/test_gpu_hot.py -q -x -p no:cacheprovider 2>&1 | tail -1
for px in split 0 split 0; do
HBP_PACKED_X=$px timeout 400 python bench.py --config cfg5 --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_cfg5.json 2>gpurun_out/b_cfg5.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg5.json').read().splitlines()[-1]);print('$px cfg5',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['hot_columns'],d['config']['warm_columns'],d['config']['workers'],d['check']['max_componentwise_err_vs_cusparse_f64'])" || tail -5 gpurun_out/b_cfg5.err
done
for px in split 0; do
HBP_PACKED_X=$px timeout 400 python bench.py --config cfg2d --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_cfg2d.json 2>gpurun_out/b_cfg2d.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg2d.json').read().splitlines()[-1]);print('$px cfg2d',d['ms_per_step'],d['value'],d['config']['hot_columns'],d['config']['warm_columns'],d['check']['max_componentwise_err_vs_cusparse_f64'])" || tail -5 gpurun_out/b_cfg2d.err
done
