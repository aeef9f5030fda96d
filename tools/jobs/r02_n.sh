for h in 65536 4096 1024 256 1; do
timeout 400 python bench.py --config cfg2d --hub $h --no-cpu-baseline --no-baselines --steps 10 > gpurun_out/b_cfg2d_$h.json 2>gpurun_out/b_cfg2d_$h.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg2d_$h.json').read().splitlines()[-1]);print('cfg2d $h',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['hub_min'],d['config']['hot_columns'],d['config']['warm_columns'],d['check']['max_componentwise_err_vs_cusparse_f64'])" || tail -5 gpurun_out/b_cfg2d_$h.err
done
