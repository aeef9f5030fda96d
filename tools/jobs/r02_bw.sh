timeout 900 python -m pytest tests/test_gpu_hot.py tests/test_gpu_scale.py -q -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
for r in 0 1; do
for c in cfg5 cfg2 cfg2d; do
HBP_HOT_REFRESH=$r timeout 400 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('refresh=$r $c',d['ms_per_step'],d['value'],d['roofline']['frac'],d['check']['max_componentwise_err_vs_cusparse_f64'])" || tail -5 gpurun_out/b_$c.err
done
done
