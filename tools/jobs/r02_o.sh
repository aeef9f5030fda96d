timeout 900 python -m pytest tests/test_gpu_stripes.py -x -q -p no:cacheprovider > gpurun_out/stripes_tests.log 2>&1; echo "tests rc=$?"; grep -E "Error|error|passed|failed" gpurun_out/stripes_tests.log | tail -15
for c in cfg2 cfg5 cfg3 cfg1; do
timeout 400 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 10 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['schedule'],d['e2e']['value'],d['gpu_launches'],d['preprocess_ms'],d['check'])" || tail -5 gpurun_out/b_$c.err
done
