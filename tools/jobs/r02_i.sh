timeout 600 python -m pytest tests/test_gpu_hub.py tests/test_gpu_balanced.py -x -q -p no:cacheprovider > gpurun_out/hub_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/hub_tests.log
for h in off auto; do
timeout 400 python bench.py --config cfg2d --hub $h --no-cpu-baseline --no-baselines --steps 10 > gpurun_out/b_cfg2d_$h.json 2>gpurun_out/b_cfg2d_$h.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg2d_$h.json').read().splitlines()[-1]);print('cfg2d $h',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['hub_min'],d['check'])" || tail -5 gpurun_out/b_cfg2d_$h.err
done
