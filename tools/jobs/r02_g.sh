timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
for c in cfg3 cfg2 H; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['schedule'],d.get('gather_roofline'),d['e2e']['value'],d['clocks'])" || tail -5 gpurun_out/b_$c.err
done
