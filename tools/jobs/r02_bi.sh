nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_bi.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error" gpurun_out/gpu_tests_bi.log | head -20; tail -2 gpurun_out/gpu_tests_bi.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b_default.json 2> gpurun_out/b_default.err; echo "default rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/b_default.json').read().splitlines()[-1]);print('default',d['ms_per_step'],d['value'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'],d['cpu_baseline']['kind'],d['preprocess_gate']['gpu_preprocess_faster_than_one_cpu_spmv'],d['clocks'])" || tail -5 gpurun_out/b_default.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo "ref rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/b_ref.json').read().splitlines()[-1]);print('ref',d['value'],d['cpu_baseline'])"
for c in H cfg4 cfg3 cfg5 cfg1 cfg2d; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],(d.get('gather_roofline') or {}).get('frac'),d['config']['schedule'],d['e2e']['value'],d['gpu_launches'],d['clocks']['reasons'],d['baselines_same_gpu']['speedup_vs_cusparse'])" || tail -5 gpurun_out/b_$c.err
done
