export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02i_gpu_tests.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error" gpurun_out/r02i_gpu_tests.log | head -20; tail -1 gpurun_out/r02i_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
s=$(date +%s); timeout 900 python bench.py > gpurun_out/r02i_bench_default_cfg2.json 2> gpurun_out/b_default.err; echo "default rc=$? wall=$(( $(date +%s) - s ))s"
python -c "import json;d=json.loads(open('gpurun_out/r02i_bench_default_cfg2.json').read().splitlines()[-1]);print('default',d['ms_per_step'],d['value'],d['roofline']['frac'],d['gather_roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'],d['cpu_baseline']['kind'],d['gpu_launches'],d['clocks'])" || tail -5 gpurun_out/b_default.err
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r02i_bench_reference_cfg2.json 2> gpurun_out/b_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - s ))s"; python -c "import json;d=json.loads(open('gpurun_out/r02i_bench_reference_cfg2.json').read().splitlines()[-1]);print('ref',d['value'],d['cpu_baseline']['sample'][:60])"
for c in H cfg4 cfg3 cfg5 cfg1 cfg2d; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/r02i_bench_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/r02i_bench_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],(d.get('gather_roofline') or {}).get('frac'),d['config']['schedule'],d['e2e']['value'],d['clocks']['reasons'],d['baselines_same_gpu']['speedup_vs_cusparse'])" || tail -5 gpurun_out/b_$c.err
done
for c in cfg2 cfg5; do
HBP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config $c --steps 5 --warmup 3 > gpurun_out/r02i_bench_N2_gloo_onegpu_$c.json 2> gpurun_out/b2_$c.err; echo "N2 $c rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02i_bench_N2_gloo_onegpu_$c.json').read().splitlines()[-1]);c=d['config'];print(c.get('collective'), d['ms_per_step'], d['n_gpus'], d.get('check'))" || tail -3 gpurun_out/b2_$c.err
done
