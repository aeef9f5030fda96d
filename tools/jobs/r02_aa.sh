export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_aa.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error" gpurun_out/gpu_tests_aa.log | head -20; tail -2 gpurun_out/gpu_tests_aa.log
for c in cfg1 cfg3; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b_$c.json').read().splitlines()[-1]);print('$c',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['schedule'],d['e2e']['value'],d['gpu_launches'],d['baselines_same_gpu'])" || tail -5 gpurun_out/b_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg2.csv python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_l2.log 2>&1; echo "launch list cfg2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg1.csv python bench.py --config cfg1 --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_l1.log 2>&1; echo "launch list cfg1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_stream -s 3 -c 1 -o gpurun_out/r02_full_cfg2 python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_f2.log 2>&1; echo "full cfg2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_rowstage -s 3 -c 1 -o gpurun_out/r02_full_cfg1 python bench.py --config cfg1 --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_f1.log 2>&1; echo "full cfg1 rc=$?"
ls gpurun_out
