timeout 600 python -m pytest tests/test_gpu_seg.py -x -q -p no:cacheprovider > gpurun_out/seg_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/seg_tests.log
for s in seg stream; do
timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-baselines --schedule $s --steps 10 > gpurun_out/b_cfg3_$s.json 2>gpurun_out/b_cfg3_$s.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg3_$s.json').read().splitlines()[-1]);print('$s cfg3',d['ms_per_step'],d['roofline']['frac'],d['config']['workers'])" || tail -5 gpurun_out/b_cfg3_$s.err
done
for s in seg rowblock; do
timeout 300 python bench.py --config cfg1 --no-cpu-baseline --no-baselines --schedule $s --steps 20 > gpurun_out/b_cfg1_$s.json 2>gpurun_out/b_cfg1_$s.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg1_$s.json').read().splitlines()[-1]);print('$s cfg1',d['ms_per_step'],d['roofline']['frac'],d['config']['workers'])" || tail -5 gpurun_out/b_cfg1_$s.err
done
