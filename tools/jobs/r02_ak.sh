for v in 1 0 1; do
HBP_PACKED_X=$v timeout 400 python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_cfg2_p$v.json 2>gpurun_out/b_cfg2_p$v.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg2_p$v.json').read().splitlines()[-1]);print('packed=$v',d['ms_per_step'],d['value'],d['e2e'])" || tail -5 gpurun_out/b_cfg2_p$v.err
done
