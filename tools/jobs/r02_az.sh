export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_hot.py -q -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
timeout 400 python bench.py --config cfg5 --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_cfg5.json 2>gpurun_out/b_cfg5.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg5.json').read().splitlines()[-1]);print('cfg5',d['ms_per_step'],d['value'],d['roofline']['frac'],(d.get('gather_roofline') or {}).get('frac'),d['e2e']['value'],d['check'])" || tail -5 gpurun_out/b_cfg5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_hot_gather|k_spmv_stream|k_sumsq|sumsq" -c 6 --csv python bench.py --config cfg5 --no-cpu-baseline --no-baselines --steps 1 --warmup 3 2>/dev/null | grep -E "k_hot|k_spmv|sumsq" | awk -F'","' '{print substr($5,1,40), $NF}' | tail -6
