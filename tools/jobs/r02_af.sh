export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_rowblock.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmv_rowstage|k_csr" --csv --log-file gpurun_out/r02_launches_cfg1_csr.csv python bench.py --config cfg1 --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1; grep -E "k_spmv_row|k_csr" gpurun_out/r02_launches_cfg1_csr.csv | awk -F'","' '{print substr($5,1,60), $NF}'
timeout 400 python bench.py --config cfg1 --no-cpu-baseline --steps 20 > gpurun_out/b_cfg1.json 2>gpurun_out/b_cfg1.err
python -c "import json;d=json.loads(open('gpurun_out/b_cfg1.json').read().splitlines()[-1]);print('cfg1',d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['schedule'],d['e2e']['value'],d['baselines_same_gpu'])" || tail -5 gpurun_out/b_cfg1.err
