export PATH=/usr/local/cuda/bin:$PATH
timeout 300 ./tools/gather_mix 27 > gpurun_out/gather_mix.jsonl 2>&1; echo "mix rc=$?"; cat gpurun_out/gather_mix.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02h_launches_cfg2.csv python bench.py --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_b2.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_stream -s 2 -c 1 -o /tmp/full_cfg2 python bench.py --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_f2.log 2>&1; echo "full rc=$?"
ncu -i /tmp/full_cfg2.ncu-rep --page raw --csv > gpurun_out/r02h_ncu_cfg2_raw.csv 2>&1
ncu -i /tmp/full_cfg2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02h_cfg2_source.csv 2>&1
ls -la gpurun_out/r02h_*
