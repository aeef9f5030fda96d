export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_cfg3.csv python bench.py --config cfg3 --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_b3.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_seg -s 2 -c 1 -o gpurun_out/r02_full_cfg3 python bench.py --config cfg3 --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_f3.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/
