set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep "Model name"; nproc; free -g | head -2
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 300 ./tools/gather_peaks 27 > gpurun_out/gather_peaks.jsonl 2> gpurun_out/gather_peaks.err; echo "gp rc=$?"
timeout 300 python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/b_cfg2.json 2>gpurun_out/b_cfg2.err
timeout 300 python bench.py --config H --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b_H.json 2>gpurun_out/b_H.err
tail -c 400 gpurun_out/b_cfg2.json
