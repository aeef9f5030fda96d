set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 ./tools/gather_peaks 27 > gpurun_out/gather_peaks.jsonl 2> gpurun_out/gather_peaks.err
timeout 300 python bench.py --config cfg2 --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_cfg2.json 2>gpurun_out/b_cfg2.err
timeout 300 python bench.py --config H --no-cpu-baseline --no-baselines --steps 20 > gpurun_out/b_H.json 2>gpurun_out/b_H.err
tail -c 600 gpurun_out/b_cfg2.json; tail -c 300 gpurun_out/b_H.json
