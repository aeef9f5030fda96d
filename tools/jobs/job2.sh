timeout 120 ./tools/gather_peaks 27 tma > gpurun_out/gather_peaks_tma.jsonl 2>&1
cat gpurun_out/gather_peaks_tma.jsonl
free -g | head -2; nproc; lscpu | grep "Model name"
