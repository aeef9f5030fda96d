free -g | head -2; nproc
timeout 2700 python tools/ref_fullscale.py cfg1 cfg4 H cfg2 > gpurun_out/ref_fullscale.jsonl 2> gpurun_out/ref_fullscale.err; echo "rc=$?"
cat gpurun_out/ref_fullscale.jsonl | cut -c1-800; tail -3 gpurun_out/ref_fullscale.err
