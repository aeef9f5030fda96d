export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_stream" -c 2 -o gpurun_out/r02_tk_H python tools/ab_ticket.py --config H --runs "eq/1.0:1" --rounds 1 --iters 1 > /dev/null 2>&1; echo rc=$?
ls -la gpurun_out/r02_tk_H*
