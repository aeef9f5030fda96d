export PATH=/usr/local/cuda/bin:$PATH
HBP_PACKED_X=0 timeout 300 python tools/e2e_probe.py cfg2 20 2>&1 | tail -3
HBP_PACKED_X=1 timeout 300 python tools/e2e_probe.py cfg2 20 2>&1 | tail -3
HBP_PACKED_X=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hot_gather|k_spmv_stream" --cache-control none -c 40 --csv python tools/e2e_probe.py cfg2 5 2>/dev/null | grep -E "k_hot|k_spmv" | awk -F'","' '{print substr($5,1,40), $NF}' | tail -12
