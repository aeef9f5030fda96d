export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none -k regex:"k_hot_gather|k_spmv_stream" -c 8 --csv python tools/e2e_probe.py cfg2 2 2>/dev/null | grep -E "k_hot|k_spmv" | awk -F'","' '{print substr($5,1,40), $(NF-2), $NF}' | tail -8
