export PATH=/usr/local/cuda/bin:$PATH
for L in 128 1024 1000000000; do
HBP_PACKED_LIGHT=$L timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static" --rounds 3 --iters 10 2>&1 | tail -1 | cut -c1-120 | sed "s/^/light=$L /"
HBP_PACKED_LIGHT=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none -k regex:"k_hot_gather|k_spmv_stream" -c 4 --csv python tools/e2e_probe.py cfg2 1 2>/dev/null | grep -E "k_hot|k_spmv" | awk -F'","' '{print substr($5,1,30), $(NF-2), $NF}' | tail -4
done
