export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_hot.py -q -x -p no:cacheprovider 2>&1 | tail -2
for kb in 155 170; do
HBP_HOT_BUDGET_KB=$kb timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/c=64,24,48" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2 | sed "s/^/kb=$kb /"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hot_gather|k_spmv_stream" -c 6 --csv python tools/e2e_probe.py cfg2 2 2>/dev/null | grep -E "k_hot|k_spmv" | awk -F'","' '{print substr($5,1,40), $NF}' | tail -6
