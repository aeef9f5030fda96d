export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_rowblock.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "rowstage or cfg1" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
for xv in 1 0; do
HBP_ROWSTAGE_X=$xv timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmv_rowstage" --csv python tools/ab_sched.py --config cfg1 --flush --runs rowstage --rounds 1 --iters 6 2>/dev/null | grep -E "k_spmv_row" | awk -F'","' '{print substr($5,1,60), $NF}' | tail -4 | sed "s/^/X=$xv /"
done
