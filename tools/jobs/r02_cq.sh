export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_rowblock.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -1
for r in 1 2; do for v in old new; do
HBP_LIB_PATH=_prev/libhbp_$v.so timeout 600 python tools/ab_sched.py --config cfg1 --flush --runs rowstage --rounds 5 --iters 20 2>&1 | tail -1 | sed "s/^/$v /"
done; done
for v in old new; do
HBP_LIB_PATH=_prev/libhbp_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmv_rowstage|k_csr" -c 12 --csv python bench.py --config cfg1 --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | grep -v "==" | awk -F'","' 'NR>1{print substr($5,1,30), $NF}' | sed "s/^/$v /"
done
