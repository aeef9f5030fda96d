export PATH=/usr/local/cuda/bin:$PATH
for nt in 256 512; do
HBP_ROWSTAGE_THREADS=$nt timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmv_row|k_csr" --csv python tools/ab_sched.py --config cfg1 --flush --runs rowblock,rowstage --rounds 1 --iters 5 2>/dev/null | grep -E "k_spmv_row|k_csr" | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head; echo "--- nt=$nt"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csr" --csv python bench.py --config cfg1 --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | grep -E "csr" | awk -F'","' '{print $5, $NF}' | tail -5
