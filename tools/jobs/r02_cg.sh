export PATH=/usr/local/cuda/bin:$PATH
for c in cfg5 cfg4 cfg2d cfg1 cfg3; do
case $c in cfg1) k=k_spmv_rowstage;; cfg3) k=k_spmv_seg;; *) k=k_spmv_stream;; esac
timeout 900 ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -o /tmp/r02e_full_$c python bench.py --config $c --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > /dev/null 2>&1; echo "full $c rc=$?"
ncu -i /tmp/r02e_full_$c.ncu-rep --page raw --csv > gpurun_out/r02e_raw_$c.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02e_launches_$c.csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > /dev/null 2>&1; echo "launches $c rc=$?"
done
for c in H cfg2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02e_launches_$c.csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > /dev/null 2>&1; echo "launches $c rc=$?"
done
du -sh gpurun_out
