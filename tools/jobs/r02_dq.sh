export PATH=/usr/local/cuda/bin:$PATH
for ck in "cfg2d:k_spmv_stream" "cfg3:k_spmv_seg" "cfg1:k_spmv_rowstage"; do c=${ck%%:*}; k=${ck##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o /tmp/full_$c python bench.py --config $c --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > gpurun_out/ncu_f_$c.log 2>&1; echo "full $c rc=$?"
ncu -i /tmp/full_$c.ncu-rep --page raw --csv > gpurun_out/r02j_ncu_${c}_raw.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02j_launches_$c.csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 2 --warmup 3 > /dev/null 2>&1; echo "launches $c rc=$?"
done
