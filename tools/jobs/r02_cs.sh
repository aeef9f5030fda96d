export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmv_rowstage" -s 2 -c 1 -o /tmp/rs python bench.py --config cfg1 --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1
ncu -i /tmp/rs.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/rs_source.csv 2>&1
ncu -i /tmp/rs.ncu-rep --page raw --csv > gpurun_out/rs_raw.csv 2>&1
ls -la gpurun_out/rs_*
