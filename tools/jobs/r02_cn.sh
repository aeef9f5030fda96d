export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_|Device|cub" -c 80 --csv python bench.py --config cfg3 --no-cpu-baseline --no-baselines --steps 1 --warmup 1 2>/dev/null | grep -v "==" | awk -F'","' 'NR>1{print substr($5,1,60), $NF}' | head -80
