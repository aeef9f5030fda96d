export PATH=/usr/local/cuda/bin:$PATH
for c in cfg4 cfg2 cfg3; do
for t in 0 1; do
HBP_HASH_THREAD=$t timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hash_perm" --csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 1 --warmup 3 2>/dev/null | grep k_hash | awk -F'","' '{print substr($5,1,45), $NF}' | head -1 | sed "s/^/form=$t $c /"
done
done
