export PATH=/usr/local/cuda/bin:$PATH
for t in 0 1; do
for c in cfg3 cfg2 cfg1; do
HBP_HASH_THREAD=$t timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hash_perm" --csv python bench.py --config $c --no-cpu-baseline --no-baselines --steps 1 --warmup 3 2>/dev/null | grep k_hash | awk -F'","' '{print substr($5,1,40), $NF}' | head -3 | sed "s/^/thread=$t $c /"
done
done
