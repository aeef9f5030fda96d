for wb in 67108864 50331648 83886080 100663296; do
HBP_WARM_BYTES=$wb timeout 600 python tools/ab_ticket.py --config cfg5 --runs "static" --rounds 3 --iters 6 2>&1 | tail -1 | cut -c1-120 | sed "s/^/warm=$wb /"
done
