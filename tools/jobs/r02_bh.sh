for px in 0 1; do
HBP_PACKED_X=$px timeout 900 python tools/ab_ticket.py --config cfg2d --runs "hub" --rounds 3 --iters 5 2>&1 | tail -1 | cut -c1-220 | sed "s/^/px=$px /"
done
