for c in cfg2 cfg5 cfg2d; do
timeout 600 python tools/ab_ticket.py --config $c --runs "static/px" --rounds 3 --iters 10 2>&1 | tail -3
done
