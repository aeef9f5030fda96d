for c in cfg2 cfg5 H; do
timeout 600 python tools/ab_ticket.py --config $c --runs "static/c=64,20,40/c=66,24,48/c=80,24,48/c=96,28,56" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -5
done
