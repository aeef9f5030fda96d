timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/c=64,24,48/c=32,16,32/c=48,30,30" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -4 | cut -c1-200
