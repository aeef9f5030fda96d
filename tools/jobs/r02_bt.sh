timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/t=0.9:8/t=0.95:8/t=0.97:4" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -4 | cut -c1-220
