timeout 600 python tools/ab_ticket.py --config H --runs "eq/1.0:1/0.95:1" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -3 | cut -c1-220
timeout 600 python tools/ab_ticket.py --config cfg2 --runs "eq/static/1.0:1/0.95:1" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -4 | cut -c1-220
