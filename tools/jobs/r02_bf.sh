timeout 900 python tools/ab_ticket.py --config cfg2d --runs "hub/hub:48,20,40/hub:16,8,16" --rounds 3 --iters 5 2>&1 | tail -5 | cut -c1-220
