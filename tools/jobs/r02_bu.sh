timeout 600 python tools/warp_cost.py --config cfg2 --reps 5 2>&1 | tail -22
