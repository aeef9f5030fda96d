for c in cfg2 H cfg5; do timeout 600 python tools/warp_cost.py --config $c 2>&1 | tail -22; done
