for kb in 155 131 110; do
HBP_HOT_BUDGET_KB=$kb timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/c=64,24,48/c=40,16,32" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -3 | sed "s/^/kb=$kb /"
done
