for kb in 131 115 100 85 115; do
HBP_HOT_BUDGET_KB=$kb timeout 600 python tools/ab_ticket.py --config cfg5 --runs "static" --rounds 3 --iters 6 2>&1 | tail -1 | cut -c1-120 | sed "s/^/kb=$kb /"
done
