for kb in 155 185 200 170; do
HBP_HOT_BUDGET_KB=$kb timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static" --rounds 3 --iters 10 2>&1 | tail -1 | cut -c1-120 | sed "s/^/kb=$kb /"
done
