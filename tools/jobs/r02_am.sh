for kb in 160 170 155; do
HBP_HOT_BUDGET_KB=$kb timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/c=64,24,48/c=80,28,56" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -3 | sed "s/^/kb=$kb /"
done
