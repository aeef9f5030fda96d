timeout 900 python -m pytest tests/test_gpu_hot.py -q -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
for kb in 155 170; do
HBP_HOT_BUDGET_KB=$kb timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/c=64,24,48" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2 | sed "s/^/kb=$kb /"
done
timeout 600 python tools/ab_ticket.py --config cfg5 --runs "static/c=64,24,48" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2
timeout 600 python tools/ab_ticket.py --config H --runs "static/c=64,24,48" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2
