timeout 900 python -m pytest tests/test_gpu_balanced.py -q -p no:cacheprovider -k "cost" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
timeout 600 python tools/ab_ticket.py --config cfg2 --runs "c=48,20,40/static/c=49,26,33,76,0/c=60,30,40,90,20" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -4 | cut -c1-220
timeout 600 python tools/ab_ticket.py --config cfg5 --runs "c=48,20,40/static" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2 | cut -c1-220
timeout 600 python tools/ab_ticket.py --config H --runs "c=48,20,40/static" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2 | cut -c1-220
