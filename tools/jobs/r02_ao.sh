timeout 900 python -m pytest tests/test_gpu_hot.py -q -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -20
timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/c=64,24,48" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2
