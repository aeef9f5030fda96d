timeout 900 python -m pytest tests/test_gpu_balanced.py -q -p no:cacheprovider -k "tail" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static/t=0.95:1/t=0.9:1/t=0.97:2" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -4 | cut -c1-220
timeout 600 python tools/ab_ticket.py --config H --runs "static/t=0.95:1" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -2 | cut -c1-220
