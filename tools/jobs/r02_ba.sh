timeout 900 python -m pytest tests/test_gpu_balanced.py -q -x -p no:cacheprovider -k "stream" 2>&1 | tail -1
for wm in 0 1 0 1; do
HBP_WARP_MAP=$wm timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static" --rounds 3 --iters 10 2>&1 | tail -1 | cut -c1-220 | sed "s/^/wm=$wm /"
done
for wm in 0 1; do
HBP_WARP_MAP=$wm timeout 600 python tools/ab_ticket.py --config H --runs "static" --rounds 3 --iters 10 2>&1 | tail -1 | cut -c1-220 | sed "s/^/wm=$wm /"
HBP_WARP_MAP=$wm timeout 600 python tools/ab_ticket.py --config cfg5 --runs "static" --rounds 3 --iters 10 2>&1 | tail -1 | cut -c1-220 | sed "s/^/wm=$wm /"
done
