export PATH=/usr/local/cuda/bin:$PATH
for c in cfg5 cfg2 cfg2d; do timeout 900 python tools/ab_persist.py --config $c 2>&1 | grep -v Warn | tail -8; done
