export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python tools/ab_colwidth.py --config cfg5 --widths 0,33554432,16777216 2>&1 | grep -v Warn | tail -5
timeout 600 python tools/ab_colwidth.py --config cfg2 --widths 0,8388608 2>&1 | grep -v Warn | tail -3
timeout 600 python tools/ab_colwidth.py --config H --widths 0,3125000 2>&1 | grep -v Warn | tail -3
