timeout 600 python tools/ab_sched.py --config cfg3 --ff 0.0 --runs seg:9,seg:11,seg:12,seg:13,seg:14,seg:15 --rounds 3 --iters 5 2>&1 | tail -6
timeout 600 python tools/ab_sched.py --config cfg1 --flush --ff 0.0 --runs rowblock,seg:9,seg:11,seg:12,seg:13,seg:14,seg:15 --rounds 3 --iters 20 2>&1 | tail -7
