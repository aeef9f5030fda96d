export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python tools/ab_sched.py --config cfg1 --flush --runs rowstage,seg:0,rowblock,stream --rounds 5 --iters 20 2>&1 | tail -6
