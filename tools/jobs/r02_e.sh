timeout 600 python tools/ab_sched.py --config cfg3 --runs stream,seg:5,seg:6,seg:7,seg:8,seg:9,seg:10 --rounds 3 --iters 5 2>&1 | tail -8
timeout 600 python tools/ab_sched.py --config cfg3 --ff 1.0 --runs seg:5,seg:9 --rounds 3 --iters 5 2>&1 | tail -2
timeout 600 python tools/ab_sched.py --config cfg3 --ff 0.0 --runs seg:5,seg:9 --rounds 3 --iters 5 2>&1 | tail -2
