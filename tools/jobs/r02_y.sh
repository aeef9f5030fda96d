timeout 900 python tools/prof_sched.py 2>&1 | tail -16
