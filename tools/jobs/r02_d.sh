timeout 600 python -m pytest tests/test_gpu_seg.py -x -q -p no:cacheprovider > gpurun_out/seg_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/seg_tests.log
timeout 600 python tools/ab_sched.py --config cfg3 --runs stream,seg:0,seg:1,seg:2,seg:3,seg:4,seg:5 --rounds 3 --iters 5 2>&1 | tail -12
timeout 600 python tools/ab_sched.py --config cfg1 --flush --runs rowblock,seg:0,seg:1,seg:2,seg:3,seg:4,seg:5,stream --rounds 3 --iters 20 2>&1 | tail -12
