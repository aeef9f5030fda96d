timeout 900 python -m pytest tests/test_gpu_balanced.py tests/test_gpu_hot.py tests/test_gpu_scale.py tests/test_gpu_stripes.py -q -x -p no:cacheprovider > gpurun_out/cost_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/cost_tests.log
for c in cfg2 H cfg5 cfg4; do
timeout 600 python tools/ab_ticket.py --config $c --runs "eq/static/c=32,20,40/c=64,20,40/c=48,30,60/c=48,10,20/0.9:1" --rounds 3 --iters 10 2>&1 | grep -v "y max" | tail -8
done
timeout 600 python tools/ab_ticket.py --config cfg2d --runs "eq/c=48,20,40" --rounds 2 --iters 5 2>&1 | tail -3
