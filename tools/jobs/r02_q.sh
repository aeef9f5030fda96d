timeout 900 python -m pytest tests/test_gpu_balanced.py -q -x -p no:cacheprovider -k "ticket" > gpurun_out/ticket_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/ticket_tests.log
for c in cfg2 H cfg5 cfg4; do
timeout 600 python tools/ab_ticket.py --config $c --runs static,0.7:1,0.7:2,0.5:4,0.9:1,w2 --rounds 3 --iters 10 2>&1 | tail -8
done
