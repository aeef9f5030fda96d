export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_peers.py tests/test_gpu_stripes.py tests/test_abi.py -q -x -p no:cacheprovider > gpurun_out/peers_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/peers_tests.log; grep -E "^E " gpurun_out/peers_tests.log | head -20
for c in cfg5; do
HBP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config $c --steps 5 --warmup 3 > gpurun_out/b2f_$c.json 2> gpurun_out/b2f_$c.err; echo "$c fused rc=$?"
tail -3 gpurun_out/b2f_$c.err
python -c "import json;d=json.loads(open('gpurun_out/b2f_$c.json').read().splitlines()[-1]);c=d['config'];print(c.get('collective'), c.get('step'), d['ms_per_step'], c.get('comm_ms_per_step'), d.get('check'))"
done
# the stream kernel with the peer-store hook: no regression at N=1 (old = HEAD build)
for r in 1 2; do for v in old new; do for c in cfg2 H; do
HBP_LIB_PATH=_prev/libhbp_$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-baselines --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('$v $c',d['ms_per_step'],d['roofline']['kernel_ms'])"
done; done; done
