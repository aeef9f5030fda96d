export PATH=/usr/local/cuda/bin:$PATH
for c in cfg2 H; do
HBP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --config $c --steps 5 --warmup 3 > gpurun_out/r02j_bench_N4_gloo_onegpu_$c.json 2> gpurun_out/b4_$c.err; echo "N4 $c rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02j_bench_N4_gloo_onegpu_$c.json').read().splitlines()[-1]);c=d['config'];print(d['n_gpus'], d['ms_per_step'], c.get('stripes'), d.get('check'))" || tail -5 gpurun_out/b4_$c.err
done
HBP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 4 --config cfg1 --steps 1 --warmup 1 > gpurun_out/r02j_ref_N4.json 2> gpurun_out/r4.err; echo "ref N4 rc=$?"; wc -l gpurun_out/r02j_ref_N4.json; tail -c 300 gpurun_out/r02j_ref_N4.json
