for c in cfg3 cfg5 cfg2; do
HBP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config $c --steps 5 --warmup 3 > gpurun_out/b2_$c.json 2> gpurun_out/b2_$c.err; echo "$c rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/b2_$c.json').read().splitlines()[-1]);print('$c N=2',d['n_gpus'],d['ms_per_step'],d['value'],d['config']['parallelism'],d['config'].get('stripes'),d['config'].get('comm_ms_per_step'),d['config'].get('own_column_split'),d['check'])" || tail -12 gpurun_out/b2_$c.err
done
