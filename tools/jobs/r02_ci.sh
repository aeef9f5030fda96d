for c in cfg2 cfg4 cfg1; do
s=$(date +%s)
timeout 1200 python bench.py --impl reference --config $c --steps 20 --warmup 3 > gpurun_out/bref_$c.json 2> gpurun_out/bref_$c.err; echo "$c rc=$? wall=$(( $(date +%s) - s ))s"
python -c "import json;d=json.loads(open('gpurun_out/bref_$c.json').read().splitlines()[-1]);print('$c',d['value'],d['ms_per_step'],d['cpu_baseline']['sample'][:100],d['preprocess_ms'],d['cpu_arms'])" || tail -5 gpurun_out/bref_$c.err
done
