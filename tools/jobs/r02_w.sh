timeout 900 python -m pytest tests/test_gpu_rowblock.py -q -x -p no:cacheprovider > gpurun_out/rowstage_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rowstage_tests.log
grep -E "^E " gpurun_out/rowstage_tests.log | head -10
for nt in 512 256; do
HBP_ROWSTAGE_THREADS=$nt timeout 600 python tools/ab_sched.py --config cfg1 --flush --runs rowblock,rowstage --rounds 5 --iters 20 2>&1 | tail -2 | sed "s/^/nt=$nt /"
done
timeout 600 python bench.py --config cfg1 --no-cpu-baseline --schedule rowstage --steps 20 > gpurun_out/b_cfg1_rs.json 2> gpurun_out/b_cfg1_rs.err; python -c "import json;d=json.loads(open('gpurun_out/b_cfg1_rs.json').read().splitlines()[-1]);print('cfg1 rowstage',d['ms_per_step'],d['value'],d['roofline']['frac'],d['baselines_same_gpu'])" || tail -3 gpurun_out/b_cfg1_rs.err
