timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_bz.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error" gpurun_out/gpu_tests_bz.log | head -20; tail -2 gpurun_out/gpu_tests_bz.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
