export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02j_gpu_tests.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)" gpurun_out/r02j_gpu_tests.log | head; tail -1 gpurun_out/r02j_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
