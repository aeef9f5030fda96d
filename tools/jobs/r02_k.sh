timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_k.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error" gpurun_out/gpu_tests_k.log | head -20; tail -3 gpurun_out/gpu_tests_k.log
