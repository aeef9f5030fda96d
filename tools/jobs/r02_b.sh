timeout 900 python -m pytest tests/test_gpu_errors.py tests/test_gpu_balanced.py tests/test_gpu_parity.py tests/test_gpu_pipeline.py -x -q -p no:cacheprovider > gpurun_out/gpu_tests_b.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests_b.log
