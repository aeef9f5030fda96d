timeout 600 python -m pytest tests/test_gpu_hub.py tests/test_gpu_balanced.py -x -q -p no:cacheprovider > gpurun_out/hub_tests.log 2>&1; echo "tests rc=$?"
grep -E "^(FAILED|ERROR)|pending CUDA error|Error" gpurun_out/hub_tests.log | head; tail -3 gpurun_out/hub_tests.log
timeout 600 python -m pytest tests/test_gpu_hub.py::test_hub_min_validation tests/test_gpu_balanced.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m pytest "tests/test_gpu_hub.py::test_hub_with_partials_several_column_blocks" tests/test_gpu_balanced.py -x -q -p no:cacheprovider 2>&1 | tail -3
