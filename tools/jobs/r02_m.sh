timeout 600 python -m pytest tests/test_gpu_hub.py tests/test_gpu_balanced.py tests/test_gpu_hot.py -x -q -p no:cacheprovider 2>&1 | tail -2
