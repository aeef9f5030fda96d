timeout 600 python -m pytest tests/test_gpu_balanced.py -x -q -p no:cacheprovider -k "default_laplace_64_c512" 2>&1 | tail -5
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_balanced.py -x -q -p no:cacheprovider -k "stream and default_laplace_64_c512" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_balanced.py -x -q -p no:cacheprovider -k "stream" 2>&1 | tail -5
