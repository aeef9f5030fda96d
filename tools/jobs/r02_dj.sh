export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x -p no:cacheprovider 2>&1 | tail -30
