timeout 900 python -m pytest tests/test_gpu_rowblock.py -q -x -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
