timeout 600 python tools/diag_stream_multi.py 2>&1 | tail -8
timeout 900 python tools/prof_sched.py 2>&1 | tail -14
timeout 900 python -m pytest tests/test_gpu_rowblock.py tests/test_gpu_parity.py tests/test_gpu_balanced.py tests/test_gpu_seg.py -q -x -p no:cacheprovider 2>&1 | tail -2
