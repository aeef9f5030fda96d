"""Run the gather-ceiling calibration on a bench config's element stream.

    python tools/gather_ceiling.py [--config cfg2]

Builds the HBP matrix (so the column stream is in HBP element order) and
times gather_ceiling.cu over it, next to the production SpMV kernel.
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
a = ap.parse_args()
so = os.path.join(ROOT, "tools", "libgather.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                       "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", so,
                       os.path.join(ROOT, "tools", "gather_ceiling.cu")])
lib = ctypes.CDLL(so)
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
n = hbp.nnz
sms = torch.cuda.get_device_properties(0).multi_processor_count


def timeit(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


for order, c_arr, v_arr in (("hbp", hbp.col, hbp.data), ("csr", csr.col_idx, csr.values)):
    for blocks_per_sm in (4, 8):
        for unroll in (1, 2, 4):
            out = torch.empty(sms * blocks_per_sm * 256, device=dev)
            ms = timeit(lambda: lib.gather_ceiling(
                ctypes.c_void_p(c_arr.data_ptr()), ctypes.c_void_p(v_arr.data_ptr()),
                ctypes.c_void_p(x.data_ptr()), ctypes.c_int64(n), ctypes.c_void_p(out.data_ptr()),
                sms * blocks_per_sm, unroll, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
            print(f"gather_ceiling order={order} blocks/SM={blocks_per_sm} unroll={unroll}: "
                  f"{ms:.4f} ms  ({2 * n / ms / 1e6:.1f} GFLOP/s)")
op = H.SpmvOperator(hbp)
y = torch.empty(rows, dtype=vdt, device=dev)
print(f"k_spmv_{op.schedule}: {timeit(lambda: op(x, y)):.4f} ms")
