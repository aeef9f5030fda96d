"""Time the stages of hot-column staging (HbpMatrix.hot_columns) on a bench
config with CUDA events.

    python tools/prof_hot.py [--config cfg2]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402
from paper_2504_08860_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
cap = L.c_i64(0)
L.call("hbp_hot_capacity", L.c_int(L.dtype_code(hbp.data.dtype)), L.c_int(0), ctypes.byref(cap))
n = int(cap.value)


def stages():
    t = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record()
    deg = torch.zeros(cols, dtype=torch.int32, device=dev)
    stride = 1
    while hbp.nnz // stride > hbp.RANK_SAMPLE:
        stride *= 2
    L.call("hbp_col_degree", L.P(hbp.col), L.c_i64(hbp.nnz), L.c_i64(stride), L.P(deg),
           L.stream())
    ev[1].record()
    keys = (torch.iinfo(torch.int32).max - deg).contiguous()
    vals = torch.arange(cols, dtype=torch.int32, device=dev)
    ev[2].record()
    _, order = L.sort_pairs_u32(keys, vals, 32)
    ev[3].record()
    hot_cols = order[:n].contiguous()
    share = deg[hot_cols.long()].sum()
    slot_of = torch.full((cols,), -1, dtype=torch.int32, device=dev)
    L.call("hbp_hot_slots", L.P(hot_cols), L.c_i64(n), L.P(slot_of), L.stream())
    ev[4].record()
    scol = torch.empty(hbp.nnz + 16, dtype=torch.int32, device=dev)
    L.call("hbp_hot_remap", L.P(hbp.col), L.c_i64(hbp.nnz), L.P(slot_of), L.c_i64(n), L.P(scol),
           L.stream())
    ev[5].record()
    float(share.item())
    ev[6].record()
    torch.cuda.synchronize()
    for i, k in enumerate(["degree", "keys", "sort", "select", "remap", "sync"]):
        t[k] = round(ev[i].elapsed_time(ev[i + 1]), 3)
    return t


stages()
print(a.config, "n_hot", n, stages())
