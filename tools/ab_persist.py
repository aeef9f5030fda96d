"""A/B: an L2 persisting access-policy window over the staged x copy (hot +
warm tiers, or the packed copy) during the stream SpMV.

    python tools/ab_persist.py --config cfg5 [--ratios 0,0.5,1.0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402
from paper_2504_08860_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--ratios", default="0,1.0,0.75,0.5,0")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--rounds", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
del grid
op = H.SpmvOperator(hbp)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
y = torch.empty(rows, dtype=vdt, device=dev)
nnz = hbp.nnz
xh = None
if op.hot is not None:
    n = op.hot.n_hot + op.hot.n_warm
    xh = [t for t in op._scratch if t.numel() == n][0]
print(f"{a.config}: hot {op.hot.n_hot if op.hot else 0} warm/packed "
      f"{op.hot.n_warm if op.hot else 0} copy {0 if xh is None else xh.numel() * xh.element_size() >> 20} MB",
      flush=True)
import ctypes  # noqa: E402
l2, mp, mw = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
L.call("hbp_l2_info", ctypes.byref(l2), ctypes.byref(mp), ctypes.byref(mw))
print(f"L2 {l2.value >> 20} MB, max persisting {mp.value >> 20} MB, max window {mw.value >> 20} MB")
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
y0 = None
for r in [float(v) for v in a.ratios.split(",")]:
    if r > 0 and xh is not None:
        L.call("hbp_l2_persist", L.P(xh), ctypes.c_size_t(xh.numel() * xh.element_size()),
               ctypes.c_float(r), L.stream())
    else:
        L.call("hbp_l2_persist_reset", L.stream())
    for _ in range(3):
        op(x, y)
    ts = []
    for _ in range(a.rounds):
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            op(x, y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / a.iters)
    if y0 is None:
        y0 = y.clone()
    print(f"persist hit_ratio {r}: ms {min(ts):.4f} {[round(t, 4) for t in ts]} "
          f"GFLOP/s {2 * nnz / min(ts) / 1e6:.1f} y_equal {bool(torch.equal(y, y0))}", flush=True)
L.call("hbp_l2_persist_reset", L.stream())
