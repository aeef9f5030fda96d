"""Build one bench matrix and run a few SpMVs (target for ncu / launch lists).

    python tools/prof_spmv.py [--config cfg2] [--schedule stream] [--iters 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--schedule", default=None)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--workers", type=int, default=None)
ap.add_argument("--persist", action="store_true")
ap.add_argument("--flush", action="store_true", help="flush L2 before each timed SpMV (as bench.py does for cfg1)")
ap.add_argument("--hot", default="auto", help="auto | on | off | column count")
ap.add_argument("--persist-warm", action="store_true",
                help="L2 persisting window over the staged x copy (hot + warm tiers)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
hot = {"auto": None, "on": True, "off": False}.get(a.hot, None if a.hot == "auto" else a.hot)
op = H.SpmvOperator(hbp, workers=a.workers, schedule=a.schedule,
                    hot=int(hot) if isinstance(hot, str) else hot)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
y = torch.empty(rows, dtype=vdt, device=dev)
if a.persist_warm and op.hot is not None:
    from paper_2504_08860_b200 import _lib as L
    xh = op._scratch[[t.numel() for t in op._scratch].index(op.hot.n_hot + op.hot.n_warm)]
    L.call("hbp_l2_persist", L.P(xh), xh.numel() * xh.element_size(), 1.0, L.stream())
    print("persisting", xh.numel() * xh.element_size() >> 20, "MB")
if a.persist:
    from paper_2504_08860_b200 import _lib as L
    L.call("hbp_l2_persist", L.P(x), x.numel() * x.element_size(), 1.0, L.stream())
for _ in range(a.iters):
    op(x, y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if a.flush:
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ms = 0.0
    for _ in range(a.iters):
        scratch.fill_(1)
        s.record()
        op(x, y)
        e.record()
        torch.cuda.synchronize()
        ms += s.elapsed_time(e) / a.iters
else:
    s.record()
    for _ in range(a.iters):
        op(x, y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.iters
print(f"{a.config} schedule={op.schedule} workers={op.workers} nnz={csr.nnz} "
      f"hot={op.hot.n_hot if op.hot else 0} ms={ms:.4f} GFLOP/s={2 * csr.nnz / ms / 1e6:.1f}")
