"""A/B of the column-block width C on one bench matrix: build the HBP format at
each C, time the default SpmvOperator (CUDA events, inputs resident), check y
against the first C's result.

    python tools/ab_colwidth.py --config cfg5 --widths 0,33554432,16777216
(0 = cols)
"""
import argparse
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--widths", default="0")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--schedule", default=None)
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C0, vdt = bench.make_matrix_gpu(a.config, 0, dev)
csr = H.CsrMatrix(rows, cols, rp, col, val)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
nnz = int(rp[-1].item())
y0 = None
for w in [int(v) for v in a.widths.split(",")]:
    C = w or cols
    cfg = H.PartitionConfig(col_width=C)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                      with_add_sign=False, with_zero_row=False)
    del grid
    op = H.SpmvOperator(hbp, schedule=a.schedule)
    y = torch.empty(rows, dtype=vdt, device=dev)
    for _ in range(3):
        op(x, y)
    best = []
    for _ in range(a.rounds):
        torch.cuda.synchronize()
        t0.record()
        for _ in range(a.iters):
            op(x, y)
        t1.record()
        torch.cuda.synchronize()
        best.append(t0.elapsed_time(t1) / a.iters)
    if y0 is None:
        y0 = y.double().clone()
        err = 0.0
    else:
        err = float((y.double() - y0).abs().max() / y0.abs().max())
    ms = min(best)
    print(f"{a.config} C={C} ncb={hbp.num_col_blocks} nzb={hbp.nzb} schedule={op.schedule} "
          f"hot={'none' if op.hot is None else (op.hot.n_hot, op.hot.n_warm)} "
          f"launches={op.launches_per_call} ms={ms:.4f} (rounds {[round(b, 4) for b in best]}) "
          f"GFLOP/s={2 * nnz / ms / 1e6:.1f} maxabs_rel_vs_first={err:.2e}", flush=True)
    del op, hbp, y
    gc.collect()
    torch.cuda.empty_cache()
