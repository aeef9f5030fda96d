"""A/B the SpMV schedules (and the seg kernel's launch shapes) on one config,
interleaved in one process.

    python tools/ab_sched.py --config cfg3 --runs seg:0,seg:1,stream [--flush]

Each run is "schedule[:seg variant]"; every round times each run back to back
(CUDA events), medians reported; y of every run is compared with the first
(bitwise for f64).
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402
from paper_2504_08860_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--runs", default="seg:0,stream")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--flush", action="store_true", help="flush L2 before every SpMV")
ap.add_argument("--ff", type=float, default=None, help="fixed fraction override")
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
del csr, grid, col, val
runs = a.runs.split(",")
ops = {}
for r in runs:
    sched, _, var = r.partition(":")
    if sched == "seg":
        L.call("hbp_seg_set_variant", L.c_int(int(var or 0)))
    ops[r] = H.SpmvOperator(hbp, schedule=sched, fixed_fraction=a.ff)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
y = torch.empty(rows, dtype=vdt, device=dev)
scratch = torch.empty(2 * L.l2_bytes() // 4, dtype=torch.float32, device=dev) if a.flush else None
res = {r: [] for r in runs}
ref = None
for rnd in range(a.rounds):
    for r in runs:
        sched, _, var = r.partition(":")
        if sched == "seg":
            L.call("hbp_seg_set_variant", L.c_int(int(var or 0)))
        ops[r](x, y)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        elif rnd == 0:
            same = bool(torch.equal(ref, y))
            err = float((ref.double() - y.double()).abs().max())
            print(f"{r}: y {'bitwise equal' if same else 'differs (max abs %.3g)' % err} vs {runs[0]}")
        ts = []
        for _ in range(a.iters):
            if scratch is not None:
                scratch.fill_(1.0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            ops[r](x, y)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        res[r].append(statistics.median(ts))
esz = 4 if vdt == torch.float32 else 8
b_alg = hbp.nnz * (esz + 4) + (rows + cols) * esz
for r in runs:
    ms = statistics.median(res[r])
    print(f"{a.config} {r:10s} workers {ops[r].workers:6d}: median {ms:.4f} ms  min {min(res[r]):.4f}"
          f"  GFLOP/s {2 * hbp.nnz / ms / 1e6:.1f}  HBM frac {b_alg / ms / 1e6 / 6535.7:.3f}")
