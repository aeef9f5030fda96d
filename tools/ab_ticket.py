"""A/B of the stream kernel's work distribution on one config, interleaved in
one process: static equal slices (default) vs competitive pieces (fixed
fraction of the elements as one piece per warp, the rest claimed by an atomic
ticket -- engine.py:137-176 applied to element slices) vs more, hardware-
scheduled warps.  Also prints the per-warp end-time spread of each run
(%globaltimer, SpmvOperator.warp_clock) -- the most a dynamic schedule can win.

    python tools/ab_ticket.py --config cfg2 --runs eq,static,c=48,20,40,0.7:2,w2

(runs are separated by "/" when a cost spec holds commas: --runs "eq/c=48,20,40")
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

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--runs", default="static,0.7:1,0.7:2,0.5:4,w2")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
del csr, grid, col, val
runs = a.runs.split("/") if "/" in a.runs else a.runs.split(",")
ops = {}
for r in runs:
    if r == "static":  # the default (cost-balanced slices in fast mode)
        ops[r] = H.SpmvOperator(hbp, schedule="stream")
    elif r.startswith("hub"):  # f64 hub-row path, optional cost weights: hub or hub:48,20,40
        ops[r] = H.SpmvOperator(hbp, schedule="stream", hub_min="auto",
                                slice_cost=r[4:] if ":" in r else None)
    elif r.startswith("t="):  # tail pieces: t=0.95:1
        ops[r] = H.SpmvOperator(hbp, schedule="stream", tail=r[2:])
    elif r.startswith("hubt="):  # hub path + tail pieces
        ops[r] = H.SpmvOperator(hbp, schedule="stream", hub_min="auto", tail=r[5:])
    elif r == "px":  # packed x: degree-ordered compact copy of the used columns
        ops[r] = H.SpmvOperator(hbp, schedule="stream", packed_x=True)
    elif r == "eq":  # equal-element slices
        ops[r] = H.SpmvOperator(hbp, schedule="stream", slice_cost="0")
    elif r.startswith("c="):  # cost weights w_group,w_phase,w_modular
        ops[r] = H.SpmvOperator(hbp, schedule="stream", slice_cost=r[2:])
    elif r.startswith("w"):  # k x the resident warps, scheduled by the hardware
        base = H.SpmvOperator(hbp, schedule="stream").workers
        ops[r] = H.SpmvOperator(hbp, schedule="stream", workers=int(float(r[1:]) * base))
    else:
        ops[r] = H.SpmvOperator(hbp, schedule="stream", ticket=r)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
y = torch.empty(rows, dtype=vdt, device=dev)
res = {r: [] for r in runs}
ref = None
for rnd in range(a.rounds):
    for r in runs:
        ops[r](x, y)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        elif rnd == 0:
            err = float(((ref.double() - y.double()).abs() / (ref.double().abs() + 1e-30)).max())
            print(f"{r}: y {'bitwise equal' if torch.equal(ref, y) else 'max rel diff %.3g' % err}"
                  f" vs {runs[0]}")
        ts = []
        for _ in range(a.iters):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            ops[r](x, y)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        res[r].append(statistics.median(ts))
for r in runs:
    ms = statistics.median(res[r])
    clk = ops[r].warp_clock()
    ops[r](x, y)
    torch.cuda.synchronize()
    t = clk.cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    ends = (t[:, 1] - t0) / 1e3
    starts = (t[:, 0] - t0) / 1e3
    print(f"{a.config} {r:8s} workers {ops[r].workers:6d} pieces {getattr(ops[r], 'pieces', 0):6d}: "
          f"median {ms:.4f} ms min {min(res[r]):.4f} GFLOP/s {2 * hbp.nnz / ms / 1e6:.1f} | "
          f"warp start max {starts.max():.1f} us, end p1/p50/p99/max "
          f"{np.percentile(ends, 1):.1f}/{np.percentile(ends, 50):.1f}/"
          f"{np.percentile(ends, 99):.1f}/{ends.max():.1f} us")
