"""A/B the stream kernel's variants in one process, interleaved, on one config.

    python tools/ab_variants.py --config cfg2 --variants 0,3 [--rounds 5 --iters 10]

Variants of one operator differ only in the kernel instantiation
(hbp_stream_set_variant); each round times every variant back to back so box-to-box
and drift effects cancel.  Workers must match (same launch geometry) -- variants with
another CTA shape get their own operator.
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
ap.add_argument("--config", default="cfg2")
ap.add_argument("--variants", default="0,3")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--hot", default="auto")
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
hot = {"auto": None, "on": True, "off": False}.get(a.hot, None)
variants = [int(v) for v in a.variants.split(",")]
ops = {}
for v in variants:
    L.call("hbp_stream_set_variant", L.c_int(v))
    ops[v] = H.SpmvOperator(hbp, hot=hot)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
y = torch.empty(rows, dtype=vdt, device=dev)
res = {v: [] for v in variants}
ref = None
for r in range(a.rounds):
    for v in variants:
        L.call("hbp_stream_set_variant", L.c_int(v))
        ops[v](x, y)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.iters):
            ops[v](x, y)
        e.record()
        torch.cuda.synchronize()
        res[v].append(s.elapsed_time(e) / a.iters)
for v in variants:
    ms = statistics.median(res[v])
    print(f"{a.config} variant {v}: median {ms:.4f} ms  min {min(res[v]):.4f}  "
          f"GFLOP/s {2 * hbp.nnz / ms / 1e6:.1f}")
