"""Build one bench matrix's HBP format (target for ncu launch lists of the
preprocessing kernels).

    python tools/prof_build.py [--config cfg2] [--reps 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
torch.cuda.synchronize()
for rep in range(a.reps):
    torch.cuda.nvtx.range_push(f"build{rep}")
    t = [time.perf_counter()]
    grid = H.make_grid(csr, cfg); torch.cuda.synchronize(); t.append(time.perf_counter())
    params = H.sample_hash_params(grid, cfg); torch.cuda.synchronize(); t.append(time.perf_counter())
    perms = H.hash_permutations(grid, params); torch.cuda.synchronize(); t.append(time.perf_counter())
    hbp = H.build_hbp(csr, grid, perms, with_add_sign=False, with_zero_row=False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    hbp.ensure_phases(); torch.cuda.synchronize(); t.append(time.perf_counter())
    torch.cuda.nvtx.range_pop()
    ms = [round((t[i + 1] - t[i]) * 1e3, 3) for i in range(len(t) - 1)]
    print(f"rep {rep}: grid {ms[0]} sample {ms[1]} hash {ms[2]} build {ms[3]} phases {ms[4]} ms")
