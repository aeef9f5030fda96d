"""Time the stream and row-block schedules side by side on synthetic matrices
with several column blocks (checks SpmvOperator._auto_schedule's threshold).

    python tools/prof_sched.py

Each line: matrix, dtype, nnz, auto choice, stream / rowblock / rowstage ms (L2
flushed before every timed SpMV, CUDA events, mean of 30).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench_inputs as BI  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402

dev = torch.device("cuda", 0)
scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(op, x, y, iters=30):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        op(x, y)
    ms = 0.0
    for _ in range(iters):
        scratch.fill_(1)
        s.record()
        op(x, y)
        e.record()
        torch.cuda.synchronize()
        ms += s.elapsed_time(e) / iters
    return ms


def run(name, rows, cols, rp, col, val, C):
    cfg = H.PartitionConfig(col_width=C)
    csr = H.CsrMatrix(rows, cols, rp, col, val)
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                      with_add_sign=False, with_zero_row=False)
    x = torch.rand(cols, device=dev, dtype=torch.float64).to(val.dtype)
    y = torch.empty(rows, device=dev, dtype=val.dtype)
    auto = H.SpmvOperator._auto_schedule(hbp)
    t = {}
    for s in ("stream", "rowblock", "rowstage"):
        try:
            t[s] = timed(H.SpmvOperator(hbp, schedule=s), x, y)
        except ValueError:  # rowstage: a row block too large to stage
            t[s] = float("nan")
    print(f"{name:28s} {str(val.dtype)[6:]:8s} nnz={hbp.nnz:>10d} ncb={hbp.num_col_blocks:>5d} "
          f"auto={auto:8s} stream={t['stream']:.4f} rowblock={t['rowblock']:.4f} "
          f"rowstage={t['rowstage']:.4f}", flush=True)


for dt in (torch.float64, torch.float32):
    for rows, mean in ((1 << 18, 16), (1 << 20, 8), (1 << 20, 16), (1 << 21, 16), (1 << 22, 8)):
        r, c, rp, col, val = BI.uniform_csr_torch(rows, rows, mean, 0, dev, dt)
        run(f"uniform {rows}x{mean}", r, c, rp, col, val, 4096)
    for n in (1 << 20, 1 << 22):
        r, c, rp, col, val = BI.banded_csr_torch(n, dev, dt)
        run(f"banded {n}", r, c, rp, col, val, 4096)
