"""Stream schedule on a many-column-block uniform matrix: time the kernel
alone, the combine, and variants (cost slicing off, direct-single off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench_inputs as BI  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402

dev = torch.device("cuda", 0)


def timed(fn, iters=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for dt in (torch.float64, torch.float32):
    r, c, rp, col, val = BI.uniform_csr_torch(1 << 18, 1 << 18, 16, 0, dev, dt)
    cfg = H.PartitionConfig(col_width=4096)
    csr = H.CsrMatrix(r, c, rp, col, val)
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                      with_add_sign=False, with_zero_row=False)
    x = torch.rand(c, device=dev, dtype=torch.float64).to(dt)
    y = torch.empty(r, device=dev, dtype=dt)
    for label, kw in (("default", {}), ("eq slices", {"slice_cost": "0"}),
                      ("workers 1184", {"workers": 1184}), ("workers 296", {"workers": 296})):
        op = H.SpmvOperator(hbp, schedule="stream", **kw)
        t_all = timed(lambda: op(x, y))
        from paper_2504_08860_b200 import _lib as L
        t_k = timed(lambda: op._blocks(op._fmt, x, op.partial, y, L.stream()))
        print(f"{str(dt)[6:]} {label:14s} workers {op.workers:5d} nzb {hbp.nzb} groups "
              f"{hbp.nzb * 16} call {t_all:.4f} ms  kernel {t_k:.4f} ms", flush=True)
