"""Per-warp cost model of the stream kernel: time every persistent warp
(%globaltimer, SpmvOperator.warp_clock) and regress its busy time on the
work features of its slice (elements by phase kind, phases by kind, groups,
hot-tier gathers).  The fitted per-unit costs feed the cost-balanced slicing.

    python tools/warp_cost.py --config cfg2 [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402


def popcount32(v: torch.Tensor) -> torch.Tensor:
    v = v.to(torch.int64) & 0xFFFFFFFF
    v = v - ((v >> 1) & 0x55555555)
    v = (v & 0x33333333) + ((v >> 2) & 0x33333333)
    v = (v + (v >> 4)) & 0x0F0F0F0F
    return ((v * 0x01010101) & 0xFFFFFFFF) >> 24


def phase_table(hbp):
    """Absolute start, length, live-lane count and kind of every phase."""
    gs = hbp.group_start_c
    ptr = hbp.phase_ptr
    nph = ptr[1:] - ptr[:-1]
    total = int(ptr[-1].item())
    ph = hbp.phases[: 2 * total].view(total, 2)
    mask, off = ph[:, 0], ph[:, 1].to(torch.int64)
    g_of = torch.repeat_interleave(torch.arange(nph.numel(), device=gs.device), nph)
    start = gs[:-1][g_of] + off
    end = torch.empty_like(start)
    end[:-1] = start[1:]
    end[-1] = gs[-1]
    last = torch.zeros(total, dtype=torch.bool, device=gs.device)
    last[(ptr[1:] - 1)[nph > 0]] = True
    end[last] = gs[1:][g_of[last]]  # a group's last phase ends at the group end
    k = popcount32(mask)
    ln = end - start
    kind = torch.full_like(k, 2)  # step loop
    kind[(k < 12) & (ln > 4 * k)] = 1  # modular passes
    kind[ln <= 2 * k] = 0  # one or two steps
    return start, ln, k, kind


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(a.config, 0, dev)
    cfg = H.PartitionConfig(col_width=C)
    csr = H.CsrMatrix(rows, cols, rp, col, val)
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                      with_add_sign=False, with_zero_row=False)
    del csr, grid, col, val
    op = H.SpmvOperator(hbp, schedule="stream")
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, cols), device=dev).to(vdt)
    y = torch.empty(rows, dtype=vdt, device=dev)
    for _ in range(3):
        op(x, y)
    clk = op.warp_clock()
    times = []
    for _ in range(a.reps):
        op(x, y)
        torch.cuda.synchronize()
        t = clk.cpu().numpy().astype(np.float64)
        times.append((t[:, 1] - t[:, 0]) / 1e3)
    busy = np.median(np.stack(times), axis=0)  # us per warp
    sl = op._scratch[[i for i, s in enumerate(op._scratch)
                      if s.dtype == torch.int64 and s.numel() == op.workers + 1][0]]
    lo, hi = sl[:-1], sl[1:]

    start, ln, k, kind = phase_table(hbp)
    order = torch.argsort(start)
    start, ln, k, kind = start[order], ln[order], k[order], kind[order]
    feats, names = [], []

    def count_in(pos, weight=None):
        a_ = torch.searchsorted(pos, lo)
        b_ = torch.searchsorted(pos, hi)
        if weight is None:
            return (b_ - a_).double()
        cw = torch.cat([torch.zeros(1, dtype=torch.float64, device=dev),
                        torch.cumsum(weight.double(), 0)])
        return cw[b_] - cw[a_]

    for kd, nm in ((0, "short"), (1, "modular"), (2, "step")):
        sel = kind == kd
        feats.append(count_in(start[sel]))
        names.append(f"phases_{nm}")
        feats.append(count_in(start[sel], ln[sel]))
        names.append(f"elems_{nm}")
    gs = hbp.group_start_c[:-1].contiguous()
    feats.append(count_in(gs))
    names.append("groups")
    if op.hot is not None:
        hot = (op.hot.scol[: hbp.nnz].view(torch.int32) < 0)
        ch = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(hot, 0)])
        feats.append((ch[hi] - ch[lo]).double())
        names.append("hot_elems")
    X = torch.stack(feats, 1).cpu().numpy()
    X1 = np.concatenate([X, np.ones((X.shape[0], 1))], 1)
    coef, *_ = np.linalg.lstsq(X1, busy, rcond=None)
    pred = X1 @ coef
    r2 = 1 - ((busy - pred) ** 2).sum() / ((busy - busy.mean()) ** 2).sum()
    print(f"{a.config}: {op.workers} warps, busy us p1/p50/p99/max "
          f"{np.percentile(busy, 1):.1f}/{np.median(busy):.1f}/{np.percentile(busy, 99):.1f}/"
          f"{busy.max():.1f}")
    tot = X.sum(0)
    for n, c_, s in zip(names + ["const"], coef, list(tot) + [op.workers]):
        print(f"  {n:16s} {c_ * 1e3:10.3f} ns/unit   total units {s:14.0f}   "
              f"share of warp time {c_ * s / busy.sum():.3f}")
    print(f"  R^2 {r2:.3f}; residual p99 {np.percentile(np.abs(busy - pred), 99):.1f} us")
    # correlation of busy time with each feature
    for n, col_ in zip(names, X.T):
        print(f"  corr(busy, {n}) = {np.corrcoef(busy, col_)[0, 1]:+.3f}")
    np.savez(os.path.join("gpurun_out", f"warp_cost_{a.config}.npz"), busy=busy, X=X,
             names=np.array(names))


if __name__ == "__main__":
    main()
