"""Row-stripe sharding on the CUDA path (stripes.StripedOperator /
PowerIteration) with two processes sharing one B200 over gloo -- the
multi-GPU code the bench runs under torchrun/NCCL, exercised here without a
second GPU.

- every rank's stripe blocks (hash permutations, slot lengths, group
  starts) equal the single-process build's blocks for those rows (the
  global (a, c) draw), bitwise;
- a single SpMV of the stripes, concatenated, equals the single-process y
  (f64 bitwise; exact mode);
- the power iteration over two stripes -- with and without the own-column
  split that overlaps the all-gather -- matches the single-process power
  iteration (f32: within 1e-5; f64 unsplit: bitwise);
- the fused power iteration (the SpMV kernel stores y into the peer's x
  buffer through a CUDA IPC mapping; no all-gather) equals the all-gather
  one bitwise.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

R = 512


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(n, seed, dtype):
    """Square power-law-ish matrix in CSR (host), rows not a multiple of R."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.zipf(1.8, n), n // 3)
    r = np.repeat(np.arange(n), lens)
    c = np.concatenate([rng.choice(n, k, replace=False) for k in lens])
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    v = rng.uniform(-1, 1, r.size).astype(dtype)
    rp = np.concatenate(([0], np.cumsum(np.bincount(r, minlength=n)))).astype(np.int64)
    return rp, c.astype(np.int32), v


def _worker(rank, world, port, n, dtype_name, split, out):
    import torch
    import torch.distributed as dist
    import paper_2504_08860_b200 as H
    from paper_2504_08860_b200.stripes import (PowerIteration, StripedOperator, plan_stripes,
                                               row_block_nnz)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dtype = np.float64 if dtype_name == "f64" else np.float32
    rp, ci, v = _matrix(n, 11, dtype)
    dev = torch.device("cuda", 0)
    rp_d = torch.as_tensor(rp, device=dev)
    stripes = plan_stripes(row_block_nnz(rp_d, n, R), n, R, world)
    cfg = H.PartitionConfig(col_width=n, row_height=R, warp_size=32)
    res = {}
    g = StripedOperator(n, n, rp_d, torch.as_tensor(ci, device=dev), torch.as_tensor(v, device=dev),
                        stripes, rank, cfg, x_layout="global")
    res["params"] = (g.params.a, g.params.b, g.params.c, g.params.d)
    res["perm"] = g.hbp.perm.cpu().numpy()
    res["slot_len"] = g.hbp.slot_len.cpu().numpy()
    x = np.random.default_rng(3).uniform(-1, 1, n).astype(dtype)
    y = torch.empty(g.stripe.rows, dtype=g.dtype, device=dev)
    g(torch.as_tensor(x, device=dev), y)
    res["y"] = y.cpu().numpy()
    res["stripe"] = (g.stripe.row_lo, g.stripe.row_hi)
    p = StripedOperator(n, n, rp_d, torch.as_tensor(ci, device=dev), torch.as_tensor(v, device=dev),
                        stripes, rank, cfg, x_layout="padded", split_own=split)
    res["split"] = p.split
    pit = PowerIteration(p, torch.as_tensor(x, device=dev))
    for _ in range(5):
        pit.step()
    res["x"] = pit.x_global().cpu().numpy()
    if not split:
        # fused: y rows stored into the peer's x buffer (CUDA IPC) by the SpMV
        # kernel itself, no all-gather
        fz = PowerIteration(p, torch.as_tensor(x, device=dev), fused=True)
        for _ in range(5):
            fz.step()
        res["x_fused"] = fz.x_global().cpu().numpy()
        res["fused"] = fz.fused
        fz.close()
    torch.cuda.synchronize()
    out[rank] = res
    dist.destroy_process_group()


def _single(n, dtype):
    import torch
    import paper_2504_08860_b200 as H
    rp, ci, v = _matrix(n, 11, dtype)
    cfg = H.PartitionConfig(col_width=n, row_height=R, warp_size=32)
    csr = H.CsrMatrix(n, n, rp, ci, v)
    grid = H.make_grid(csr, cfg)
    params = H.sample_hash_params(grid, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, params))
    x = np.random.default_rng(3).uniform(-1, 1, n).astype(dtype)
    op = H.SpmvOperator(hbp)
    y = op(torch.as_tensor(x, device="cuda")).cpu().numpy()
    xi = x.astype(np.float64)
    xk = torch.as_tensor(x, device="cuda")
    for _ in range(5):
        yk = op(xk)
        xk = yk / torch.sqrt((yk.double() ** 2).sum()).to(yk.dtype)
    xs = xk.double().cpu().numpy()
    return hbp, params, y, xs / np.sqrt((xs ** 2).sum()), xi


@pytest.mark.parametrize("dtype_name,split", [("f64", False), ("f32", False), ("f32", True)])
def test_two_stripes_on_one_gpu(dtype_name, split):
    import torch.multiprocessing as mp
    n = 5000
    dtype = np.float64 if dtype_name == "f64" else np.float32
    hbp, params, y_ref, x_ref, _ = _single(n, dtype)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), n, dtype_name, split, out), nprocs=2, join=True)
    perm_full = hbp.perm.cpu().numpy().reshape(-1, R)
    len_full = hbp.slot_len.cpu().numpy().reshape(-1, R)
    br_full = hbp.blk_br.cpu().numpy()
    ys = []
    for k in range(2):
        o = out[k]
        assert o["params"] == (params.a, params.b, params.c, params.d)
        lo, hi = o["stripe"]
        sel = (br_full * R >= lo) & (br_full * R < hi)  # C = cols: one block per row block
        np.testing.assert_array_equal(o["perm"].reshape(-1, R), perm_full[sel])
        np.testing.assert_array_equal(o["slot_len"].reshape(-1, R), len_full[sel])
        ys.append(o["y"])
        assert o["split"] == split
    y = np.concatenate(ys)
    if dtype == np.float64:
        np.testing.assert_array_equal(y, y_ref)
    else:
        np.testing.assert_allclose(y, y_ref, rtol=0, atol=1e-5 * np.abs(y_ref).max())
    for k in range(2):
        if not split:  # the fused step computes the same values: bitwise
            assert out[k]["fused"]
            np.testing.assert_array_equal(out[k]["x_fused"], out[k]["x"])
        if dtype == np.float64 and not split:
            np.testing.assert_allclose(out[k]["x"], x_ref, rtol=1e-13, atol=1e-15)
        else:
            np.testing.assert_allclose(out[k]["x"], x_ref, rtol=0, atol=2e-5)
