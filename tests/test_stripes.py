"""Row-stripe sharding (paper_2504_08860_b200/stripes.py) with world_size 2
over gloo on CPU.  The per-rank compute is the oracle (test
infrastructure); the orchestration -- stripe planning, the global hash
parameter draw, the y all-gather and the power iteration -- is product code.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_08860_b200.stripes import (Stripe, plan_stripes, power_iteration,
                                           sample_hash_params_global)

C, R, W = 128, 64, 8
N = 700  # square, rows not a multiple of R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(n=N, seed=3):
    rng = np.random.default_rng(seed)
    lens = rng.poisson(7, n)
    lens[rng.choice(n, 5, replace=False)] = 150
    r = np.repeat(np.arange(n), lens)
    c = np.concatenate([rng.choice(n, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size)
    return r, c, v


def test_plan_stripes_balanced_and_covering():
    w = np.array([5, 1, 1, 1, 8, 0, 3, 3, 2, 9])
    st = plan_stripes(w, rows=10 * 64 - 7, row_height=64, world=3)
    assert st[0].rb_lo == 0 and st[-1].rb_hi == 10
    for a, b in zip(st, st[1:]):
        assert a.rb_hi == b.rb_lo
    sums = [int(w[s.rb_lo:s.rb_hi].sum()) for s in st]
    assert max(sums) - min(sums) <= max(w)
    assert st[-1].row_hi == 10 * 64 - 7
    assert plan_stripes(w, 640, 64, 1) == [Stripe(0, 0, 10, 0, 640)]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    r, c, v = _matrix()
    rp, ci, vals = O.coo_to_csr(N, N, r, c, v)
    full = O.make_grid(rp, ci, N, N, C, R, W)
    stripes = plan_stripes(full.block_nnz.sum(axis=1), N, R, world)
    s = stripes[rank]
    lo, hi = rp[s.row_lo], rp[s.row_hi]
    rp_l = rp[s.row_lo:s.row_hi + 1] - lo
    g_l = O.make_grid(rp_l, ci[lo:hi], s.rows, N, C, R, W)
    params = sample_hash_params_global(lambda flat: g_l.row_counts.reshape(-1)[flat], s, N,
                                       full.ncb, R, sample_size=200, seed=5)
    params = (params.a, params.b, params.c, params.d)
    perms_l, _ = O.hash_permutations(g_l, params)
    h_l = O.build_hbp(rp_l, ci[lo:hi], vals[lo:hi], g_l, perms_l)
    x0 = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, N))
    x = power_iteration(lambda xx: torch.as_tensor(O.hbp_spmv(h_l, xx.numpy(), workers=2)),
                        x0, stripes, iters=4)
    out[rank] = dict(params=params, perms=perms_l,
                     stripe=s, x=x.numpy())
    dist.destroy_process_group()


def test_world2_matches_single_process():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from oracle import oracle as O
    r, c, v = _matrix()
    rp, ci, vals = O.coo_to_csr(N, N, r, c, v)
    full = O.make_grid(rp, ci, N, N, C, R, W)
    pop = full.row_counts.reshape(-1)
    flat = np.random.default_rng(5).choice(pop.size, 200, replace=False)
    want = O.params_from_sample(pop[flat], R)
    perms, _ = O.hash_permutations(full, want)
    for k in range(world):
        assert out[k]["params"] == want
        s = out[k]["stripe"]
        # stripe blocks are bit-identical to the single-GPU build's blocks
        np.testing.assert_array_equal(out[k]["perms"].reshape(full.ncb, s.rows),
                                      perms.reshape(full.ncb, N)[:, s.row_lo:s.row_hi])
    h = O.build_hbp(rp, ci, vals, full, perms)
    x = np.random.default_rng(0).uniform(-1, 1, N)
    for _ in range(4):
        y = O.hbp_spmv(h, x, workers=2)
        x = y / np.sqrt((y ** 2).sum())
    for k in range(world):
        np.testing.assert_allclose(out[k]["x"], x, rtol=1e-12, atol=1e-15)


def test_padded_columns_and_row_block_nnz():
    from paper_2504_08860_b200.stripes import padded_columns, row_block_nnz
    rp = torch.tensor([0, 2, 2, 5, 6, 9, 9, 10], dtype=torch.int64)  # 7 rows
    np.testing.assert_array_equal(row_block_nnz(rp, 7, 3), [5, 4, 1])
    st = plan_stripes([5, 4, 1], rows=7, row_height=3, world=2)
    assert [(s.row_lo, s.row_hi) for s in st] == [(0, 3), (3, 7)]
    pad = max(s.rows for s in st)  # 4
    cols = torch.arange(7, dtype=torch.int32)
    np.testing.assert_array_equal(padded_columns(cols, st, pad), [0, 1, 2, 4, 5, 6, 7])
    # an empty stripe (fewer row blocks than ranks) owns no column
    st3 = plan_stripes([5, 4, 1], rows=7, row_height=3, world=4)
    pad3 = max(s.rows for s in st3)
    got = padded_columns(cols, st3, pad3).numpy()
    owner = got // pad3
    for c, o in zip(range(7), owner):
        assert st3[o].row_lo <= c < st3[o].row_hi
    assert np.all(np.diff(got) > 0)
