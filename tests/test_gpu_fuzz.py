"""Randomised geometry sweep: the whole GPU pipeline against the oracle.

Each seeded case draws a matrix (skewed row lengths, empty rows, hub rows,
rows/cols from 1 to ~3000) and a geometry (W in 4..32, R a multiple of W up
to 512, C anywhere from 1 to cols), then checks what the reference's own
acceptance tests check (pkg/tests/test_acceptance.py:52-123) plus the
integer metadata:

- hash parameters (reorder.py:40-136), the six HBP arrays (hbp.py:51-238)
  bit-exact against the oracle's restatement;
- fp64: hbp_spmv bitwise equal to the oracle's engine.py:228-232, and for
  W = 32 every applicable B200 schedule bitwise equal as well;
- fp32: componentwise error <= 1e-5 of (|A||x|)_i (north_star tolerance).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch
    import paper_2504_08860_b200 as H
    from oracle import oracle as O

N_CASES = 150


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    rows = int(rng.integers(1, 3000))
    cols = int(rng.integers(1, 3000))
    lens = rng.poisson(rng.uniform(0.5, 12), rows)
    if rows > 4 and rng.random() < 0.6:  # a few hub rows
        hubs = rng.choice(rows, int(rng.integers(1, 4)), replace=False)
        lens[hubs] = rng.integers(cols // 2, cols + 1, hubs.size)
    if rng.random() < 0.3:  # a band of empty rows
        a = int(rng.integers(0, rows))
        lens[a:a + int(rng.integers(1, 600))] = 0
    lens = np.minimum(lens, cols)
    if lens.sum() == 0:
        lens[int(rng.integers(0, rows))] = 1
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens if k]) if lens.sum() else \
        np.zeros(0, np.int64)
    v = rng.uniform(-1, 1, r.size)
    W = int(rng.choice([4, 8, 16, 32, 32, 32]))
    R = W * int(rng.integers(1, 512 // W + 1))
    C = cols if rng.random() < 0.4 else int(rng.integers(1, cols + 1))
    f32 = bool(rng.random() < 0.4)
    x = rng.uniform(-1, 1, cols)
    if f32:
        v = v.astype(np.float32)
        x = x.astype(np.float32)
    return rows, cols, r, c, v, x, C, R, W, f32


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_geometry_pipeline(seed):
    rows, cols, r, c, v, x, C, R, W, f32 = _case(seed)
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    params = H.sample_hash_params(grid, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, params))

    p = O.pipeline(rows, cols, r, c, np.asarray(v, np.float64), C, R, W)
    assert (params.a, params.b, params.c, params.d) == tuple(p["params"])
    ref = hbp.to_reference()
    for k in ("col", "add_sign", "zero_row", "group_start", "output_hash"):
        assert np.array_equal(ref[k], getattr(p["hbp"], k)), k

    y = H.hbp_spmv(hbp, x).cpu().numpy()
    x64 = np.asarray(x, np.float64)
    if not f32:
        y_ref = O.hbp_spmv(p["hbp"], x64, workers=3)
        assert np.array_equal(y, y_ref), "fp64 hbp_spmv not bitwise the reference"
    else:
        err = O.componentwise_error(rows, r, c, np.asarray(v, np.float64), x64,
                                    np.asarray(y, np.float64))
        assert err <= 1e-5, err


@pytest.mark.parametrize("seed", range(0, N_CASES, 3))
def test_random_geometry_every_schedule_fp64(seed):
    """W = 32, fp64: every schedule the operator accepts is bitwise the
    reference (stream / balanced / plan / rowblock, rowstage and seg where
    the geometry allows them)."""
    rows, cols, r, c, v, x, C, R, _, _ = _case(seed)
    W = 32
    R = max(32, R - R % 32)
    v = np.asarray(v, np.float64)
    x = np.asarray(x, np.float64)
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    p = O.pipeline(rows, cols, r, c, v, C, R, W)
    y_ref = O.hbp_spmv(p["hbp"], x, workers=2)
    xd = torch.as_tensor(x, device="cuda")
    ran = []
    for sched in ("stream", "balanced", "plan", "rowblock", "rowstage", "seg"):
        try:
            op = H.SpmvOperator(hbp, schedule=sched)
        except ValueError:
            continue  # geometry outside this schedule's domain (its documented error)
        y = op(xd).cpu().numpy()
        assert np.array_equal(y, y_ref), sched
        ran.append(sched)
    assert {"stream", "balanced", "plan", "rowblock"} <= set(ran)


@pytest.mark.parametrize("seed", range(1, N_CASES, 5))
def test_random_geometry_codec_and_walk(seed):
    """hbp.py:241-391 on random geometries: the .hbp codec round-trips to the
    same bytes and the same six arrays, and the inverse walk
    (hbp_to_triplets) gives back exactly the canonical input triplets."""
    import io
    rows, cols, r, c, v, x, C, R, W, f32 = _case(seed)
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    buf = io.BytesIO()
    H.serialize_hbp(hbp, buf)
    raw = buf.getvalue()
    back = H.deserialize_hbp(io.BytesIO(raw))
    buf2 = io.BytesIO()
    H.serialize_hbp(back, buf2)
    assert buf2.getvalue() == raw
    a, b = hbp.to_reference(), back.to_reference()
    for k in ("col", "add_sign", "zero_row", "group_start", "output_hash"):
        assert np.array_equal(a[k], b[k]), k
    t = H.hbp_to_triplets(hbp)
    tr = np.asarray(t.row.cpu() if hasattr(t.row, "cpu") else t.row, np.int64)
    tc = np.asarray(t.col.cpu() if hasattr(t.col, "cpu") else t.col, np.int64)
    tv = np.asarray(t.val.cpu() if hasattr(t.val, "cpu") else t.val, np.float64)
    order = np.lexsort((tc, tr))
    ref_order = np.lexsort((c, r))
    assert np.array_equal(tr[order], r[ref_order]) and np.array_equal(tc[order], c[ref_order])
    assert np.array_equal(tv[order], np.asarray(v, np.float64)[ref_order])


@pytest.mark.parametrize("seed", range(24))
def test_random_rmat_fp32_fast_paths(seed):
    """Skewed R-MAT graphs (2^12 .. 2^17 vertices, the bench generator) in
    fp32 through the stream schedule with randomly drawn knobs -- hot-column
    staging on / off, packed x on / off, persistent-warp count, competitive
    pieces (ticket) or tail pieces -- every result within 1e-5 of (|A||x|)_i
    against the oracle, and repeat calls identical (deterministic)."""
    import bench_inputs
    rng = np.random.default_rng(500 + seed)
    scale = int(rng.integers(12, 18))
    n, _, rp, col, val = bench_inputs.rmat_csr_torch(scale, int(rng.integers(4, 17)), seed,
                                                     torch.device("cuda"), torch.float32)
    rows_t = torch.repeat_interleave(torch.arange(n, device="cuda"), rp[1:] - rp[:-1])
    r, c = rows_t.cpu().numpy(), col.cpu().numpy().astype(np.int64)
    v = val.cpu().numpy()
    x = rng.uniform(-1, 1, n).astype(np.float32)
    cfg = H.PartitionConfig(col_width=n)
    csr = H.CsrMatrix(n, n, rp, col, val)
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    knobs = dict(hot=[None, False][int(rng.integers(0, 2))],
                 packed_x=[None, True, False][int(rng.integers(0, 3))],
                 workers=[None, int(rng.integers(1, 5000))][int(rng.integers(0, 2))])
    extra = int(rng.integers(0, 3))
    if extra == 1:
        knobs["ticket"] = ["0.7:2", "0.3:5"][int(rng.integers(0, 2))]
    elif extra == 2:
        knobs["tail"] = ["0.9:2", "0.6:4"][int(rng.integers(0, 2))]
    op = H.SpmvOperator(hbp, schedule="stream", **knobs)
    xd = torch.as_tensor(x, device="cuda")
    y = op(xd).cpu().numpy()
    np.testing.assert_array_equal(op(xd).cpu().numpy(), y)
    err = O.componentwise_error(n, r, c, v.astype(np.float64), x.astype(np.float64),
                                y.astype(np.float64))
    assert err <= 1e-5, (knobs, err)
