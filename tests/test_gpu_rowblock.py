"""The row-block-owner schedule (hbp_spmv_rowblock: SpMV + combine in one
launch) vs the reference golden vectors and the plan path.

It runs block_spmv over a row block's nonzero blocks in ascending bc and
folds them as combine does, with the plan kernel's per-slot sums, so it is
bitwise equal to hbp_spmv_blocks + hbp_combine for f64 and f32 alike.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_names, has_gpu, load_golden

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch
    import paper_2504_08860_b200 as H
    from oracle import oracle as O


def _hbp(rows, cols, r, c, v, C, R=512, W=32, seed=0):
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    params = H.sample_hash_params(grid, cfg, seed=seed)
    return H.build_hbp(csr, grid, H.hash_permutations(grid, params))


@pytest.mark.parametrize("name", golden_names())
def test_rowblock_matches_golden(name):
    g = load_golden(name)
    val = g["trip_val"].astype(np.float32) if g["fp32"] else g["trip_val"]
    hbp = _hbp(g["rows"], g["cols"], g["trip_row"], g["trip_col"], val, g["C"], g["R"], g["W"],
               g["seed"])
    x = g["x"].astype(np.float32) if g["fp32"] else g["x"]
    op = H.SpmvOperator(hbp, schedule="rowblock")
    assert op.launches_per_call == 1
    y = op(torch.as_tensor(x, device="cuda")).cpu().numpy()
    if g["fp32"]:
        err = O.componentwise_error(g["rows"], g["trip_row"], g["trip_col"], g["trip_val"],
                                    g["x"], y.astype(np.float64))
        assert err <= 1e-5
    else:
        np.testing.assert_array_equal(y, g["y"])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("rows,cols,C,R,W", [
    (1000, 3000, 256, 64, 32),     # ragged last row block, 12 column blocks
    (5000, 5000, 512, 512, 32),    # cfg1 geometry, small
    (777, 2049, 100, 96, 8),       # W = 8: four groups per warp
    (300, 9000, 1000, 32, 32),     # one group per row block
    (4096, 4096, 4096, 1024, 16),  # one column block
    (2000, 70000, 1024, 2048, 32), # R > threads: warps loop over groups
])
def test_rowblock_equals_plan_bitwise(dtype, rows, cols, C, R, W):
    rng = np.random.default_rng(rows + cols)
    lens = rng.poisson(7, rows)
    lens[rng.choice(rows, rows // 10, replace=False)] = 0   # empty rows
    lens[rows // 3: rows // 3 + 5] = min(cols, 600)          # long rows
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size).astype(dtype)
    hbp = _hbp(rows, cols, r, c, v, C, R, W)
    x = torch.as_tensor(rng.uniform(-1, 1, cols).astype(dtype), device="cuda")
    y_row = H.SpmvOperator(hbp, schedule="rowblock")(x).cpu().numpy()
    y_plan = H.SpmvOperator(hbp, schedule="plan")(x).cpu().numpy()
    np.testing.assert_array_equal(y_row.view(np.uint8), y_plan.view(np.uint8))


def test_rowblock_empty_row_blocks():
    """Row blocks without any nonzero block get +0.0 (combine's value)."""
    rows, cols, R = 4096, 4096, 256
    r = np.concatenate([np.arange(0, 256), np.arange(2048, 2100)])
    c = (r * 7) % cols
    v = np.full(r.size, -1.5)
    hbp = _hbp(rows, cols, r, c, v, C=512, R=R)
    x = torch.full((cols,), 2.0, dtype=torch.float64, device="cuda")
    y = torch.full((rows,), np.nan, dtype=torch.float64, device="cuda")
    H.SpmvOperator(hbp, schedule="rowblock")(x, y)
    y = y.cpu().numpy()
    want = np.zeros(rows)
    want[r] = -3.0
    np.testing.assert_array_equal(y, want)
    assert not np.signbit(y[300])


def test_rowblock_empty_matrix():
    hbp = _hbp(700, 900, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), C=128, R=64)
    y = H.SpmvOperator(hbp, schedule="rowblock")(torch.ones(900, dtype=torch.float64,
                                                           device="cuda"))
    assert (y == 0).all()


def test_auto_schedule():
    """Small, evenly spread, several column blocks -> rowblock; one skewed
    row block, one column block, or a hot-staging request -> stream."""
    n = 64 * 64
    i = np.arange(n)
    r = np.concatenate([i, i[1:], i[:-1], i[64:], i[:-64]])
    c = np.concatenate([i, i[:-1], i[1:], i[:-64], i[64:]])
    v = np.ones(r.size)
    hbp = _hbp(n, n, r, c, v, C=512)
    op = H.SpmvOperator(hbp)
    assert op.schedule == "rowstage" and op.launches_per_call == 1  # f64, fits a CTA
    h32 = _hbp(n, n, r, c, v.astype(np.float32), C=512)
    assert H.SpmvOperator(h32).schedule == "rowblock"
    assert H.SpmvOperator(hbp, hot=False).schedule == "stream"
    assert H.SpmvOperator(_hbp(n, n, r, c, v, C=n)).schedule == "stream"
    # one dense row block among sparse ones
    rr = np.concatenate([r, np.repeat(np.arange(100), 2000)])
    cc = np.concatenate([c, np.tile(np.arange(2000) * 2 + 1, 100)])
    key = np.unique(rr * n + cc)
    skew = _hbp(n, n, key // n, key % n, np.ones(key.size), C=512, R=64)
    assert H.SpmvOperator(skew).schedule == "stream"
    assert H.SpmvOperator(_hbp(n, n, r, c, v, C=512, R=64)).schedule == "rowstage"
    # uniform columns over many column blocks: many small blocks per row block
    rng = np.random.default_rng(4)
    ru = np.repeat(np.arange(n), 16)
    key = np.unique(ru * n + rng.integers(0, n, ru.size))
    many = _hbp(n, n, key // n, key % n, np.ones(key.size), C=256)
    assert many.nzb > 4 * many.num_row_blocks
    assert H.SpmvOperator(many).schedule == "stream"
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n), device="cuda")
    np.testing.assert_array_equal(op(x).cpu().numpy(),
                                  H.SpmvOperator(hbp, schedule="plan")(x).cpu().numpy())


# ---- TMA-staged row-block owner (hbp_spmv_rowstage, W = 32)

@pytest.mark.parametrize("name", [n for n in golden_names() if load_golden(n)["W"] == 32])
def test_rowstage_matches_golden(name):
    g = load_golden(name)
    val = g["trip_val"].astype(np.float32) if g["fp32"] else g["trip_val"]
    hbp = _hbp(g["rows"], g["cols"], g["trip_row"], g["trip_col"], val, g["C"], g["R"], g["W"],
               g["seed"])
    x = g["x"].astype(np.float32) if g["fp32"] else g["x"]
    op = H.SpmvOperator(hbp, schedule="rowstage")
    assert op.launches_per_call == 1
    y = op(torch.as_tensor(x, device="cuda")).cpu().numpy()
    if g["fp32"]:
        err = O.componentwise_error(g["rows"], g["trip_row"], g["trip_col"], g["trip_val"],
                                    g["x"], y.astype(np.float64))
        assert err <= 1e-5
    else:
        np.testing.assert_array_equal(y, g["y"])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("rows,cols,C,R", [
    (1000, 3000, 256, 64),      # ragged last row block, 12 column blocks
    (5000, 5000, 512, 512),     # cfg1 geometry, small
    (300, 9000, 1000, 32),      # one group per row block
    (4096, 4096, 4096, 1024),   # one column block
    (3000, 70000, 2400, 256),   # up to 30 blocks per row block
    (2000, 2000, 70, 96),       # C not a multiple of 4: unaligned staged ranges
])
def test_rowstage_equals_plan_bitwise(dtype, rows, cols, C, R):
    rng = np.random.default_rng(rows + cols + 1)
    lens = rng.poisson(7, rows)
    lens[rng.choice(rows, rows // 10, replace=False)] = 0
    lens[rows // 3: rows // 3 + 5] = min(cols, 600)
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size).astype(dtype)
    hbp = _hbp(rows, cols, r, c, v, C, R, 32)
    x = torch.as_tensor(rng.uniform(-1, 1, cols).astype(dtype), device="cuda")
    op = H.SpmvOperator(hbp, schedule="rowstage")
    y_st = op(x).cpu().numpy()
    np.testing.assert_array_equal(op(x).cpu().numpy(), y_st)
    y_plan = H.SpmvOperator(hbp, schedule="plan")(x).cpu().numpy()
    np.testing.assert_array_equal(y_st.view(np.uint8), y_plan.view(np.uint8))


def test_rowstage_empty_row_blocks_and_matrix():
    rows, cols, R = 4096, 4096, 256
    r = np.concatenate([np.arange(0, 256), np.arange(2048, 2100)])
    c = (r * 7) % cols
    hbp = _hbp(rows, cols, r, c, np.full(r.size, -1.5), C=512, R=R)
    x = torch.full((cols,), 2.0, dtype=torch.float64, device="cuda")
    y = torch.full((rows,), np.nan, dtype=torch.float64, device="cuda")
    H.SpmvOperator(hbp, schedule="rowstage")(x, y)
    want = np.zeros(rows)
    want[r] = -3.0
    np.testing.assert_array_equal(y.cpu().numpy(), want)
    empty = _hbp(700, 900, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), C=128, R=64)
    y = H.SpmvOperator(empty, schedule="rowstage")(torch.ones(900, dtype=torch.float64,
                                                              device="cuda"))
    assert (y == 0).all()


def test_rowstage_rejects_oversized_row_blocks(monkeypatch):
    rng = np.random.default_rng(0)
    rows, cols = 512, 4096
    lens = np.full(rows, 300)
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    hbp = _hbp(rows, cols, r, c, rng.uniform(-1, 1, r.size), C=4096, R=512)
    with pytest.raises(ValueError, match="shared memory"):
        H.SpmvOperator(hbp, schedule="rowstage")


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("rows,cols,C,R", [(5000, 5000, 512, 512), (2000, 2000, 70, 96),
                                          (3001, 9000, 1000, 64)])
def test_rowstage_x_windows_bitwise(dtype, rows, cols, C, R, monkeypatch):
    """hbp_spmv_rowstage with each block's x window staged by TMA (opt-in,
    HBP_ROWSTAGE_X=1; unaligned window ends copied by hand) == plan bitwise."""
    monkeypatch.setenv("HBP_ROWSTAGE_X", "1")
    monkeypatch.setattr(H.SpmvOperator, "ROWSTAGE_X_SMEM", 200 * 1024)
    rng = np.random.default_rng(rows + 7)
    lens = rng.poisson(6, rows)
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size).astype(dtype)
    hbp = _hbp(rows, cols, r, c, v, C, R, 32)
    x = torch.as_tensor(rng.uniform(-1, 1, cols).astype(dtype), device="cuda")
    op = H.SpmvOperator(hbp, schedule="rowstage")
    assert op.rowstage_caps[2] > 0
    y = op(x).cpu().numpy()
    y_plan = H.SpmvOperator(hbp, schedule="plan")(x).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint8), y_plan.view(np.uint8))
    # an x view at an odd offset falls back to global gathers (same bits)
    xb = torch.empty(cols + 1, dtype=x.dtype, device="cuda")
    xb[1:] = x
    np.testing.assert_array_equal(op(xb[1:]).cpu().numpy(), y)
