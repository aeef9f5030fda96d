"""The column-segment schedule (hbp_spmv_seg: x-segment staged in shared
memory per block, CTA per block, fixed chunks + atomic ticket) against the
reference golden vectors, the oracle and the other schedules.

Exact mode sums each row in step order (_kernels.py:41-46), so f64 results
are bitwise the reference's for any CTA count and fixed fraction.
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
    import bench_inputs as BI

W32 = [n for n in golden_names() if load_golden(n)["W"] == 32
       and load_golden(n)["R"] % 32 == 0] if has_gpu() else []


def _hbp(rows, cols, r, c, v, C, R=512, W=32, seed=0, ff=0.7):
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W, fixed_fraction=ff)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    params = H.sample_hash_params(grid, cfg, seed=seed)
    return H.build_hbp(csr, grid, H.hash_permutations(grid, params))


@pytest.mark.parametrize("name", W32)
@pytest.mark.parametrize("workers", [1, 3, None])
def test_seg_matches_golden(name, workers):
    g = load_golden(name)
    val = g["trip_val"].astype(np.float32) if g["fp32"] else g["trip_val"]
    hbp = _hbp(g["rows"], g["cols"], g["trip_row"], g["trip_col"], val, g["C"], g["R"], g["W"],
               g["seed"])
    x = g["x"].astype(np.float32) if g["fp32"] else g["x"]
    op = H.SpmvOperator(hbp, schedule="seg", workers=workers)
    xd = torch.as_tensor(x, device="cuda")
    y = op(xd).cpu().numpy()
    y2 = op(xd).cpu().numpy()  # the ticket pair resets itself
    np.testing.assert_array_equal(y, y2)
    if g["fp32"]:
        err = O.componentwise_error(g["rows"], g["trip_row"], g["trip_col"], g["trip_val"],
                                    g["x"], y.astype(np.float64))
        assert err <= 1e-5
    else:
        np.testing.assert_array_equal(y, g["y"])


@pytest.mark.parametrize("ff", [0.0, 0.3, 0.7, 1.0])
@pytest.mark.parametrize("workers", [1, 7, None])
def test_seg_banded_bitwise(ff, workers):
    """cfg3's structure (33 diagonals at even offsets, fp64, C=4096) at
    2^16 rows: bitwise the oracle for every split of fixed / competitive."""
    rows, cols, rp, ci, v = BI.banded_csr(1 << 16)
    r = np.repeat(np.arange(rows), np.diff(rp))
    hbp = _hbp(rows, cols, r, ci, v, 4096, ff=ff)
    x = np.random.default_rng(1).uniform(-1, 1, cols)
    y = H.SpmvOperator(hbp, schedule="seg", workers=workers)(
        torch.as_tensor(x, device="cuda")).cpu().numpy()
    p = O.pipeline(rows, cols, r, ci, v, 4096, 512, 32)
    np.testing.assert_array_equal(y, O.hbp_spmv(p["hbp"], x, workers=3))


def test_seg_laplacian_matches_rowblock():
    """cfg1's structure (5-point Laplacian, C=4096) at 256^2."""
    rows, cols, rp, ci, v = BI.laplacian_csr(256)
    r = np.repeat(np.arange(rows), np.diff(rp))
    hbp = _hbp(rows, cols, r, ci, v, 4096)
    xd = torch.as_tensor(np.random.default_rng(2).uniform(-1, 1, cols), device="cuda")
    a = H.SpmvOperator(hbp, schedule="seg")(xd).cpu().numpy()
    b = H.SpmvOperator(hbp, schedule="rowblock")(xd).cpu().numpy()
    c = H.SpmvOperator(hbp, schedule="stream")(xd).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, c)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("rows,cols,C,R", [
    (1000, 3000, 256, 64),      # ragged last row block, 12 column blocks
    (5000, 5000, 512, 512),
    (300, 9000, 1000, 32),      # one group per row block
    (3000, 3001, 3001, 96),     # one column block (direct y), odd window widths
    (2000, 70000, 1024, 2048),  # more groups than warps
])
def test_seg_equals_plan(dtype, rows, cols, C, R):
    rng = np.random.default_rng(rows + cols)
    lens = rng.poisson(7, rows)
    lens[rng.choice(rows, 5, replace=False)] = min(cols // 2, 900)  # long rows
    lens[rows // 3: rows // 3 + R] = 0  # an empty row block
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size).astype(dtype)
    hbp = _hbp(rows, cols, r, c, v, C, R)
    xd = torch.as_tensor(rng.uniform(-1, 1, cols).astype(dtype), device="cuda")
    a = H.SpmvOperator(hbp, schedule="seg")(xd).cpu().numpy()
    if dtype == np.float64:
        b = H.SpmvOperator(hbp, schedule="plan")(xd).cpu().numpy()
        np.testing.assert_array_equal(a, b)
    err = O.componentwise_error(rows, r, c, v.astype(np.float64),
                                xd.cpu().numpy().astype(np.float64), a.astype(np.float64))
    assert err <= (1e-12 if dtype == np.float64 else 1e-5)


def test_seg_unaligned_x_view():
    """x given as a view at an odd element offset: the window's bulk copy
    covers only the 16-byte-aligned interior, the head/tail are plain loads."""
    rows, cols, rp, ci, v = BI.banded_csr(1 << 13)
    r = np.repeat(np.arange(rows), np.diff(rp))
    hbp = _hbp(rows, cols, r, ci, v, 1000)
    base = torch.as_tensor(np.random.default_rng(3).uniform(-1, 1, cols + 1), device="cuda")
    xv = base[1:]
    assert xv.data_ptr() % 16 != 0
    a = H.SpmvOperator(hbp, schedule="seg")(xv).cpu().numpy()
    p = O.pipeline(rows, cols, r, ci, v, 1000, 512, 32)
    np.testing.assert_array_equal(a, O.hbp_spmv(p["hbp"], xv.cpu().numpy(), workers=2))
