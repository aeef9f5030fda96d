"""Hot-column staging of x in shared memory (hbp_hot.cu, hbp_spmv_stream HOT).

Staging changes where the x value of a hot column is read from (the SM's
shared copy instead of global memory), never which value or in which order
it is summed, so a staged SpMV must be BITWISE equal to the unstaged one
(f32 fast mode and f64 exact mode) -- and hence to the oracle wherever the
unstaged path is.  The metadata (degrees, hot order, staged stream) is
checked against numpy.
"""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch
    import paper_2504_08860_b200 as H
    from paper_2504_08860_b200 import _lib as L
    from oracle import oracle as O

FLAG = 0x80000000


def _powerlaw(seed=0, rows=20000, cols=30000, per_row=12):
    """Zipf-like column popularity (a few columns carry most nonzeros) and
    skewed row lengths."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.zipf(1.7, rows) + per_row // 2, cols // 4)
    r = np.repeat(np.arange(rows), lens)
    w = 1.0 / np.arange(1, cols + 1) ** 1.1
    relabel = rng.permutation(cols)
    c = relabel[rng.choice(cols, r.size, p=w / w.sum())]
    key = np.unique(r.astype(np.int64) * cols + c)
    r, c = key // cols, key % cols
    v = rng.uniform(-1, 1, r.size)
    return rows, cols, r, c, v


def _hbp(rows, cols, r, c, v, C=None, R=512):
    cfg = H.PartitionConfig(col_width=C or cols, row_height=R, warp_size=32)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    return H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))


@pytest.fixture(scope="module")
def mat():
    return _powerlaw()


def test_hot_metadata(mat):
    rows, cols, r, c, v = mat
    hbp = _hbp(rows, cols, r, c, v)
    hc = hbp.hot_columns(1000)
    assert hc.n_hot == 1000
    deg = np.bincount(c, minlength=cols)
    order = np.argsort(-deg, kind="stable")  # descending degree, ties by column
    np.testing.assert_array_equal(hc.hot_cols.cpu().numpy(), order[:1000])
    assert hc.share == pytest.approx(deg[order[:1000]].sum() / c.size, rel=1e-12)
    col = hbp.col.cpu().numpy().view(np.uint32).astype(np.int64)
    slot = np.full(cols, -1, np.int64)
    slot[order[:1000]] = np.arange(1000)
    want = np.where(slot[col] >= 0, FLAG | slot[col], col).astype(np.uint32)
    np.testing.assert_array_equal(hc.scol.cpu().numpy().view(np.uint32), want)


def test_warm_metadata(mat):
    rows, cols, r, c, v = mat
    hbp = _hbp(rows, cols, r, c, v)
    hc = hbp.hot_columns(64, 3000)
    assert (hc.n_hot, hc.n_warm) == (64, 3000)
    deg = np.bincount(c, minlength=cols)
    order = np.argsort(-deg, kind="stable")
    np.testing.assert_array_equal(hc.hot_cols.cpu().numpy(), order[:3064])
    assert hc.warm_share == pytest.approx(deg[order[64:3064]].sum() / c.size, rel=1e-12)
    col = hbp.col.cpu().numpy().view(np.uint32).astype(np.int64)
    slot = np.full(cols, -1, np.int64)
    slot[order[:3064]] = np.arange(3064)
    s = slot[col]
    want = np.where(s < 0, col, np.where(s < 64, FLAG | s, 0x40000000 | (s - 64)))
    np.testing.assert_array_equal(hc.scol.cpu().numpy().view(np.uint32), want.astype(np.uint32))


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n_hot,warm", [(4, 0), (64, 0), (1000, 0), (None, 0), (4, 20000),
                                        (64, 2000), (None, 1 << 30)])
@pytest.mark.parametrize("workers", [1, 37, 500, None])
def test_staged_bitwise_equals_unstaged(mat, dtype, n_hot, warm, workers):
    rows, cols, r, c, v = mat
    vv = v.astype(np.float32) if dtype == "f32" else v
    hbp = _hbp(rows, cols, r, c, vv)
    x = np.random.default_rng(5).uniform(-1, 1, cols)
    xd = torch.as_tensor(x.astype(vv.dtype), device="cuda")
    plain = H.SpmvOperator(hbp, workers=workers, hot=False)
    staged = H.SpmvOperator(hbp, workers=workers, hot=True if n_hot is None else n_hot,
                            warm_bytes=warm * vv.itemsize)
    assert plain.hot is None and staged.hot is not None
    y0 = plain(xd).cpu().numpy()
    y1 = staged(xd).cpu().numpy()
    y2 = staged(xd).cpu().numpy()
    np.testing.assert_array_equal(y1, y0)
    np.testing.assert_array_equal(y2, y1)
    if dtype == "f64":  # exact mode: the reference's bits
        p = O.pipeline(rows, cols, r, c, v, cols, 512, 32)
        np.testing.assert_array_equal(y1, O.hbp_spmv(p["hbp"], x, workers=2))
    else:
        err = O.componentwise_error(rows, r, c, vv.astype(np.float64),
                                    x.astype(np.float32).astype(np.float64),
                                    y1.astype(np.float64))
        assert err <= 1e-5


def test_auto_staging_policy(mat):
    rows, cols, r, c, v = mat
    hbp = _hbp(rows, cols, r, c, v.astype(np.float32))
    op = H.SpmvOperator(hbp)
    assert op.hot is not None and op.hot.share >= H.SpmvOperator.HOT_MIN_SHARE
    assert op.launches_per_call == 2  # hot gather + stream kernel
    # uniform columns over many more columns than the capacity: not staged
    rng = np.random.default_rng(2)
    n = 2_000_000
    rr = np.repeat(np.arange(n), 2)
    cc = rng.integers(0, n, rr.size)
    key = np.unique(rr * n + cc)
    hb2 = _hbp(n, n, key // n, key % n, rng.uniform(-1, 1, key.size).astype(np.float32))
    assert H.SpmvOperator(hb2).hot is None


def test_staged_multi_col_block(mat):
    """Staging with a partial + combine (C < cols) stays bitwise."""
    rows, cols, r, c, v = mat
    hbp = _hbp(rows, cols, r, c, v, C=4096)
    x = torch.as_tensor(np.random.default_rng(9).uniform(-1, 1, cols), device="cuda")
    y0 = H.SpmvOperator(hbp, hot=False)(x).cpu().numpy()
    y1 = H.SpmvOperator(hbp, hot=True)(x).cpu().numpy()
    np.testing.assert_array_equal(y1, y0)


def test_hot_gather_and_capacity():
    cap = L.c_i64(0)
    caps = {}
    for mode in (0, 1, 2):  # hot only, warm tier, packed x
        L.call("hbp_hot_capacity", L.c_int(L.HBP_F32), L.c_int(mode), ctypes.byref(cap))
        cap32 = caps[mode] = int(cap.value)
        L.call("hbp_hot_capacity", L.c_int(L.HBP_F64), L.c_int(mode), ctypes.byref(cap))
        assert cap32 >= 4096 and int(cap.value) >= 1024 and cap32 % 1024 == 0
    assert caps[1] < caps[0] < caps[2]
    with pytest.raises(ValueError):
        L.call("hbp_hot_capacity", L.c_int(L.HBP_F32), L.c_int(3), ctypes.byref(cap))
    x = torch.randn(100000, device="cuda", dtype=torch.float64)
    hot = torch.randint(0, 100000, (4096,), device="cuda", dtype=torch.int32)
    out = torch.empty(4096, device="cuda", dtype=torch.float64)
    L.call("hbp_hot_gather", L.P(x), L.c_int(L.HBP_F64), L.P(hot), L.c_i64(4096), L.P(out),
           L.stream())
    assert torch.equal(out, x[hot.long()])


def test_n_hot_beyond_capacity_rejected(mat):
    rows, cols, r, c, v = mat
    hbp = _hbp(rows, cols, r, c, v.astype(np.float32))
    op = H.SpmvOperator(hbp, hot=True)
    f = L.FormatT.from_buffer_copy(op._fmt)
    f.n_hot = 1 << 20
    x = torch.zeros(cols, device="cuda", dtype=torch.float32)
    y = torch.empty(rows, device="cuda", dtype=torch.float32)
    with pytest.raises(ValueError):
        L.call("hbp_spmv_stream", ctypes.byref(f), ctypes.byref(op.bal), L.P(x), L.P(y),
               L.P(None), L.stream())


@pytest.mark.parametrize("stride", [1, 3, 16])
def test_col_degree_sampled(mat, stride):
    rows, cols, r, c, v = mat
    hbp = _hbp(rows, cols, r, c, v.astype(np.float32))
    deg = torch.zeros(cols, dtype=torch.int32, device="cuda")
    L.call("hbp_col_degree", L.P(hbp.col), L.c_i64(hbp.nnz), L.c_i64(stride), L.P(deg),
           L.stream())
    col = hbp.col.cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(deg.cpu().numpy(), np.bincount(col[::stride], minlength=cols))


@pytest.mark.parametrize("rows,cols,per_row", [(1, 1, 1), (5, 3, 2), (31, 7, 3), (33, 4, 4),
                                               (1000, 5, 3), (700, 64, 40)])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_staging_tiny_shapes(rows, cols, per_row, dtype):
    """Few columns (all of them hot, or fewer than 4 -> no staging), short row
    blocks, dense rows: staged == unstaged bitwise, and the oracle."""
    rng = np.random.default_rng(rows * 31 + cols)
    lens = np.minimum(rng.integers(0, per_row + 1, rows), cols)
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens]) if r.size else \
        np.zeros(0, np.int64)
    v = rng.uniform(-1, 1, r.size)
    vv = v.astype(np.float32) if dtype == "f32" else v
    for R in (32, 96, 512, 1024):
        hbp = _hbp(rows, cols, r, c, vv, R=R)
        x = rng.uniform(-1, 1, cols)
        xd = torch.as_tensor(x.astype(vv.dtype), device="cuda")
        y0 = H.SpmvOperator(hbp, hot=False)(xd).cpu().numpy()
        st = H.SpmvOperator(hbp, hot=True)
        assert (st.hot is None) == (cols < 4)
        y1 = st(xd).cpu().numpy()
        np.testing.assert_array_equal(y1, y0)
        if dtype == "f64":
            p = O.pipeline(rows, cols, r, c, v, cols, R, 32)
            np.testing.assert_array_equal(y1, O.hbp_spmv(p["hbp"], x, workers=2))


def test_staging_empty_matrix():
    hbp = _hbp(100, 50, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    op = H.SpmvOperator(hbp, hot=True)
    y = op(torch.ones(50, dtype=torch.float64, device="cuda"))
    assert torch.equal(y, torch.zeros(100, dtype=torch.float64, device="cuda"))


# ---- packed x (HBP_FLAG_PACKED_X): every used column after the hot ones in a
# degree-ordered compact copy of x

@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n_hot", [4, 1000, None])
@pytest.mark.parametrize("workers", [1, 37, None])
def test_packed_bitwise_equals_unstaged(mat, dtype, n_hot, workers):
    rows, cols, r, c, v = mat
    vv = v.astype(np.float32) if dtype == "f32" else v
    hbp = _hbp(rows, cols, r, c, vv)
    x = np.random.default_rng(6).uniform(-1, 1, cols)
    xd = torch.as_tensor(x.astype(vv.dtype), device="cuda")
    plain = H.SpmvOperator(hbp, workers=workers, hot=False)
    packed = H.SpmvOperator(hbp, workers=workers, hot=True if n_hot is None else n_hot,
                            packed_x=True)
    assert packed.hot is not None and packed.hot.packed
    y0 = plain(xd).cpu().numpy()
    y1 = packed(xd).cpu().numpy()
    np.testing.assert_array_equal(y1, y0)
    np.testing.assert_array_equal(packed(xd).cpu().numpy(), y1)


@pytest.mark.parametrize("sample", [None, 1000])
def test_packed_metadata(mat, monkeypatch, sample):
    """hot_cols = the n_hot heaviest columns (the ranking's order), then every
    other used column ascending -- exactly the used ones, from exact
    presence even when the ranking is sampled; scol decodes back to col."""
    rows, cols, r, c, v = mat
    if sample is not None:  # force the sampled ranking + exact presence pass
        monkeypatch.setattr(H.HbpMatrix, "RANK_SAMPLE", sample)
    hbp = _hbp(rows, cols, r, c, v.astype(np.float32))
    hc = hbp.hot_columns(64, packed=True)
    used = np.unique(c)
    n_used = hc.n_hot + hc.n_warm
    hot_cols = hc.hot_cols.cpu().numpy().astype(np.int64)
    assert hc.n_hot == 64 and n_used == used.size == hot_cols.size
    np.testing.assert_array_equal(np.sort(hot_cols), used)
    _, order = hbp.column_ranking()
    np.testing.assert_array_equal(hot_cols[:64], order[:64].cpu().numpy())
    assert np.all(np.diff(hot_cols[64:]) > 0)
    col = hbp.col.cpu().numpy().astype(np.int64)
    sc = hc.scol[:hbp.nnz].cpu().numpy().astype(np.uint32).astype(np.int64)
    hot = (sc & FLAG) != 0
    dec = np.where(hot, hot_cols[sc & (FLAG - 1)], hot_cols[np.minimum(hc.n_hot + sc, n_used - 1)])
    np.testing.assert_array_equal(dec, col)


def test_packed_is_the_default_when_x_fits_l2(mat):
    rows, cols, r, c, v = mat
    hbp = _hbp(rows, cols, r, c, v.astype(np.float32))
    op = H.SpmvOperator(hbp)
    assert op.hot is not None and op.hot.packed
    assert not H.SpmvOperator(hbp, packed_x=False).hot.packed
