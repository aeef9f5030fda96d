"""The element-balanced B200 schedule (hbp_spmv_balanced) vs the oracle.

f64: cuts on group boundaries -> bitwise equal to the reference for any
worker count.  f32: step-aligned cuts + last-arriver combine -> within 1e-5
componentwise of the reference (fp64 on the fp32-rounded inputs), and
deterministic run to run.
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

W32 = [n for n in golden_names() if load_golden(n)["W"] == 32]


def _hbp(rows, cols, r, c, v, C, R=512, W=32, seed=0):
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    params = H.sample_hash_params(grid, cfg, seed=seed)
    return H.build_hbp(csr, grid, H.hash_permutations(grid, params))


@pytest.mark.parametrize("name", W32)
@pytest.mark.parametrize("workers", [1, 3, 17, 200, None])
@pytest.mark.parametrize("schedule", ["balanced", "stream"])
def test_balanced_matches_golden(name, workers, schedule):
    g = load_golden(name)
    val = g["trip_val"].astype(np.float32) if g["fp32"] else g["trip_val"]
    hbp = _hbp(g["rows"], g["cols"], g["trip_row"], g["trip_col"], val, g["C"], g["R"], g["W"],
               g["seed"])
    x = g["x"].astype(np.float32) if g["fp32"] else g["x"]
    op = H.SpmvOperator(hbp, workers=workers, schedule=schedule)
    y = op(torch.as_tensor(x, device="cuda")).cpu().numpy()
    if g["fp32"]:
        err = O.componentwise_error(g["rows"], g["trip_row"], g["trip_col"], g["trip_val"],
                                    g["x"], y.astype(np.float64))
        assert err <= 1e-5
    else:
        np.testing.assert_array_equal(y, g["y"])


def _hot_matrix(seed=3, rows=4096, cols=50000):
    """Rows of wildly different lengths: a few 20k-40k-element rows among
    short ones, so groups split across many warps."""
    rng = np.random.default_rng(seed)
    lens = rng.poisson(6, rows)
    hot = rng.choice(rows, 12, replace=False)
    lens[hot] = rng.integers(min(20000, cols // 2), min(40000, cols), hot.size)
    lens[rows // 2: rows // 2 + 40] = 900  # one long, fully live group
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size)
    return rows, cols, r, c, v


@pytest.mark.parametrize("workers", [2, 9, 64, 333, 1500, None])
@pytest.mark.parametrize("schedule", ["balanced", "stream"])
def test_balanced_f32_hot_rows(workers, schedule):
    rows, cols, r, c, v = _hot_matrix()
    v32 = v.astype(np.float32)
    x = np.random.default_rng(1).uniform(-1, 1, cols).astype(np.float32)
    hbp = _hbp(rows, cols, r, c, v32, C=cols)
    op = H.SpmvOperator(hbp, workers=workers, schedule=schedule)
    xd = torch.as_tensor(x, device="cuda")
    y1 = op(xd).cpu().numpy()
    y2 = op(xd).cpu().numpy()
    np.testing.assert_array_equal(y1, y2)  # deterministic (counters self-reset)
    err = O.componentwise_error(rows, r, c, v32.astype(np.float64), x.astype(np.float64),
                                y1.astype(np.float64))
    assert err <= 1e-5


@pytest.mark.parametrize("workers", [2, 9, 333, None])
@pytest.mark.parametrize("schedule", ["balanced", "stream"])
def test_balanced_f64_hot_rows_bitwise(workers, schedule):
    rows, cols, r, c, v = _hot_matrix(seed=4)
    x = np.random.default_rng(2).uniform(-1, 1, cols)
    hbp = _hbp(rows, cols, r, c, v, C=cols)
    y = H.SpmvOperator(hbp, workers=workers, schedule=schedule)(
        torch.as_tensor(x, device="cuda")).cpu().numpy()
    p = O.pipeline(rows, cols, r, c, v, cols, 512, 32)
    np.testing.assert_array_equal(y, O.hbp_spmv(p["hbp"], x, workers=4))


def test_balanced_multi_column_blocks_f32():
    rows, cols, r, c, v = _hot_matrix(seed=5, rows=3000, cols=60000)
    v32 = v.astype(np.float32)
    x = np.random.default_rng(3).uniform(-1, 1, cols).astype(np.float32)
    hbp = _hbp(rows, cols, r, c, v32, C=4096)
    assert hbp.num_col_blocks > 1
    for workers, schedule in ((5, "balanced"), (100, "balanced"), (None, "balanced"),
                              (5, "stream"), (100, "stream"), (None, "stream")):
        y = H.SpmvOperator(hbp, workers=workers, schedule=schedule)(
            torch.as_tensor(x, device="cuda"))
        err = O.componentwise_error(rows, r, c, v32.astype(np.float64), x.astype(np.float64),
                                    y.cpu().numpy().astype(np.float64))
        assert err <= 1e-5


def test_plan_schedule_still_available():
    rows, cols, r, c, v = _hot_matrix(seed=6, rows=1024, cols=5000)
    x = np.random.default_rng(4).uniform(-1, 1, cols)
    hbp = _hbp(rows, cols, r, c, v, C=cols)
    xd = torch.as_tensor(x, device="cuda")
    a = H.SpmvOperator(hbp, schedule="plan")(xd).cpu().numpy()
    b = H.SpmvOperator(hbp, schedule="balanced")(xd).cpu().numpy()
    c = H.SpmvOperator(hbp, schedule="stream")(xd).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, c)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("workers", [1, 7, 333, None])
def test_stream_precomputed_slices(dtype, workers):
    """hbp_stream_slices (one-time slice bounds) == the in-kernel search."""
    rows, cols, r, c, v = _hot_matrix(seed=5)
    hbp = _hbp(rows, cols, r, c, v.astype(dtype), C=cols)
    x = torch.as_tensor(np.random.default_rng(2).uniform(-1, 1, cols).astype(dtype),
                        device="cuda")
    op = H.SpmvOperator(hbp, workers=workers, hot=False, schedule="stream", slice_cost="0")
    assert op.bal.slice_lo and op.bal.slice_g
    y1 = op(x).cpu().numpy()
    lo = op.slice_lo_t.cpu().numpy()
    assert lo[0] == 0 and lo[-1] == hbp.nnz and np.all(np.diff(lo) >= 0)
    op.bal.slice_lo = op.bal.slice_g = 0
    y2 = op(x).cpu().numpy()
    np.testing.assert_array_equal(y1, y2)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("C,workers", [(4096, None), (4096, 3), (1000, 77), (777, None)])
def test_stream_fused_combine(dtype, C, workers, monkeypatch):
    """Several column blocks: the kernel's last-arriver combine == hbp_combine
    (bitwise), including row blocks without nonzero blocks."""
    rows, cols, r, c, v = _hot_matrix(seed=7)
    keep = (r < 1500) | (r >= 2100)  # a gap of empty row blocks (R = 512 -> block 3)
    r, c, v = r[keep], c[keep], v[keep]
    hbp = _hbp(rows, cols, r, c, v.astype(dtype), C=C)
    x = torch.as_tensor(np.random.default_rng(3).uniform(-1, 1, cols).astype(dtype),
                        device="cuda")
    monkeypatch.setenv("HBP_FUSED_COMBINE", "1")
    fused = H.SpmvOperator(hbp, workers=workers, hot=False, schedule="stream")
    assert fused.fused_combine
    monkeypatch.setenv("HBP_FUSED_COMBINE", "0")
    plain = H.SpmvOperator(hbp, workers=workers, hot=False, schedule="stream")
    assert not plain.fused_combine
    y0 = plain(x).cpu().numpy()
    y1 = fused(x).cpu().numpy()
    y2 = fused(x).cpu().numpy()  # counters self-reset
    np.testing.assert_array_equal(y1, y0)
    np.testing.assert_array_equal(y2, y0)
    if dtype == np.float64:
        p = O.pipeline(rows, cols, r, c, v, C, 512, 32)
        np.testing.assert_array_equal(y1, O.hbp_spmv(p["hbp"], x.cpu().numpy(), workers=2))


@pytest.mark.parametrize("R", [32, 96, 160])
def test_stream_fused_combine_short_row_blocks(R, monkeypatch):
    """Fused combine with row_height not a multiple of 128: the
    last-arriver combine reads only its own row block's partial rows."""
    rows, cols, r, c, v = _hot_matrix(seed=8, rows=1000, cols=6000)
    hbp = _hbp(rows, cols, r, c, v, C=1500, R=R)
    x = torch.as_tensor(np.random.default_rng(5).uniform(-1, 1, cols), device="cuda")
    monkeypatch.setenv("HBP_FUSED_COMBINE", "1")
    fused = H.SpmvOperator(hbp, hot=False, schedule="stream")
    assert fused.fused_combine
    y1 = fused(x).cpu().numpy()
    p = O.pipeline(rows, cols, r, c, v, 1500, R, 32)
    np.testing.assert_array_equal(y1, O.hbp_spmv(p["hbp"], x.cpu().numpy(), workers=2))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("C", [700, 4096])
def test_stream_direct_single_row_blocks(dtype, C, monkeypatch):
    """Row blocks with one nonzero block are written to y by the SpMV kernel
    (HBP_FLAG_DIRECT_SINGLE) and skipped by the combine: bitwise the same as
    routing everything through the partial."""
    rows, cols, r, c, v = _hot_matrix(seed=9)
    keep = (c < 600) | (r % 5 == 0)  # mostly one column block per row block, some more
    r, c, v = r[keep], c[keep], v[keep]
    hbp = _hbp(rows, cols, r, c, v.astype(dtype), C=C)
    x = torch.as_tensor(np.random.default_rng(4).uniform(-1, 1, cols).astype(dtype),
                        device="cuda")
    direct = H.SpmvOperator(hbp, hot=False, schedule="stream")
    assert direct._fmt.reserved & 4
    monkeypatch.setenv("HBP_DIRECT_SINGLE", "0")
    routed = H.SpmvOperator(hbp, hot=False, schedule="stream")
    assert not routed._fmt.reserved & 4
    np.testing.assert_array_equal(direct(x).cpu().numpy(), routed(x).cpu().numpy())


TICKETS = ["0.7:2", "0.0:3", "1.0:1", "0.5:7"]


@pytest.mark.parametrize("name", [n for n in W32 if not n.startswith("kat")][:12])
@pytest.mark.parametrize("ticket", TICKETS)
@pytest.mark.parametrize("workers", [1, 5, None])
def test_stream_ticket_matches_golden(name, ticket, workers):
    """Competitive pieces (fixed element chunk per warp + atomic ticket): f64
    bitwise the reference, f32 within 1e-5; the ticket self-resets, so
    repeated calls give the same y."""
    g = load_golden(name)
    val = g["trip_val"].astype(np.float32) if g["fp32"] else g["trip_val"]
    hbp = _hbp(g["rows"], g["cols"], g["trip_row"], g["trip_col"], val, g["C"], g["R"], g["W"],
               g["seed"])
    x = torch.as_tensor(g["x"].astype(np.float32) if g["fp32"] else g["x"], device="cuda")
    op = H.SpmvOperator(hbp, workers=workers, schedule="stream", ticket=ticket)
    y = op(x).cpu().numpy()
    np.testing.assert_array_equal(op(x).cpu().numpy(), y)
    if g["fp32"]:
        err = O.componentwise_error(g["rows"], g["trip_row"], g["trip_col"], g["trip_val"],
                                    g["x"], y.astype(np.float64))
        assert err <= 1e-5
    else:
        np.testing.assert_array_equal(y, g["y"])


@pytest.mark.parametrize("ticket", TICKETS)
@pytest.mark.parametrize("workers", [2, 64, None])
def test_stream_ticket_f32_hot_rows(ticket, workers):
    rows, cols, r, c, v = _hot_matrix()
    v32 = v.astype(np.float32)
    x = np.random.default_rng(1).uniform(-1, 1, cols).astype(np.float32)
    hbp = _hbp(rows, cols, r, c, v32, C=cols)
    op = H.SpmvOperator(hbp, workers=workers, schedule="stream", ticket=ticket)
    xd = torch.as_tensor(x, device="cuda")
    y1 = op(xd).cpu().numpy()
    for _ in range(3):
        np.testing.assert_array_equal(op(xd).cpu().numpy(), y1)
    err = O.componentwise_error(rows, r, c, v32.astype(np.float64), x.astype(np.float64),
                                y1.astype(np.float64))
    assert err <= 1e-5
    clk = op.warp_clock()
    op(xd)
    t = clk.cpu().numpy()
    assert (t[:, 1] >= t[:, 0]).all() and (t[:, 0] > 0).all()


def test_stream_ticket_rejects_bad_fraction():
    rows, cols, r, c, v = _hot_matrix()
    hbp = _hbp(rows, cols, r, c, v.astype(np.float32), C=cols)
    with pytest.raises(ValueError, match="fixed fraction"):
        H.SpmvOperator(hbp, schedule="stream", ticket="1.5:2")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("workers", [1, 7, 333, None])
@pytest.mark.parametrize("cost", ["48,20,40", "0,0,0", "500,100,0", "1,300,900",
                                  "49,26,33,76,17", "0,0,0,0,64"])
def test_stream_cost_balanced_slices(dtype, workers, cost):
    """Cost-balanced slice cuts (hbp_group_costs + prefix): valid monotone
    bounds, f64 bitwise the reference (exact mode), f32 within 1e-5 and
    deterministic; the cut positions move with the weights."""
    rows, cols, r, c, v = _hot_matrix(seed=5)
    vv = v.astype(dtype)
    hbp = _hbp(rows, cols, r, c, vv, C=cols)
    xh = np.random.default_rng(2).uniform(-1, 1, cols).astype(dtype)
    x = torch.as_tensor(xh, device="cuda")
    op = H.SpmvOperator(hbp, workers=workers, schedule="stream", slice_cost=cost)
    lo = op.slice_lo_t.cpu().numpy()
    assert lo[0] == 0 and lo[-1] == hbp.nnz and np.all(np.diff(lo) >= 0)
    y1 = op(x).cpu().numpy()
    np.testing.assert_array_equal(op(x).cpu().numpy(), y1)
    err = O.componentwise_error(rows, r, c, vv.astype(np.float64), xh.astype(np.float64),
                                y1.astype(np.float64))
    assert err <= (1e-12 if dtype == np.float64 else 1e-5)
    if dtype == np.float64:  # exact mode: bitwise the equal-element schedule
        ref = H.SpmvOperator(hbp, workers=workers, schedule="stream", slice_cost="0")
        np.testing.assert_array_equal(ref(x).cpu().numpy(), y1)


def test_stream_cost_weights_default_and_validation():
    rows, cols, r, c, v = _hot_matrix(seed=5)
    h32 = _hbp(rows, cols, r, c, v.astype(np.float32), C=cols)
    h64 = _hbp(rows, cols, r, c, v, C=cols)
    assert H.SpmvOperator(h32, schedule="stream").slice_cost == H.SpmvOperator.SLICE_COST
    assert H.SpmvOperator(h64, schedule="stream").slice_cost is None  # exact: equal elements
    assert H.SpmvOperator(h64, schedule="stream", hub_min=1000).slice_cost == \
        H.SpmvOperator.SLICE_COST  # the hub-row path balances by cost too
    with pytest.raises(ValueError, match="weights"):
        H.SpmvOperator(h32, schedule="stream", slice_cost="1,2")
    with pytest.raises(ValueError, match="weights"):
        H.SpmvOperator(h32, schedule="stream", slice_cost="1,2,3,4,99")


TAILS = ["0.95:1", "0.8:2", "0.5:4", "1.0:1"]


@pytest.mark.parametrize("name", [n for n in W32 if not n.startswith("kat")][:10])
@pytest.mark.parametrize("tail", TAILS)
@pytest.mark.parametrize("workers", [1, 5, None])
def test_stream_tail_matches_golden(name, tail, workers):
    """Tail pieces (a second, programmatically dependent launch over the last
    pieces): f64 bitwise the reference, f32 within 1e-5, repeat calls equal."""
    g = load_golden(name)
    val = g["trip_val"].astype(np.float32) if g["fp32"] else g["trip_val"]
    hbp = _hbp(g["rows"], g["cols"], g["trip_row"], g["trip_col"], val, g["C"], g["R"], g["W"],
               g["seed"])
    x = torch.as_tensor(g["x"].astype(np.float32) if g["fp32"] else g["x"], device="cuda")
    op = H.SpmvOperator(hbp, workers=workers, schedule="stream", tail=tail)
    assert op.launches_per_call >= 2
    y = op(x).cpu().numpy()
    for _ in range(3):
        np.testing.assert_array_equal(op(x).cpu().numpy(), y)
    if g["fp32"]:
        err = O.componentwise_error(g["rows"], g["trip_row"], g["trip_col"], g["trip_val"],
                                    g["x"], y.astype(np.float64))
        assert err <= 1e-5
    else:
        np.testing.assert_array_equal(y, g["y"])


@pytest.mark.parametrize("tail", TAILS)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("hub", [None, 2000])
def test_stream_tail_hot_rows(tail, dtype, hub):
    rows, cols, r, c, v = _hot_matrix()
    vv = v.astype(dtype)
    x = np.random.default_rng(1).uniform(-1, 1, cols).astype(dtype)
    hbp = _hbp(rows, cols, r, c, vv, C=cols)
    xd = torch.as_tensor(x, device="cuda")
    op = H.SpmvOperator(hbp, schedule="stream", tail=tail, hub_min=hub)
    y1 = op(xd).cpu().numpy()
    for _ in range(5):  # back to back: the dependent launch must not overtake later work
        y2 = op(xd)
    np.testing.assert_array_equal(y2.cpu().numpy(), y1)
    err = O.componentwise_error(rows, r, c, vv.astype(np.float64), x.astype(np.float64),
                                y1.astype(np.float64))
    assert err <= (1e-12 if dtype == np.float64 else 1e-5)
    if dtype == np.float64 and hub is None:  # exact: bitwise the static schedule
        ref = H.SpmvOperator(hbp, schedule="stream")(xd).cpu().numpy()
        np.testing.assert_array_equal(y1, ref)
