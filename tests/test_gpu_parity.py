"""CUDA path vs the reference's golden vectors (and the oracle), bit-exact.

Integer metadata (grid, hash params, probe counts, permutations, col,
add_sign, zero_row, group_start, output_hash, plan) must match exactly; fp64
partials and y bitwise (reference summation order, unfused); fp32 y within
1e-5 componentwise of the reference run in fp64 on the fp32-rounded inputs
(BASELINE.json north_star tolerance).
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

NAMES = golden_names()
FP32_TOL = 1e-5


def _cfg(g, f=None):
    return H.PartitionConfig(col_width=g["C"], row_height=g["R"], warp_size=g["W"],
                             fixed_fraction=g["fixed_fraction"] if f is None else f)


def _trip(g):
    val = g["trip_val"].astype(np.float32) if g["fp32"] else g["trip_val"]
    return H.TripletMatrix(g["rows"], g["cols"], g["trip_row"], g["trip_col"], val)


def _perms(g, grid, cfg, ctr=None):
    if g["ordering"] == "hash":
        params = H.sample_hash_params(grid, cfg, seed=g["seed"])
        return H.hash_permutations(grid, params, counter=ctr), params
    if g["ordering"] == "identity":
        return H.identity_permutations(grid), None
    return H.sort_permutations(grid), None


def _build(g):
    cfg = _cfg(g)
    csr = H.coo_to_csr(_trip(g))
    grid = H.make_grid(csr, cfg)
    perms, params = _perms(g, grid, cfg)
    return cfg, csr, grid, perms, params, H.build_hbp(csr, grid, perms)


def _np(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def _fp32_err(g, y):
    return O.componentwise_error(g["rows"], g["trip_row"], g["trip_col"], g["trip_val"], g["x"],
                                 _np(y).astype(np.float64))


@pytest.mark.parametrize("name", NAMES)
def test_pipeline_bit_exact(name):
    g = load_golden(name)
    cfg = _cfg(g)
    csr = H.coo_to_csr(_trip(g))
    np.testing.assert_array_equal(_np(csr.row_ptr), g["row_ptr"])
    np.testing.assert_array_equal(_np(csr.col_idx), g["trip_col"])
    grid = H.make_grid(csr, cfg)
    ref = grid.to_reference()
    for k in ("row_counts", "row_starts", "block_nnz", "block_elem_start"):
        np.testing.assert_array_equal(ref[k], g[k], err_msg=k)
    ctr = H.OpCounter()
    perms, params = _perms(g, grid, cfg, ctr)
    if params is not None:
        assert [params.a, params.b, params.c, params.d] == g["params"].tolist()
        assert ctr.probes == g["probes"]
    np.testing.assert_array_equal(np.asarray(perms), g["perms"])
    np.testing.assert_array_equal(np.asarray(H.sort_permutations(grid)), g["sort_perms"])
    hbp = H.build_hbp(csr, grid, perms)
    out = hbp.to_reference()
    for k in ("col", "add_sign", "zero_row", "group_start", "output_hash"):
        np.testing.assert_array_equal(out[k], g[k], err_msg=k)
    np.testing.assert_array_equal(out["data"], g["data"])
    np.testing.assert_array_equal(hbp.block_nnz_matrix(), g["block_nnz"])


@pytest.mark.parametrize("name", NAMES)
def test_spmv_and_combine(name):
    g = load_golden(name)
    cfg, csr, grid, perms, params, hbp = _build(g)
    plan = H.plan_execution(hbp, cfg, g["workers"])
    np.testing.assert_array_equal(plan.block_order, g["block_order"])
    assert plan.fixed_count == g["fixed_count"]
    np.testing.assert_array_equal(np.asarray(plan.worker_ranges).reshape(-1, 2),
                                  g["worker_ranges"])
    x = g["x"].astype(np.float32) if g["fp32"] else g["x"]
    partial, log = H.run_spmv(hbp, x, plan, g["workers"])
    assert (log.worker >= 0).all()
    kinds = np.where(np.arange(plan.num_blocks) < plan.fixed_count, 0, 1)
    np.testing.assert_array_equal(log.kind, kinds)
    for w, (a, b) in enumerate(plan.worker_ranges):
        assert (log.worker[a:b] == w).all()
    y = H.combine(partial)
    y_fast = H.hbp_spmv(hbp, x)
    if g["fp32"]:
        assert _fp32_err(g, y) <= FP32_TOL
        assert _fp32_err(g, y_fast) <= FP32_TOL
    else:
        np.testing.assert_array_equal(_np(partial.values), g["partial"])
        np.testing.assert_array_equal(_np(y), g["y"])
        np.testing.assert_array_equal(_np(y_fast), g["y"])


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith(("corpus_powerlaw_2000",
                                                                   "default", "geo"))])
def test_bitwise_across_workers_and_splits(name):
    """test_engine.py:156-169 / test_acceptance.py:164-197 on the GPU."""
    g = load_golden(name)
    x = g["x"].astype(np.float32) if g["fp32"] else g["x"]
    ref = None
    for f in (0.0, 0.3, 0.7, 1.0):
        cfg = _cfg(g, f)
        csr = H.coo_to_csr(_trip(g))
        grid = H.make_grid(csr, cfg)
        perms, _ = _perms(g, grid, cfg)
        hbp = H.build_hbp(csr, grid, perms)
        for workers in (1, 2, 5, None):
            plan = H.plan_execution(hbp, cfg, workers)
            partial, log = H.run_spmv(hbp, x, plan, plan.workers)
            y = _np(H.combine(partial))
            assert (log.worker >= 0).all()
            if ref is None:
                ref = y
            np.testing.assert_array_equal(y, ref)
    if not g["fp32"]:
        np.testing.assert_array_equal(ref, g["y"])


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith(("kat", "special", "geo"))])
def test_walker_inverts_format(name):
    g = load_golden(name)
    *_, hbp = _build(g)
    back = H.hbp_to_triplets(hbp).canonicalized()
    r, c, v = back.to_numpy()
    np.testing.assert_array_equal(r, g["trip_row"])
    np.testing.assert_array_equal(c, g["trip_col"])
    np.testing.assert_array_equal(v, g["trip_val"] if not g["fp32"] else
                                  g["trip_val"].astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("name", ["corpus_uniform_64x64_s0", "geo_w4_r16_c64",
                                  "special_indivisible_130x70", "kat_eye8"])
def test_codec_byte_identical(name, tmp_path):
    """The .hbp bytes written from the GPU-built format equal the reference's
    layout (hbp.py:318-391), and load back to the same arrays."""
    import io
    g = load_golden(name)
    *_, hbp = _build(g)
    buf = io.BytesIO()
    H.serialize_hbp(hbp, buf)
    raw = buf.getvalue()
    back = H.deserialize_hbp(io.BytesIO(raw))
    buf2 = io.BytesIO()
    H.serialize_hbp(back, buf2)
    assert buf2.getvalue() == raw
    y = H.hbp_spmv(back, g["x"])
    np.testing.assert_array_equal(_np(y), g["y"])
    if name == "kat_eye8":
        assert len(raw) == 448  # test_hbp.py:224-232


@pytest.mark.parametrize("name", NAMES)
def test_baselines_bitwise(name):
    """GPU csr_spmv / block2d_spmv_baseline vs the reference's (f64 bitwise)."""
    g = load_golden(name)
    cfg = _cfg(g)
    csr = H.coo_to_csr(_trip(g))
    grid = H.make_grid(csr, cfg)
    x = g["x"].astype(np.float32) if g["fp32"] else g["x"]
    y_csr = _np(H.csr_spmv(csr, x))
    y_2d = _np(H.block2d_spmv_baseline(csr, grid, x, workers=2))
    if g["fp32"]:
        assert _fp32_err(g, y_csr) <= FP32_TOL
        assert _fp32_err(g, y_2d) <= FP32_TOL
    else:
        np.testing.assert_array_equal(y_csr, g["y_csr"])
        np.testing.assert_array_equal(y_2d, g["y_2d"])
