"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference.

Every array the reference produced for every golden case must be reproduced
bit-exactly by the oracle restatement before the oracle is trusted as the
checker for the CUDA path.  CPU only.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import oracle as O

NAMES = golden_names()


def test_golden_corpus_present():
    assert len(NAMES) >= 74  # 48 acceptance-corpus matrices (seeds 0-3) included


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_reference(name):
    g = load_golden(name)
    rows, cols, C, R, W = g["rows"], g["cols"], g["C"], g["R"], g["W"]
    row_ptr, col_idx, values = O.coo_to_csr(rows, cols, g["trip_row"], g["trip_col"],
                                             g["trip_val"])
    np.testing.assert_array_equal(row_ptr, g["row_ptr"])
    grid = O.make_grid(row_ptr, col_idx, rows, cols, C, R, W)
    for k in ("row_counts", "row_starts", "block_nnz", "block_elem_start"):
        np.testing.assert_array_equal(getattr(grid, k), g[k], err_msg=k)
    params = O.sample_hash_params(grid, seed=g["seed"])
    np.testing.assert_array_equal(params, g["params"])
    if g["ordering"] == "hash":
        perms, probes = O.hash_permutations(grid, params)
        assert probes == g["probes"]
    elif g["ordering"] == "identity":
        perms = O.identity_permutations(grid)
    else:
        perms = O.sort_permutations(grid)
    np.testing.assert_array_equal(perms, g["perms"])
    np.testing.assert_array_equal(O.sort_permutations(grid), g["sort_perms"])
    h = O.build_hbp(row_ptr, col_idx, values, grid, perms)
    for k in ("col", "data", "add_sign", "zero_row", "group_start", "output_hash"):
        np.testing.assert_array_equal(getattr(h, k), g[k], err_msg=k)
    order, fixed, ranges = O.plan_execution(h.block_nnz_matrix(), g["fixed_fraction"],
                                            g["workers"])
    np.testing.assert_array_equal(order, g["block_order"])
    assert fixed == g["fixed_count"]
    np.testing.assert_array_equal(np.asarray(ranges).reshape(-1, 2), g["worker_ranges"])
    partial, log = O.run_spmv(h, g["x"], (order, fixed, ranges), g["workers"], with_log=True)
    np.testing.assert_array_equal(partial, g["partial"])
    y = O.combine(partial, rows, h.ncb)
    np.testing.assert_array_equal(y, g["y"])  # bitwise: unfused, same order
    assert (log["worker"] >= 0).all()


@pytest.mark.parametrize("name", NAMES)
def test_rows_blocked_restatement_matches_reference_y(name):
    """O.rows_blocked (per-block step-order sums folded in ascending bc, no
    dense layout) reproduces the reference's y bit for bit on every golden
    case: it is the checker the full-size parity tests use."""
    g = load_golden(name)
    row_ptr, col_idx, values = O.coo_to_csr(g["rows"], g["cols"], g["trip_row"], g["trip_col"],
                                             g["trip_val"])
    y = O.rows_blocked(row_ptr, col_idx, values, g["x"], g["C"], np.arange(g["rows"]))
    np.testing.assert_array_equal(y, g["y"])


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith(("kat", "special", "geo"))])
def test_oracle_walker_inverts_format(name):
    g = load_golden(name)
    p = O.pipeline(g["rows"], g["cols"], g["trip_row"], g["trip_col"], g["trip_val"],
                   g["C"], g["R"], g["W"], seed=g["seed"], ordering=g["ordering"])
    r, c, v = O.hbp_to_triplets(p["hbp"])
    r2, c2, v2 = O.canonicalize(g["rows"], g["cols"], r, c, v)
    np.testing.assert_array_equal(r2, g["trip_row"])
    np.testing.assert_array_equal(c2, g["trip_col"])
    np.testing.assert_array_equal(v2, g["trip_val"])


def test_known_answers_from_reference_tests():
    """Hand-computed vectors quoted in the reference tests (test_hbp.py:69-91,
    test_reorder.py:41-79, test_partition.py:68-100)."""
    g = load_golden("kat_single_group")
    assert g["col"].tolist() == [0, 1, 3, 2]
    assert g["add_sign"].tolist() == [-1, 2, -1, -1]
    assert g["zero_row"].tolist() == [-1, 1, 1, 1]
    assert g["group_start"].tolist() == [0, 4]
    g = load_golden("kat_strides_cross_group")
    assert g["add_sign"].tolist() == [2, -1, -1, 2, -1, 1, -1]
    assert g["group_start"].tolist() == [0, 3, 7]
    g = load_golden("kat_survey_8x8")
    assert g["col"].tolist() == [0, 3, 1, 2, 0, 1, 2, 3, 5, 4, 6, 7, 7]
    assert g["add_sign"].tolist() == [2, -1, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, -1]
    assert g["zero_row"].tolist() == [0, 0, 0, -1, -1, 1, -1, -1, 0, -1, 0, -1, -1, -1, -1, 1]
    assert g["group_start"].tolist() == [0, 4, 5, 8, 8, 9, 12, 12, 13]
    # reorder goldens
    assert O.hash_slot(100, 5, 0, 4, 1, 4) == 33
    assert O.hash_slot(13, 4, 1, 7, 3, 7) == 47
    perm, _ = O.hash_perm_block([5, 1, 0, 2, 1, 1, 6, 0], 0, 1, 1, 1)
    assert perm.tolist() == [2, 1, 3, 4, 5, 0, 6, 7]
    _, probes = O.hash_perm_block([0] * 6, 0, 1, 1, 1)
    assert probes == 15
    perm, _ = O.hash_perm_block([3, 2], 0, 1, 1, 1)
    assert perm.tolist() == [1, 0]
    g = load_golden("kat_grid_4x4")
    assert g["row_counts"].tolist() == [[1, 0, 2, 0], [1, 0, 1, 1]]
    assert g["row_starts"].tolist() == [[0, 2, 2, 5], [1, 2, 4, 5]]
    assert g["block_elem_start"].tolist() == [[0, 3], [1, 4]]


def test_quantile_restatement_matches_numpy(rng):
    for n in (1, 2, 9, 10, 11, 4096, 333):
        v = rng.integers(0, 50, n)
        assert O.quantile_inverted_cdf(v, 0.9) == np.quantile(v, 0.9, method="inverted_cdf")


def test_shift_follows_quantile():
    """test_reorder.py:108-118: q90 = 35 needs a = 2."""
    dense = np.zeros((64, 64))
    dense[:56, :4] = 1.0
    dense[56:, :35] = 1.0
    r, c = np.nonzero(dense)
    rp, ci, v = O.coo_to_csr(64, 64, r, c, dense[r, c])
    grid = O.make_grid(rp, ci, 64, 64, 64, 64, 8)
    assert O.sample_hash_params(grid)[0] == 2


def test_duplicates_rejected():
    with pytest.raises(ValueError, match="duplicate"):
        O.coo_to_csr(2, 2, [0, 0], [1, 1], [1.0, 2.0])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_baselines(name):
    """csr_spmv and block2d_spmv_baseline (the paper's comparison kernels)."""
    g = load_golden(name)
    rp, ci, vals = O.coo_to_csr(g["rows"], g["cols"], g["trip_row"], g["trip_col"], g["trip_val"])
    np.testing.assert_array_equal(O.csr_spmv(rp, ci, vals, g["x"]), g["y_csr"])
    grid = O.make_grid(rp, ci, g["rows"], g["cols"], g["C"], g["R"], g["W"])
    np.testing.assert_array_equal(O.block2d_spmv_baseline(rp, ci, vals, grid, g["x"]), g["y_2d"])
