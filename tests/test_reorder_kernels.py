"""Row orderings (reorder.py:106-231) on their own: the warp-per-block hash
(and its thread-per-block fallback for R > 1024), the block radix sort2D and
the merge-sort comparison count, each against the oracle restatement of the
reference (oracle/oracle.py, pinned here to reference-made fixtures) across
block heights, hash constants and key distributions the golden cases do not
reach one by one."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O

AUX = os.path.join(os.path.dirname(__file__), "golden", "aux")


def _sortcmp():
    z = np.load(os.path.join(AUX, "sortcmp.npz"))
    n = len([k for k in z.files if k.startswith("keys_")])
    return [(z[f"keys_{i}"], z[f"perm_{i}"], int(z[f"cmp_{i}"])) for i in range(n)]


def test_oracle_merge_sort_matches_reference_fixture():
    for keys, perm, cmp in _sortcmp():
        p, c = O.counting_merge_sort(keys)
        np.testing.assert_array_equal(p, perm)
        assert c == cmp
        np.testing.assert_array_equal(O.sort_permutation(keys), perm)


HASH_CASES = [
    # (n, a, b, c, bucket_max, distribution)
    (1, 0, 1, 1, 8, "uniform"),
    (5, 0, 1, 3, 8, "uniform"),
    (31, 1, 3, 2, 8, "powerlaw"),
    (32, 0, 3, 5, 8, "uniform"),
    (33, 0, 3, 5, 8, "same"),
    (100, 2, 11, 7, 8, "powerlaw"),
    (512, 0, 56, 73, 8, "same"),       # cfg3-like: every row in one bucket
    (512, 1, 56, 51, 8, "powerlaw"),   # cfg2 constants
    (512, 2, 56, 27, 8, "uniform"),
    (512, 0, 56, 57, 8, "zeros"),      # empty block: all homes in one 56-slot window
    (777, 3, 86, 3, 8, "powerlaw"),
    (1000, 0, 111, 7, 8, "same"),
    (1024, 0, 113, 9, 8, "uniform"),
    (1025, 0, 113, 9, 8, "uniform"),   # thread-per-block fallback
    (3000, 1, 333, 7, 8, "powerlaw"),
    (512, 40, 56, 73, 8, "uniform"),   # a >= 32
    (300, 0, 33, 1, 3, "uniform"),     # other bucket_max
]


def _lens(n, dist, rng):
    if dist == "uniform":
        return rng.integers(0, 40, n)
    if dist == "powerlaw":
        return (rng.zipf(1.6, n) - 1) % 100000
    if dist == "same":
        return np.full(n, 33)
    return np.zeros(n, np.int64)


@pytest.mark.gpu
@pytest.mark.parametrize("case", HASH_CASES, ids=lambda c: f"n{c[0]}_a{c[1]}_{c[5]}")
def test_hash_block_matches_oracle(case):
    import paper_2504_08860_b200 as H
    n, a, b, c, bmax, dist = case
    rng = np.random.default_rng(n * 7 + a)
    lens = _lens(n, dist, rng)
    params = H.HashParams(a=a, b=b, c=c, d=b, bucket_max=bmax)
    ctr = H.OpCounter()
    perm = H.build_block_permutation(lens, params, ctr)
    want, probes = O.hash_perm_block(lens, a, b, c, b, bmax)
    np.testing.assert_array_equal(perm, want)
    assert ctr.probes == probes


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 56, 64, 96, 500, 512, 1024, 1500])
def test_hash_empty_block_matches_oracle(n):
    import paper_2504_08860_b200 as H
    from paper_2504_08860_b200.reorder import BlockPermutations
    params = H.HashParams(a=1, b=56, c=57, d=56)
    bp = BlockPermutations.__new__(BlockPermutations)
    bp.kind, bp.params = "hash", params
    import torch
    bp.compact = torch.empty(0, device="cuda")
    want, _ = O.hash_perm_block(np.zeros(n, np.int64), 1, 56, 57, 56)
    np.testing.assert_array_equal(bp.empty_block_perm(n), want)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 5, 100, 128, 129, 256, 511, 512, 1024, 2048, 2049, 3000])
@pytest.mark.parametrize("dist", ["uniform", "powerlaw", "same", "zeros", "wide"])
def test_sort_permutation_matches_oracle(n, dist):
    import paper_2504_08860_b200 as H
    rng = np.random.default_rng(n)
    lens = rng.integers(0, 1 << 30, n) if dist == "wide" else _lens(n, dist, rng)
    np.testing.assert_array_equal(H.sort_permutation(lens), O.sort_permutation(lens))


@pytest.mark.gpu
def test_sort_comparisons_match_reference_fixture():
    import paper_2504_08860_b200 as H
    for keys, perm, cmp in _sortcmp():
        ctr = H.OpCounter()
        np.testing.assert_array_equal(H.sort_permutation(keys, counter=ctr), perm)
        assert ctr.comparisons == cmp
        assert ctr.probes == 0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 17, 100, 4097])
def test_sort_comparisons_match_oracle(n):
    import paper_2504_08860_b200 as H
    rng = np.random.default_rng(n)
    for keys in (rng.integers(0, 9, n), rng.integers(0, 1 << 31, n), np.sort(rng.integers(0, 9, n))):
        ctr = H.OpCounter()
        H.sort_permutation(keys, counter=ctr)
        assert ctr.comparisons == O.counting_merge_sort(keys)[1]
        assert 0 < ctr.comparisons <= n * int(np.ceil(np.log2(n)))  # test_reorder.py:97


@pytest.mark.gpu
@pytest.mark.parametrize("R", [8, 24, 128, 512, 1024, 2048])
def test_block_orderings_of_a_grid(R):
    """hash_permutations / sort_permutations over a whole grid (ragged last
    row block, empty blocks) against the oracle's dense tables."""
    import paper_2504_08860_b200 as H
    rows = 3 * R + R // 3 + 1
    trip = H.generate(H.SyntheticSpec(rows, 4 * R, "powerlaw", 9.0, seed=R))
    cfg = H.PartitionConfig(col_width=2 * R, row_height=R, warp_size=8)
    csr = H.coo_to_csr(trip)
    grid = H.make_grid(csr, cfg)
    params = H.sample_hash_params(grid, cfg)
    rp, ci, _ = O.coo_to_csr(rows, 4 * R, *[t.cpu().numpy() for t in
                                            (trip.row, trip.col, trip.val)])
    dg = O.make_grid(rp, ci, rows, 4 * R, 2 * R, R, 8)
    want_h, want_probes = O.hash_permutations(dg, (params.a, params.b, params.c, params.d))
    ctr = H.OpCounter()
    np.testing.assert_array_equal(np.asarray(H.hash_permutations(grid, params, ctr)), want_h)
    assert ctr.probes == want_probes
    np.testing.assert_array_equal(np.asarray(H.sort_permutations(grid)), O.sort_permutations(dg))

