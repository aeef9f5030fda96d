"""GPU side of the data-format rows: group statistics from the hbp_group_stats
kernel, Matrix Market canonicalisation / symmetric expansion on the device
and the device TripletMatrix of the generator -- all against fixtures the
reference produced (tests/golden/make_golden_aux.py)."""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_2504_08860_b200 as H

AUX = os.path.join(os.path.dirname(__file__), "golden", "aux")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(AUX, "stats_*.npz"))),
                         ids=os.path.basename)
def test_group_stats_bitwise(path):
    g = np.load(path)
    rows, cols, C, R, W, seed = (int(v) for v in g["geom"])
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W)
    trip = H.generate(H.SyntheticSpec(rows, cols, str(g["pattern"]), float(g["mean_nnz"]),
                                      seed=seed))
    grid = H.make_grid(H.coo_to_csr(trip), cfg)
    params = H.sample_hash_params(grid, cfg)
    tables = {}
    for name, perms in (("none", None), ("hash", H.hash_permutations(grid, params)),
                        ("sort", H.sort_permutations(grid))):
        t = H.group_stats(grid, perms)
        tables[name] = t
        np.testing.assert_array_equal(t.keys(), g[f"{name}_keys"])
        np.testing.assert_array_equal(t.sizes, g[f"{name}_sizes"])
        lanes = g[f"{name}_lanes"]
        np.testing.assert_array_equal(t.lanes, lanes)
        np.testing.assert_array_equal(t.mean, g[f"{name}_mean"])
        np.testing.assert_array_equal(t.std_dev, g[f"{name}_std"])
        np.testing.assert_array_equal(t.max, g[f"{name}_max"])
        np.testing.assert_array_equal(t.utilization, g[f"{name}_util"])
        assert H.mean_group_std(t, W) == float(g[f"{name}_mean_std"])
        assert H.mean_group_std(t, W, full_only=False) == float(g[f"{name}_mean_std_all"])
    assert H.reduction_summary(tables["none"], tables["hash"], W) == float(g["reduction_hash"])
    assert H.reduction_summary(tables["none"], tables["sort"], W) == float(g["reduction_sort"])
    head = [tables["hash"][i] for i in range(min(50, len(tables["hash"])))]
    assert H.group_stats_csv(head, "hash") == str(g["csv_hash_head"])
    # a dense reference-layout table gives the same statistics
    dense = np.asarray(H.hash_permutations(grid, params))
    np.testing.assert_array_equal(H.group_stats(grid, dense).std_dev, g["hash_std"])


def test_hash_reorder_lowers_mean_std():
    """test_metrics.py:65-75."""
    cfg = H.PartitionConfig(col_width=256, row_height=64, warp_size=8)
    trip = H.generate(H.SyntheticSpec(512, 256, "powerlaw", 8.0, seed=2))
    grid = H.make_grid(H.coo_to_csr(trip), cfg)
    params = H.sample_hash_params(grid, cfg)
    before = H.mean_group_std(H.group_stats(grid, None), 8)
    after = H.mean_group_std(H.group_stats(grid, H.hash_permutations(grid, params)), 8)
    sorted_ = H.mean_group_std(H.group_stats(grid, H.sort_permutations(grid)), 8)
    assert sorted_ <= after < before


def test_matrix_market_on_device():
    m = np.load(os.path.join(AUX, "mtx.npz"))
    k = 0
    while f"text_{k}" in m:
        hd, t = H.parse_matrix_market(str(m[f"text_{k}"]))
        assert [hd.object, hd.format, hd.field, hd.symmetry] == m[f"hdr_{k}"].tolist()
        r, c, v = t.to_numpy()
        np.testing.assert_array_equal(r, m[f"row_{k}"])
        np.testing.assert_array_equal(c, m[f"col_{k}"])
        np.testing.assert_array_equal(v, m[f"val_{k}"])
        assert H.write_matrix_market(t) == str(m[f"written_{k}"])
        if f"sym_row_{k}" in m:
            e = H.expand_symmetric(t)
            r, c, v = e.to_numpy()
            np.testing.assert_array_equal(r, m[f"sym_row_{k}"])
            np.testing.assert_array_equal(c, m[f"sym_col_{k}"])
            np.testing.assert_array_equal(v, m[f"sym_val_{k}"])
        k += 1
    with pytest.raises(ValueError, match="square"):
        H.expand_symmetric(H.TripletMatrix(2, 3, [0], [1], [1.0]))
    with pytest.raises(ValueError, match="ambiguous"):
        H.expand_symmetric(H.TripletMatrix(3, 3, [0, 1], [1, 0], [1.0, 2.0]))


def test_mtx_file_round_trip_and_dense(tmp_path):
    rng = np.random.default_rng(0)
    dense = rng.uniform(-1, 1, (6, 5)) * (rng.random((6, 5)) < 0.4)
    r, c = np.nonzero(dense)
    t = H.TripletMatrix(6, 5, r, c, dense[r, c])
    path = tmp_path / "m.mtx"
    H.save_mtx(t, path)
    _, back = H.load_mtx(path)
    np.testing.assert_array_equal(H.to_dense(back), dense)
    x = rng.uniform(-1, 1, 5)
    np.testing.assert_allclose(H.dense_oracle_spmv(back, x), dense @ x, rtol=1e-14, atol=1e-15)
    with pytest.raises(ValueError, match="length"):
        H.dense_oracle_spmv(back, np.zeros(4))


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(AUX, "synth_*.npz")))[:4],
                         ids=os.path.basename)
def test_generate_on_device(path):
    g = np.load(path)
    rows, cols, mean, alpha, seed = g["spec"]
    t = H.generate(H.SyntheticSpec(int(rows), int(cols), str(g["pattern"]), float(mean),
                                   alpha=float(alpha), seed=int(seed)))
    r, c, v = t.to_numpy()
    np.testing.assert_array_equal(r, g["row"])
    np.testing.assert_array_equal(c, g["col"])
    np.testing.assert_array_equal(v, g["val"])
