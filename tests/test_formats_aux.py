"""Host-side data formats around the hot path (CPU): the synthetic generator,
Matrix Market tokenizer / writer and the metrics helpers, pinned to fixtures
the reference produced (tests/golden/make_golden_aux.py) and to the
reference tests' known answers (test_synth.py, test_formats.py:41-130,
test_metrics.py)."""
from __future__ import annotations

import glob
import io
import os
import types

import numpy as np
import pytest

from paper_2504_08860_b200.metrics import (BenchReport, GroupStats, Timing, gflops,
                                           group_stats_csv, mean_group_std, reduction_summary,
                                           time_kernel)
from paper_2504_08860_b200.mtx import (MatrixMarketError, read_matrix_market_arrays,
                                       write_matrix_market)
from paper_2504_08860_b200.synth import SyntheticSpec, generate_arrays

AUX = os.path.join(os.path.dirname(__file__), "golden", "aux")


def _synth_cases():
    return sorted(glob.glob(os.path.join(AUX, "synth_*.npz")))


@pytest.mark.parametrize("path", _synth_cases(), ids=os.path.basename)
def test_generator_is_the_reference_matrix(path):
    g = np.load(path)
    rows, cols, mean, alpha, seed = g["spec"]
    spec = SyntheticSpec(int(rows), int(cols), str(g["pattern"]), float(mean), alpha=float(alpha),
                         seed=int(seed))
    r, c, v = generate_arrays(spec)
    np.testing.assert_array_equal(r, g["row"])
    np.testing.assert_array_equal(c, g["col"])
    np.testing.assert_array_equal(v, g["val"])


@pytest.mark.parametrize("kwargs", [{"rows": 0}, {"cols": 0}, {"pattern": "gaussian"},
                                    {"mean_nnz_per_row": 0.0}, {"mean_nnz_per_row": 100.0},
                                    {"pattern": "powerlaw", "alpha": 1.0}])
def test_spec_validation(kwargs):
    base = dict(rows=10, cols=10, pattern="uniform", mean_nnz_per_row=3.0)
    base.update(kwargs)
    with pytest.raises(ValueError):
        SyntheticSpec(**base)


def test_generator_properties():
    r, c, v = generate_arrays(SyntheticSpec(8, 5, "uniform", 5.0, seed=2))
    assert r.size == 40  # dense request fills rows
    r, c, v = generate_arrays(SyntheticSpec(100, 100, "uniform", 6.0, seed=1))
    assert np.all(np.abs(v) <= 1.0) and np.all(v != 0.0)
    assert np.unique(r * 100 + c).size == r.size


SIMPLE = ("%%MatrixMarket matrix coordinate real general\n% a comment line\n3 4 4\n"
          "1 1 2.5\n3 4 -1.0\n2 2 7.25\n3 1 0.5\n")


def test_tokenizer_simple():
    hd, rows, cols, i, j, v = read_matrix_market_arrays(SIMPLE)
    assert (hd.format, hd.field, hd.symmetry) == ("coordinate", "real", "general")
    assert (rows, cols) == (3, 4)
    assert set(zip(i.tolist(), j.tolist(), v.tolist())) == {(0, 0, 2.5), (2, 3, -1.0),
                                                            (1, 1, 7.25), (2, 0, 0.5)}
    hd2, *_ = read_matrix_market_arrays(io.StringIO(SIMPLE.replace("%%MatrixMarket",
                                                                   "%%matrixmarket")))
    assert hd2 == hd


@pytest.mark.parametrize("text, fragment", [
    ("", "empty"),
    ("not a banner\n1 1 0\n", "banner"),
    ("%%MatrixMarket vector coordinate real general\n1 1 0\n", "object"),
    ("%%MatrixMarket matrix array real general\n1 1\n", "format"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", "field"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n", "symmetry"),
    ("%%MatrixMarket matrix coordinate real general\n", "size"),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", "3 integers"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 x\n", "size"),
    ("%%MatrixMarket matrix coordinate real general\n-1 2 0\n", "negative"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "entries"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "bounds"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n", "value"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1.5 1 1.0\n", "index"),
])
def test_tokenizer_rejects(text, fragment):
    with pytest.raises(MatrixMarketError, match=fragment):
        read_matrix_market_arrays(text)


def test_writer_matches_reference_text():
    m = np.load(os.path.join(AUX, "mtx.npz"))
    k = 0
    while f"text_{k}" in m:
        rows, cols = m[f"shape_{k}"]
        host = types.SimpleNamespace(rows=int(rows), cols=int(cols), nnz=m[f"val_{k}"].size,
                                     row=m[f"row_{k}"], col=m[f"col_{k}"], val=m[f"val_{k}"])
        assert write_matrix_market(host) == str(m[f"written_{k}"])
        k += 1
    assert k >= 5


def _stats_cases():
    return sorted(glob.glob(os.path.join(AUX, "stats_*.npz")))


@pytest.mark.parametrize("path", _stats_cases(), ids=os.path.basename)
def test_from_lanes_and_summaries_match_reference(path):
    g = np.load(path)
    W = int(g["geom"][4])
    tables = {}
    for name in ("none", "hash", "sort"):
        keys, sizes, lanes = g[f"{name}_keys"], g[f"{name}_sizes"], g[f"{name}_lanes"]
        st = [GroupStats.from_lanes(int(k[0]), int(k[1]), int(k[2]), lanes[i, :sizes[i]], W)
              for i, k in enumerate(keys)]
        np.testing.assert_array_equal([s.mean for s in st], g[f"{name}_mean"])
        np.testing.assert_array_equal([s.std_dev for s in st], g[f"{name}_std"])
        np.testing.assert_array_equal([s.utilization for s in st], g[f"{name}_util"])
        assert mean_group_std(st, W) == float(g[f"{name}_mean_std"])
        assert mean_group_std(st, W, full_only=False) == float(g[f"{name}_mean_std_all"])
        tables[name] = st
    assert reduction_summary(tables["none"], tables["hash"], W) == float(g["reduction_hash"])
    assert group_stats_csv(tables["hash"][:50], "hash") == str(g["csv_hash_head"])


def test_metrics_known_answers():
    s = GroupStats.from_lanes(0, 0, 0, np.array([0, 1, 2, 1]), 4)
    assert s.mean == 1.0 and s.max == 2 and s.utilization == 0.5
    assert s.std_dev == pytest.approx(np.sqrt(0.5))
    z = GroupStats.from_lanes(0, 0, 0, np.zeros(4, dtype=int), 4)
    assert z.std_dev == 0.0 and z.utilization == 1.0
    stats = [GroupStats.from_lanes(0, 0, 0, np.array([2, 2]), 2)]
    assert reduction_summary(stats, stats, 2) == 0.0
    with pytest.raises(ValueError, match="coverage"):
        reduction_summary([GroupStats.from_lanes(0, 0, 0, np.array([1, 2]), 2)],
                          [GroupStats.from_lanes(1, 0, 0, np.array([1, 2]), 2)], 2)
    lines = group_stats_csv([GroupStats.from_lanes(0, 1, 2, np.array([1, 3]), 2)],
                            "hash").strip().split("\n")
    assert lines[0] == "block_br,block_bc,group,ordering,mean,std_dev,utilization"
    assert lines[1].startswith("0,1,2,hash,2,1,")
    assert gflops(1_000_000, 0.001) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        gflops(100, 0.0)
    full = GroupStats.from_lanes(0, 0, 0, np.array([0, 4]), 2)
    partial = GroupStats.from_lanes(1, 0, 0, np.array([9]), 2)
    assert mean_group_std([full, partial], 2) == full.std_dev
    assert mean_group_std([], 2) == 0.0


def test_time_kernel_and_report():
    calls = []
    t = time_kernel(lambda: calls.append(1), iterations=5, warmup=2, device=False)
    assert len(calls) == 7 and t.iterations == 5 and t.min <= t.median <= t.max
    with pytest.raises(ValueError):
        time_kernel(lambda: None, iterations=0, device=False)
    r = BenchReport(matrix="m", rows=10, cols=10, nnz=1234, workers=2, fixed_fraction=0.7,
                    config={"col_width": 16})
    r.add_kernel("csr", Timing(0.5, 0.4, 0.6, 3))
    r.add_kernel("hbp", Timing(0.3, 0.2, 0.4, 2), spmv_s=0.25, combine_s=0.05)
    assert r.kernels["csr"]["gflops"] == pytest.approx(2.0 * 1234 / 0.5 / 1e9, rel=1e-15)
    assert r.kernels["hbp"]["combine_s"] == 0.05
    import json
    back = json.loads(r.to_json())
    assert back["config"]["col_width"] == 16 and "csr" in back["kernels"]
