"""Golden fixtures for the data-format rows around the hot path, produced by
running the REFERENCE package (build container only; /root/reference is
absent on the GPU box, the .npz files travel instead).  Usage:

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden_aux.py

Writes tests/golden/aux/:
  synth_<i>.npz   spec + the canonical triplets of generate(SyntheticSpec)
                  (synth.py:116-125);
  stats_<i>.npz   group_stats lanes / mean / std_dev / max / utilization in
                  the reference's group order for the unordered, hash and
                  sort orderings (metrics.py:53-75), plus mean_group_std and
                  reduction_summary;
  sortcmp.npz     sort_permutation(row_nnz, counter) of a few key arrays:
                  the permutation and OpCounter.comparisons of the
                  instrumented merge sort (reorder.py:139-171);
  mtx.npz         parse_matrix_market of a few texts (formats.py:124-194):
                  canonical triplets, incl. duplicates, pattern and integer
                  fields and a symmetric expansion (formats.py:222-240).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "aux")

SYNTH = [
    (60, 45, "uniform", 5.0, 2.0, 0),
    (60, 45, "powerlaw", 5.0, 2.0, 0),
    (100, 100, "uniform", 6.0, 2.0, 1),
    (8, 5, "uniform", 5.0, 2.0, 2),
    (128, 96, "powerlaw", 7.0, 2.0, 11),
    (1024, 1024, "powerlaw", 8.0, 2.0, 3),
    (2000, 300, "powerlaw", 40.0, 1.5, 4),   # dense rows (> cols/2) exercised
    (4096, 1024, "uniform", 16.0, 2.0, 3),
    (1, 977, "uniform", 60.0, 2.0, 0),
    (771, 1, "uniform", 1.0, 2.0, 0),
]

STATS = [
    # (rows, cols, pattern, mean, seed, C, R, W)
    (20, 30, "uniform", 4.0, 0, 16, 8, 4),
    (64, 64, "powerlaw", 5.0, 1, 16, 8, 4),
    (512, 256, "powerlaw", 8.0, 2, 256, 64, 8),
    (256, 256, "powerlaw", 8.0, 3, 256, 64, 8),
    (1000, 700, "powerlaw", 9.0, 5, 256, 96, 32),
    (3000, 2500, "uniform", 12.0, 6, 1024, 512, 32),
]

MTX = [
    "%%MatrixMarket matrix coordinate real general\n% a comment line\n3 4 4\n"
    "1 1 2.5\n3 4 -1.0\n2 2 7.25\n3 1 0.5\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 1 2.0\n2 2 5.0\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 2\n2 3\n",
    "%%MatrixMarket matrix coordinate integer general\n2 2 1\n2 1 -3\n",
    "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n1 1 1.0\n3 1 4.0\n",
    "%%matrixmarket matrix coordinate real general\n4 4 6\n4 4 0.1\n1 2 1e-300\n"
    "1 2 3.3\n2 1 -0.5\n1 2 7\n3 3 1.7976931348623157e308\n",
]


def _ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
    sys.path.insert(0, REF)
    import hbp_spmv  # noqa: E402
    return hbp_spmv


def main():
    h = _ref()
    os.makedirs(OUT, exist_ok=True)
    for i, (rows, cols, pat, mean, alpha, seed) in enumerate(SYNTH):
        t = h.generate(h.SyntheticSpec(rows, cols, pat, mean, alpha=alpha, seed=seed))
        np.savez_compressed(os.path.join(OUT, f"synth_{i}.npz"),
                            spec=np.array([rows, cols, mean, alpha, seed], np.float64),
                            pattern=np.array(pat), row=t.row, col=t.col, val=t.val)
    for i, (rows, cols, pat, mean, seed, C, R, W) in enumerate(STATS):
        cfg = h.PartitionConfig(col_width=C, row_height=R, warp_size=W)
        trip = h.generate(h.SyntheticSpec(rows, cols, pat, mean, seed=seed))
        grid = h.make_grid(h.coo_to_csr(trip), cfg)
        params = h.sample_hash_params(grid, cfg)
        out = dict(geom=np.array([rows, cols, C, R, W, seed], np.int64), pattern=np.array(pat),
                   mean_nnz=np.array(mean))
        per = {}
        for name, perms in (("none", None), ("hash", h.hash_permutations(grid, params)),
                            ("sort", h.sort_permutations(grid))):
            st = h.group_stats(grid, perms)
            per[name] = st
            lanes = np.zeros((len(st), W), np.int64)
            sizes = np.array([s.lane_nnz.size for s in st], np.int64)
            for k, s in enumerate(st):
                lanes[k, :s.lane_nnz.size] = s.lane_nnz
            out[f"{name}_keys"] = np.array([(s.br, s.bc, s.group) for s in st], np.int64)
            out[f"{name}_sizes"] = sizes
            out[f"{name}_lanes"] = lanes
            out[f"{name}_mean"] = np.array([s.mean for s in st])
            out[f"{name}_std"] = np.array([s.std_dev for s in st])
            out[f"{name}_max"] = np.array([s.max for s in st], np.int64)
            out[f"{name}_util"] = np.array([s.utilization for s in st])
            out[f"{name}_mean_std"] = np.array(h.mean_group_std(st, W))
            out[f"{name}_mean_std_all"] = np.array(h.mean_group_std(st, W, full_only=False))
        out["reduction_hash"] = np.array(h.reduction_summary(per["none"], per["hash"], W))
        out["reduction_sort"] = np.array(h.reduction_summary(per["none"], per["sort"], W))
        out["csv_hash_head"] = np.array(h.group_stats_csv(per["hash"][:50], "hash"))
        np.savez_compressed(os.path.join(OUT, f"stats_{i}.npz"), **out)
    mtx = {}
    for i, text in enumerate(MTX):
        hd, t = h.parse_matrix_market(text)
        mtx[f"text_{i}"] = np.array(text)
        mtx[f"hdr_{i}"] = np.array([hd.object, hd.format, hd.field, hd.symmetry])
        mtx[f"shape_{i}"] = np.array([t.rows, t.cols], np.int64)
        mtx[f"row_{i}"], mtx[f"col_{i}"], mtx[f"val_{i}"] = t.row, t.col, t.val
        mtx[f"written_{i}"] = np.array(h.write_matrix_market(t))
        if hd.symmetry == "symmetric":
            e = h.expand_symmetric(t)
            mtx[f"sym_row_{i}"], mtx[f"sym_col_{i}"], mtx[f"sym_val_{i}"] = e.row, e.col, e.val
    np.savez_compressed(os.path.join(OUT, "mtx.npz"), **mtx)
    sort_counts(h)
    print("wrote", OUT)


def sort_counts(h):
    rng = np.random.default_rng(5)
    arrays = [np.array([3]), np.array([1, 0]), np.array([1, 1, 1]),
              np.array([5, 0, 3, 3, 9, 1, 0, 7]), np.zeros(512, np.int64),
              np.arange(100)[::-1].copy(), np.arange(64), rng.integers(0, 9, 17),
              rng.integers(0, 9, 100), rng.integers(0, 40, 512), rng.integers(0, 3, 1000),
              rng.zipf(1.8, 2048) % 5000, rng.integers(0, 1 << 20, 777)]
    out = {}
    for i, a in enumerate(arrays):
        ctr = h.OpCounter()
        out[f"keys_{i}"] = np.asarray(a, np.int64)
        out[f"perm_{i}"] = h.sort_permutation(a, counter=ctr)
        out[f"cmp_{i}"] = np.array(ctr.comparisons, np.int64)
    np.savez_compressed(os.path.join(OUT, "sortcmp.npz"), **out)


if __name__ == "__main__":
    main()
