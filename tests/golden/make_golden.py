"""Generate the golden vectors by running the REFERENCE package itself.

Runs only in the build container, where the reference is mounted read-only at
/root/reference (it does not exist on the GPU box; the .npz files this script
writes are committed and travel instead).  Usage:

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py

For every case it runs the reference's documented flow (pkg/README.md:34-39):
coo_to_csr -> make_grid -> sample_hash_params -> hash_permutations ->
build_hbp -> plan_execution -> run_spmv -> combine, and stores every
intermediate array in the reference's own dense layout.  fp32 cases round A
and x to float32 first and run the (fp64-only) reference on the rounded
values: that is the fp32 oracle.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cases")


def _ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
    sys.path.insert(0, REF)
    import hbp_spmv  # noqa: E402
    return hbp_spmv


def dense_trip(h, dense):
    dense = np.asarray(dense, np.float64)
    r, c = np.nonzero(dense)
    return h.TripletMatrix(dense.shape[0], dense.shape[1], r, c, dense[r, c])


def laplacian(h, n):
    """5-point Laplacian on an n x n grid: 4 on the diagonal, -1 off."""
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i, j = i.ravel(), j.ravel()
    rows, cols, vals = [i * n + j], [i * n + j], [np.full(n * n, 4.0)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ok = (i + di >= 0) & (i + di < n) & (j + dj >= 0) & (j + dj < n)
        rows.append((i * n + j)[ok])
        cols.append(((i + di) * n + (j + dj))[ok])
        vals.append(np.full(int(ok.sum()), -1.0))
    return h.TripletMatrix(n * n, n * n, np.concatenate(rows), np.concatenate(cols),
                           np.concatenate(vals)).canonicalized()


def cases(h):
    P = h.PartitionConfig
    G = lambda *a, **k: h.generate(h.SyntheticSpec(*a, **k))  # noqa: E731
    corpus = P(col_width=256, row_height=64, warp_size=8)
    # --- hand-computed known-answer matrices from the reference tests
    yield "kat_single_group", dense_trip(h, [[0, 0, 0, 0], [1, 0, 0, 0], [0, 2, 2.5, 0],
                                              [0, 0, 0, 3]]), P(4, 4, 4), "identity", 0
    d = np.zeros((4, 4))
    d[3, 0] = 1.0
    yield "kat_zero_row_lanes", dense_trip(h, d), P(4, 4, 4), "identity", 0
    yield "kat_strides_cross_group", dense_trip(h, [[1, 2, 0, 0], [3, 0, 0, 0], [0, 4, 5, 6],
                                                     [7, 0, 0, 0]]), P(4, 4, 2), "identity", 0
    yield "kat_eye8", dense_trip(h, np.eye(8)), P(4, 4, 2), "identity", 0
    d = np.zeros((8, 8))
    d[0, [0, 1, 2, 5]] = [1, 2, 3, 4]
    d[1, 3] = 5
    d[2, [0, 4, 6, 7]] = [6, 7, 8, 9]
    d[5, [1, 2, 3]] = [10, 11, 12]
    d[7, 7] = 13
    yield "kat_survey_8x8", dense_trip(h, d), P(4, 4, 2), "identity", 0
    yield "kat_grid_4x4", dense_trip(h, [[1, 0, 0, 2], [0, 0, 0, 0], [3, 4, 5, 0],
                                          [0, 0, 0, 6]]), P(2, 2, 2), "hash", 0
    # --- the acceptance corpus (test_acceptance.py:52-96): every size, seeds 0-3
    for pattern in ("uniform", "powerlaw"):
        for rows, cols in ((64, 64), (200, 333), (512, 512), (1000, 500), (333, 1000),
                           (2000, 2000)):
            for seed in range(4):
                yield (f"corpus_{pattern}_{rows}x{cols}_s{seed}",
                       G(rows, cols, pattern, 8.0, seed=seed), corpus, "hash", seed)
    eye = np.arange(64)
    yield "special_identity_64", h.TripletMatrix(64, 64, eye, eye, np.ones(64)), corpus, "hash", 0
    e = np.array([], np.int64)
    yield "special_zero_32x48", h.TripletMatrix(32, 48, e, e, np.array([])), corpus, "hash", 0
    yield "special_single_row_1x977", G(1, 977, "uniform", 60.0, seed=0), corpus, "hash", 0
    yield "special_single_col_771x1", G(771, 1, "uniform", 1.0, seed=0), corpus, "hash", 0
    yield "special_indivisible_130x70", G(130, 70, "powerlaw", 6.0, seed=1), P(48, 24, 8), "hash", 0
    yield "special_dense_rows_40x30", G(40, 30, "uniform", 30.0, seed=2), corpus, "hash", 0
    rng = np.random.default_rng(99)
    yield ("special_one_per_row_100x37",
           h.TripletMatrix(100, 37, np.arange(100), rng.integers(0, 37, 100),
                           rng.uniform(-1, 1, 100)).canonicalized(), corpus, "hash", 0)
    # --- odd geometries: sub-warp groups, W=1, non-power-of-two C and R
    yield "geo_w2_r8_c16", G(97, 61, "powerlaw", 5.0, seed=3), P(16, 8, 2), "hash", 3
    yield "geo_w4_r16_c64", G(300, 500, "powerlaw", 7.0, seed=4), P(64, 16, 4), "hash", 4
    yield "geo_w1_r4_c5", G(37, 23, "uniform", 3.0, seed=5), P(5, 4, 1), "hash", 5
    yield "geo_w8_r24_c10", G(130, 70, "uniform", 4.0, seed=6), P(10, 24, 8), "hash", 6
    yield "geo_w3_r9_c7", G(50, 40, "uniform", 4.0, seed=7), P(7, 9, 3), "hash", 7
    yield "geo_sort_w4_r16_c32", G(100, 100, "powerlaw", 5.0, seed=2), P(32, 16, 4), "sort", 2
    # --- the paper's default geometry (C=4096, R=512, W=32)
    dflt = P()
    yield "default_uniform_3000x5000", G(3000, 5000, "uniform", 8.0, seed=11), dflt, "hash", 11
    yield "default_powerlaw_4096", G(4096, 4096, "powerlaw", 16.0, seed=12), dflt, "hash", 12
    yield "default_laplace_64_c512", laplacian(h, 64), P(512, 512, 32), "hash", 0
    yield "default_uniform_8192_ccols", G(8192, 8192, "uniform", 8.0, seed=13), P(8192, 512, 32), "hash", 13
    yield "default_powerlaw_hot_ccols", G(2048, 8192, "powerlaw", 24.0, alpha=1.5, seed=14), \
        P(8192, 512, 32), "hash", 14
    # --- fp32 variants: A and x rounded to float32, reference run in fp64
    yield "fp32_uniform_2000", G(2000, 2000, "uniform", 8.0, seed=21), corpus, "hash", 21
    yield "fp32_powerlaw_hot_ccols", G(2048, 8192, "powerlaw", 24.0, alpha=1.5, seed=22), \
        P(8192, 512, 32), "hash", 22


def run_case(h, name, trip, cfg, ordering, seed):
    fp32 = name.startswith("fp32_")
    if fp32:
        trip = h.TripletMatrix(trip.rows, trip.cols, trip.row, trip.col,
                               trip.val.astype(np.float32).astype(np.float64))
    csr = h.coo_to_csr(trip)
    grid = h.make_grid(csr, cfg)
    params = h.sample_hash_params(grid, cfg, seed=seed)
    ctr = h.OpCounter()
    if ordering == "hash":
        perms = h.hash_permutations(grid, params, counter=ctr)
    elif ordering == "identity":
        perms = h.identity_permutations(grid)
    else:
        perms = h.sort_permutations(grid)
    hbp = h.build_hbp(csr, grid, perms)
    assert np.array_equal(csr.col_idx, trip.col) and np.array_equal(csr.values, trip.val)
    x = np.random.default_rng(1000 + seed).uniform(-1.0, 1.0, trip.cols)
    if fp32:
        x = x.astype(np.float32).astype(np.float64)
    workers = 3
    plan = h.plan_execution(hbp, cfg, workers)
    partial, log = h.run_spmv(hbp, x, plan, workers)
    y = h.combine(partial)
    sort_perms = h.sort_permutations(grid)
    y_csr = h.csr_spmv(csr, x)
    y_2d = h.block2d_spmv_baseline(csr, grid, x, workers=2)
    return dict(
        name=np.array(name), fp32=np.array(fp32), ordering=np.array(ordering),
        rows=np.array(trip.rows), cols=np.array(trip.cols),
        C=np.array(cfg.col_width), R=np.array(cfg.row_height), W=np.array(cfg.warp_size),
        fixed_fraction=np.array(cfg.fixed_fraction), seed=np.array(seed),
        trip_row=trip.row, trip_col=trip.col, trip_val=trip.val,
        row_ptr=csr.row_ptr,  # col_idx/values equal trip_col/trip_val (asserted)
        row_counts=grid.row_counts, row_starts=grid.row_starts,
        block_nnz=grid.block_nnz, block_elem_start=grid.block_elem_start,
        params=np.array([params.a, params.b, params.c, params.d]),
        probes=np.array(ctr.probes), perms=perms, sort_perms=sort_perms,
        col=hbp.col, data=hbp.data, add_sign=hbp.add_sign, zero_row=hbp.zero_row,
        group_start=hbp.group_start, output_hash=hbp.output_hash,
        block_order=plan.block_order, fixed_count=np.array(plan.fixed_count),
        worker_ranges=np.array(plan.worker_ranges, np.int64).reshape(-1, 2),
        workers=np.array(workers), x=x, partial=partial.values, y=y, y_csr=y_csr, y_2d=y_2d,
    )


def main():
    h = _ref()
    os.makedirs(OUT, exist_ok=True)
    total = 0
    only_new = "--only-new" in sys.argv  # keep committed fixtures byte-stable
    for name, trip, cfg, ordering, seed in cases(h):
        path = os.path.join(OUT, name + ".npz")
        if only_new and os.path.exists(path):
            continue
        arrays = run_case(h, name, trip, cfg, ordering, seed)
        np.savez_compressed(path, **arrays)
        total += os.path.getsize(path)
        print(f"{name}: nnz={trip.nnz} C={cfg.col_width} R={cfg.row_height} "
              f"W={cfg.warp_size} -> {os.path.getsize(path)} B")
    print(f"total {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
