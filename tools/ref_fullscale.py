"""The reference package itself (baseline/_ref, numba) at FULL benchmark scale
on the host (the full HBP convert plus SpMV for cfg1, and
at C=cols for cfg4 / H / cfg2; hbp_spmv at workers = cpu_count / 4 / 1;
csr_spmv on one thread).  One JSON line per config; run once on the GPU
box's host and commit the output under profiles/ (bench.py's default run
keeps to bounded samples).

    python tools/ref_fullscale.py cfg1 cfg4 H cfg2
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import bench_inputs as BI  # noqa: E402


def matrix(name):
    if name == "cfg1":
        rows, cols, rp, col, val = BI.laplacian_csr(1024)
        return rows, cols, rp, col, val, 4096
    if name in ("cfg4", "H"):
        from paper_2504_08860_b200.synth import SyntheticSpec, generate_arrays
        n = 8388608 if name == "cfg4" else 6250000
        r, c, val = generate_arrays(SyntheticSpec(n, n, "uniform", 16.0, seed=0))
        rp = np.concatenate(([0], np.cumsum(np.bincount(r, minlength=n)))).astype(np.int64)
        return n, n, rp, c, val.astype(np.float32).astype(np.float64), n
    if name == "cfg2":
        rows, cols, rp, col, val = BI.rmat_csr_numpy(24, 16, 0)
        return rows, cols, rp, col, val.astype(np.float32).astype(np.float64), cols
    raise SystemExit(f"unknown config {name}")


def timed(fn, n=3):
    fn()
    ts = []
    for _ in range(n):
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts)


def main():
    h = bench._reference_pkg()
    if h is None:
        raise SystemExit("baseline/_ref (the reference package) is not installed")
    for name in sys.argv[1:] or ["cfg1", "cfg4"]:
        t0 = time.perf_counter()
        rows, cols, rp, col, val, C = matrix(name)
        gen_s = time.perf_counter() - t0
        nnz = int(rp[-1])
        cfg = h.PartitionConfig(col_width=C, row_height=512, warp_size=32)
        csr = h.CsrMatrix(rows, cols, rp, col, val)
        st = {}
        a = time.perf_counter()
        grid = h.make_grid(csr, cfg)
        st["grid"] = time.perf_counter() - a
        a = time.perf_counter()
        params = h.sample_hash_params(grid, cfg)
        st["sample"] = time.perf_counter() - a
        a = time.perf_counter()
        perms = h.hash_permutations(grid, params)
        st["hash"] = time.perf_counter() - a
        a = time.perf_counter()
        hbp = h.build_hbp(csr, grid, perms, cfg)
        st["build"] = time.perf_counter() - a
        del grid, perms
        x = np.random.default_rng(0).uniform(-1.0, 1.0, cols)
        ncpu = os.cpu_count() or 1
        spmv = {}
        for wk in sorted({ncpu, 4, 1}, reverse=True):
            t = timed(lambda: h.hbp_spmv(hbp, x, workers=wk), n=3 if wk > 1 else 1)
            spmv[str(wk)] = {"ms": round(t * 1e3, 1), "gflops": round(2 * nnz / t / 1e9, 4)}
        t_csr = timed(lambda: h.csr_spmv(csr, x), n=1)
        out = {"config": name, "rows": rows, "cols": cols, "nnz": nnz, "col_width": C,
               "host_threads": ncpu, "cpu_model": bench._cpu_model(),
               "generate_s": round(gen_s, 1),
               "reference_preprocess_ms": {k: round(v * 1e3, 1) for k, v in st.items()},
               "reference_preprocess_total_ms": round(sum(st.values()) * 1e3, 1),
               "reference_hbp_spmv": spmv,
               "reference_csr_spmv_1thread": {"ms": round(t_csr * 1e3, 1),
                                               "gflops": round(2 * nnz / t_csr / 1e9, 4)},
               "what": "reference package (baseline/_ref, numba) at full scale on the host"}
        print(json.dumps(out), flush=True)
        del hbp, csr


if __name__ == "__main__":
    main()
