#!/usr/bin/env python
"""HBP SpMV benchmark on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg1|cfg3|cfg4|cfg5|H]
    python bench.py --impl reference ...      # the reference CPU path (oracle port)

A step is one y = A x (HBP kernel + combine when the grid has several column
blocks) over the configured matrix, inputs resident in HBM (`value`); cfg5's
step is one power-iteration step (SpMV, ||y|| all-reduce, y all-gather into
the next x).  `e2e` repeats the SpMV through the public API with x copied in
from pinned host memory and y copied back every step.  Timing: CUDA events
on the launching stream, barrier + synchronize on both sides, max over
ranks; when a rank's working set is below 2x L2 (cfg1) L2 is flushed between
timed steps (untimed), otherwise the inputs exceed L2 and x stays
cache-resident by design.
Multi-GPU (torchrun): every config but cfg1 is strong -- one global matrix
split into nnz-balanced row stripes (stripes.plan_stripes / StripedOperator),
x replicated; a single SpMV has no collective.  cfg5's power iteration
by default has the SpMV kernel store its y rows straight into every rank's
next x (CUDA IPC mappings over NVLink; `--collective fused`), leaving only
an 8-byte all-reduce; `--collective gather` all-gathers the y stripes with
NCCL instead (overlapped with the next step's own-column part).
cfg1 (5M nnz) runs an independent full instance per rank (weak).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HBP SpMV GFLOP/s and % HBM roofline at 1/2/4/8 B200; preprocess ms vs CPU"
UNIT = "GFLOP/s"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)

CONFIGS = {
    # name: (description, generator kwargs, dtype, col_width (None = cols))
    "cfg2": ("R-MAT scale 24 (16,777,216 rows), edge factor 16, Graph500 (0.57,0.19,0.19,0.05), "
             "random vertex relabel, duplicates removed, fp32, C=cols R=512 W=32",
             dict(kind="rmat", scale=24, edge_factor=16), "f32", None),
    "cfg2d": ("R-MAT scale 24 as cfg2 in fp64 (exact mode; hub rows split over warps with "
              "--hub auto), C=cols R=512 W=32",
              dict(kind="rmat", scale=24, edge_factor=16), "f64", None),
    "cfg4": ("the reference generator's SyntheticSpec(8388608, 8388608, 'uniform', 16.0, seed=0) "
             "(134,197,939 nnz), fp32, C=cols R=512 W=32",
             dict(kind="synth", rows=8388608, cols=8388608, mean=16.0), "f32", None),
    "H": ("the reference generator's SyntheticSpec(6250000, 6250000, 'uniform', 16.0, seed=0) "
          "(~100M nnz), fp32, C=cols R=512 W=32",
          dict(kind="synth", rows=6250000, cols=6250000, mean=16.0), "f32", None),
    "cfg1": ("5-point Laplacian 1024x1024 grid, fp64, C=4096 R=512 W=32",
             dict(kind="laplacian", n=1024), "f64", 4096),
    "cfg3": ("banded FEM-like 33,554,432 rows, 33 diagonals at even offsets -32..32 "
             "(nnz = 33n - 544), fp64, C=4096 R=512 W=32, row stripes over the ranks",
             dict(kind="banded", n=33554432), "f64", 4096),
    "cfg5": ("R-MAT scale 26 (67,108,864 rows), edge factor 16, fp32, C=cols R=512 W=32; "
             "power iteration x <- Ax/||Ax|| with y all-gather, row stripes over the ranks",
             dict(kind="rmat", scale=26, edge_factor=16), "f32", None),
}
# one global matrix, nnz-balanced row stripes over the ranks (stripes.py); cfg1
# (5M nnz, 38 us) runs an independent instance per rank instead
STRONG = {"cfg2", "cfg2d", "cfg3", "cfg4", "cfg5", "H"}
ITERATED = {"cfg5"}          # a step is one power-iteration step


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def gather_roofline(nnz: int, hot_share: float, warm_share: float, x_fits_l2: bool,
                    kernel_ms: float, sm_mhz, sms: int):
    """Random-column SpMV bound by the measured gather rates
    (profiles/gather_peaks.json, tools/gather_peaks.cu, tools/gather_mix.cu):
    every element's x gather through global memory costs one L1 line request
    -- ~0.93 per SM-cycle while x is L2-resident, ~0.24 beyond L2 -- and a
    hot-tier gather one shared-memory load (~4 per SM-cycle).  The two paths
    overlap (gather_mix: time follows the L2 share alone), so
    t_min = max(t_l1_miss_path, t_shared); frac = t_min / kernel time."""
    p = os.path.join(ROOT, "profiles", "gather_peaks.json")
    if not os.path.exists(p) or not sm_mhz:
        return None
    with open(p) as fh:
        g = json.load(fh)
    hz = float(sm_mhz) * 1e6 * sms
    r_l2 = g["ldg_l2_resident"]["per_sm_cycle"]
    r_far = g["ldg_beyond_l2"]["per_sm_cycle"]
    r_lds = g["lds_mix"]["per_sm_cycle_pure_lds"]
    cold = 1.0 - hot_share - warm_share
    t_miss = nnz * (warm_share / r_l2 + cold / (r_l2 if x_fits_l2 else r_far)) / hz
    t_lds = nnz * hot_share / r_lds / hz
    t = max(t_miss, t_lds)
    return {"bound": "l1_gather", "unit": "Ggathers/s", "achieved": round(nnz / (kernel_ms * 1e-3) / 1e9, 2),
            "peak": round(nnz / t / 1e9, 2), "frac": round(t * 1e3 / kernel_ms, 4),
            "min_ms": round(t * 1e3, 5), "sm_mhz": sm_mhz, "model": "max(l1_miss_path, shared)",
            "tiers": {"hot_lds": round(hot_share, 4), "warm_l2": round(warm_share, 4),
                      "cold": round(cold, 4), "cold_rate": "l2_resident" if x_fits_l2 else "beyond_l2"},
            "source": "profiles/gather_peaks.json (measured on B200: random 4-byte gathers per SM-cycle; "
                      "lds_mix: shared-memory gathers overlap the L1 miss path)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [s.strip() for s in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ inputs
def make_matrix_gpu(cfg_name: str, seed: int, device):
    import torch
    import bench_inputs as BI
    desc, gen, dt, C = CONFIGS[cfg_name]
    vdt = torch.float32 if dt == "f32" else torch.float64
    if gen["kind"] == "rmat":
        rows, cols, rp, col, val = BI.rmat_csr_torch(gen["scale"], gen["edge_factor"], seed,
                                                     device, vdt)
    elif gen["kind"] == "uniform":
        rows, cols, rp, col, val = BI.uniform_csr_torch(gen["rows"], gen["cols"], gen["mean"],
                                                        seed, device, vdt)
    elif gen["kind"] == "synth":
        rows, cols, rp, col, val = BI.synth_csr_torch(gen["rows"], gen["cols"], "uniform",
                                                      gen["mean"], seed, device, vdt)
    elif gen["kind"] == "banded":
        rows, cols, rp, col, val = BI.banded_csr_torch(gen["n"], device, vdt)
    else:
        rows, cols, rp, col, val = BI.laplacian_csr(gen["n"])
        rp = torch.as_tensor(rp, device=device)
        col = torch.as_tensor(col, device=device).to(torch.int32)
        val = torch.as_tensor(val, device=device).to(vdt)
    return desc, rows, cols, rp, col, val, (C or cols), vdt


def make_matrix_cpu_sample(cfg_name: str, seed: int):
    """A bounded sample of the same workload for the CPU reference path."""
    import bench_inputs as BI
    desc, gen, dt, C = CONFIGS[cfg_name]
    if gen["kind"] == "rmat":
        scale = int(os.environ.get("HBP_CPU_SCALE", "20"))
        rows, cols, rp, col, val = BI.rmat_csr_numpy(scale, gen["edge_factor"], seed)
        sample = f"R-MAT scale {scale} (same generator, edge factor, geometry C=cols)"
    elif gen["kind"] == "synth":
        from paper_2504_08860_b200.synth import SyntheticSpec, generate_arrays
        n = int(os.environ.get("HBP_CPU_ROWS", str(1 << 20)))
        r, c, val = generate_arrays(SyntheticSpec(n, n, "uniform", gen["mean"], seed=seed))
        rp = np.concatenate(([0], np.cumsum(np.bincount(r, minlength=n)))).astype(np.int64)
        rows = cols = n
        col = c
        sample = (f"the reference generator's SyntheticSpec({n}, {n}, 'uniform', {gen['mean']}, "
                  f"seed={seed}) (same generator at 1/{gen['rows'] // n} size, C=cols)")
    elif gen["kind"] == "uniform":
        n = int(os.environ.get("HBP_CPU_ROWS", str(1 << 20)))
        rng = np.random.default_rng(seed)
        counts = rng.poisson(gen["mean"], n)
        r = np.repeat(np.arange(n), counts)
        c = rng.integers(0, n, r.size)
        key = np.unique(r * n + c)
        r, c = key // n, key % n
        rp = np.concatenate(([0], np.cumsum(np.bincount(r, minlength=n)))).astype(np.int64)
        rows = cols = n
        col, val = c, rng.uniform(-1, 1, key.size)
        sample = f"uniform {n}^2 Poisson({gen['mean']}) rows (same generator family, C=cols)"
    elif gen["kind"] == "banded":
        n = int(os.environ.get("HBP_CPU_ROWS", str(1 << 20)))
        rows, cols, rp, col, val = BI.banded_csr(n)
        sample = f"banded {n} rows (same band structure, C=4096)"
    else:
        rows, cols, rp, col, val = BI.laplacian_csr(gen["n"])
        sample = "full matrix"
    if dt == "f32":
        val = val.astype(np.float32).astype(np.float64)
    return rows, cols, rp, col, val, (C or cols), sample


# ------------------------------------------------------- CPU reference arm
def cpu_reference(cfg_name: str, steps: int, warmup: int, seed: int = 0):
    """The reference's CPU HBP path (oracle port of _kernels.py / engine.py:
    fixed + ticket worker threads, dense partial zero-fill, combine) on a
    bounded sample, all host threads.  Returns a dict."""
    from oracle import oracle as O
    rows, cols, rp, col, val, C, sample = make_matrix_cpu_sample(cfg_name, seed)
    R, W = 512, 32
    t0 = time.perf_counter()
    grid = O.make_grid(rp, col, rows, cols, C, R, W)
    t1 = time.perf_counter()
    params = O.sample_hash_params(grid)
    t2 = time.perf_counter()
    perms, _ = O.hash_permutations(grid, params)
    t3 = time.perf_counter()
    h = O.build_hbp(rp, col, val, grid, perms)
    t4 = time.perf_counter()
    workers = os.cpu_count() or 1
    plan = O.plan_execution(grid.block_nnz, 0.7, workers)
    x = np.random.default_rng(0).uniform(-1.0, 1.0, cols)
    for _ in range(max(1, warmup)):
        part, _ = O.run_spmv(h, x, plan, workers)
        O.combine(part, rows, h.ncb)
    times = []
    deadline = time.perf_counter() + 30.0
    for i in range(max(1, steps)):
        a = time.perf_counter()
        part, _ = O.run_spmv(h, x, plan, workers)
        O.combine(part, rows, h.ncb)
        times.append(time.perf_counter() - a)
        if time.perf_counter() > deadline and i >= 2:
            break
    t = statistics.median(times)
    nnz = int(rp[-1])
    # the reference also at 1 and 4 workers (it regresses past 4
    # with Python threads; the C port's threads do not) -- informational
    by_workers = {}
    for wk in (1, 4):
        pl = O.plan_execution(grid.block_nnz, 0.7, wk)
        O.run_spmv(h, x, pl, wk)
        ts = []
        for _ in range(3):
            a = time.perf_counter()
            part, _ = O.run_spmv(h, x, pl, wk)
            O.combine(part, rows, h.ncb)
            ts.append(time.perf_counter() - a)
        by_workers[str(wk)] = round(2.0 * nnz / statistics.median(ts) / 1e9, 3)
    by_workers[str(workers)] = round(2.0 * nnz / t / 1e9, 3)
    return dict(value=2.0 * nnz / t / 1e9, unit=UNIT, cores=workers, kind="port",
                gflops_by_workers=by_workers,
                sample=f"{sample}: {rows} rows, {nnz} nnz, median of {len(times)} SpMV+combine",
                ms_per_step=t * 1e3, nnz=nnz, rows=rows,
                preprocess_ms=dict(grid=(t1 - t0) * 1e3, sample=(t2 - t1) * 1e3,
                                   hash=(t3 - t2) * 1e3, build=(t4 - t3) * 1e3,
                                   total=(t4 - t0) * 1e3))


def _reference_pkg():
    """The UNMODIFIED reference package (Python + numba), pip-installed into
    baseline/_ref (git-ignored, travels with the repo): its own public API
    and stock code path.  None when it is absent or numba is missing."""
    ref = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "hbp_spmv")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hbp_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import hbp_spmv as ref_pkg
        return ref_pkg
    except Exception:  # numba or numpy missing on this host
        return None


# the reference at FULL scale for these configs in `bench.py --impl reference`
# (its dense layout makes cfg3 / cfg5 infeasible on the host: bounded samples)
REF_FULL = {"cfg1", "cfg2", "cfg2d", "cfg4", "H"}


def make_matrix_full_host(cfg_name: str, seed: int = 0):
    """The benchmarked matrix itself on the host: generated on the GPU when
    one is visible (generation is not timed; numpy's R-MAT at scale 24 takes
    minutes), else with the host generators; values rounded to the config's
    dtype, as the GPU arm sees them."""
    import bench_inputs as BI
    desc, gen, dt, C = CONFIGS[cfg_name]
    try:
        import torch
        if torch.cuda.is_available():
            _, rows, cols, rp, col, val, C2, _ = make_matrix_gpu(cfg_name, seed,
                                                                 torch.device("cuda", 0))
            out = (rows, cols, rp.cpu().numpy().astype(np.int64),
                   col.cpu().numpy().astype(np.int64), val.double().cpu().numpy(), C2)
            del rp, col, val
            torch.cuda.empty_cache()
            return out + (f"the benchmarked matrix itself ({desc})",)
    except Exception:  # no usable GPU: host generators below
        pass
    if gen["kind"] == "rmat":
        rows, cols, rp, col, val = BI.rmat_csr_numpy(gen["scale"], gen["edge_factor"], seed)
    elif gen["kind"] == "laplacian":
        rows, cols, rp, col, val = BI.laplacian_csr(gen["n"])
    else:
        from paper_2504_08860_b200.synth import SyntheticSpec, generate_arrays
        r, c, val = generate_arrays(SyntheticSpec(gen["rows"], gen["cols"], "uniform",
                                                  gen["mean"], seed=seed))
        rows, cols = gen["rows"], gen["cols"]
        rp = np.concatenate(([0], np.cumsum(np.bincount(r, minlength=rows)))).astype(np.int64)
        col = c
    if dt == "f32":
        val = val.astype(np.float32).astype(np.float64)
    return rows, cols, rp, col, val, (C or cols), f"the benchmarked matrix itself ({desc})"


def numba_reference(cfg_name: str, steps: int, warmup: int, seed: int = 0, full: bool = False):
    """The reference itself (baseline/_ref: engine.py:228-232 hbp_spmv with
    numba kernels and Python worker threads, formats.py:266-273 csr_spmv) at
    workers = cpu_count / 4 / 1, on the same bounded sample as cpu_reference
    or (full, REF_FULL configs) on the benchmarked matrix itself.  Returns a
    dict, or None without the reference package."""
    h = _reference_pkg()
    if h is None:
        return None
    if full and cfg_name in REF_FULL:
        rows, cols, rp, col, val, C, sample = make_matrix_full_host(cfg_name, seed)
    else:
        rows, cols, rp, col, val, C, sample = make_matrix_cpu_sample(cfg_name, seed)
    cfg = h.PartitionConfig(col_width=C, row_height=512, warp_size=32)
    csr = h.CsrMatrix(rows, cols, rp, col, val)
    t0 = time.perf_counter()
    grid = h.make_grid(csr, cfg)
    t1 = time.perf_counter()
    params = h.sample_hash_params(grid, cfg)
    t2 = time.perf_counter()
    perms = h.hash_permutations(grid, params)
    t3 = time.perf_counter()
    hbp = h.build_hbp(csr, grid, perms, cfg)
    t4 = time.perf_counter()
    x = np.random.default_rng(0).uniform(-1.0, 1.0, cols)
    nnz = int(rp[-1])
    ncpu = os.cpu_count() or 1

    def timed(fn, n, budget=20.0):
        for _ in range(max(1, warmup)):
            fn()
        ts, deadline = [], time.perf_counter() + budget
        for i in range(max(1, n)):
            a = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - a)
            if time.perf_counter() > deadline and i >= 1:
                break
        return statistics.median(ts), len(ts)

    by_workers = {}
    t_main, n_main = timed(lambda: h.hbp_spmv(hbp, x, workers=ncpu), steps)
    by_workers[str(ncpu)] = round(2.0 * nnz / t_main / 1e9, 4)
    for wk in sorted({1, 4} - {ncpu}):
        tw, _ = timed(lambda: h.hbp_spmv(hbp, x, workers=wk), 3, budget=10.0)
        by_workers[str(wk)] = round(2.0 * nnz / tw / 1e9, 4)
    best = max(by_workers, key=lambda k: by_workers[k])
    t_csr, _ = timed(lambda: h.csr_spmv(csr, x), 3, budget=10.0)
    return dict(value=by_workers[best], unit=UNIT, cores=int(best), kind="reference",
                workers_best=int(best), gflops_by_workers=by_workers,
                csr_spmv_gflops_1thread=round(2.0 * nnz / t_csr / 1e9, 4),
                sample=(f"{sample}: {rows} rows, {nnz} nnz; the reference package itself "
                        f"(baseline/_ref, numba), hbp_spmv(workers={best}) = its best worker "
                        f"count, median of {n_main if best == str(ncpu) else 3}"),
                ms_per_step=2.0 * nnz / by_workers[best] / 1e6, nnz=nnz, rows=rows,
                preprocess_ms=dict(grid=(t1 - t0) * 1e3, sample=(t2 - t1) * 1e3,
                                   hash=(t3 - t2) * 1e3, build=(t4 - t3) * 1e3,
                                   total=(t4 - t0) * 1e3))


def format_bytes(op, hbp, esz: int) -> dict:
    """SURVEY §8(d) "format bytes": what this schedule must move per SpMV on
    top of the elements -- slot / group metadata, the phase stream, x
    staging copies and the partial round trip -- as an estimate next to the
    algorithmic bytes (x once, y once)."""
    R = hbp.config.row_height
    ngroups = hbp.nzb * (R // 32)
    slots = hbp.nzb * R
    elements = hbp.nnz * (4 + esz)
    if op.schedule == "stream":
        nph = int(hbp.phase_ptr[-1].item()) if hbp.phases is not None else 0
        meta = ngroups * 16 + slots * 4 + nph * 8  # group_start + phase_ptr, perm, phases
    else:
        meta = ngroups * 8 + slots * 8  # group_start, slot_len + perm
    staging = 0
    if getattr(op, "hot", None) is not None:
        n = op.hot.n_hot + op.hot.n_warm
        staging = n * (4 + 2 * esz)  # hot_cols + gathered x read + copy written
    partial = 0 if op.partial is None else op.partial.numel() * 8 * 2
    total = elements + meta + staging + partial + (hbp.cols + hbp.rows) * esz
    return {"elements": elements, "metadata": meta, "x_staging": staging,
            "partial_round_trip": partial, "total": total}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ GPU arm
def _dist():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        lr = int(os.environ.get("LOCAL_RANK", "0"))
        # HBP_DIST_BACKEND=gloo: a functional run of the multi-process path
        # when fewer GPUs than ranks are visible (ranks share devices round
        # robin; the numbers are then not a scaling measurement)
        backend = os.environ.get("HBP_DIST_BACKEND", "nccl")
        dev = lr % max(1, torch.cuda.device_count()) if backend == "gloo" else lr
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        return dist, dist.get_rank(), ws, dev
    torch.cuda.set_device(0)
    return None, 0, 1, 0


def _l2_bytes() -> int:
    import torch
    try:
        return int(torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size)
    except Exception:  # noqa: BLE001
        return 126 * 1024 * 1024


def run_gpu(args):
    import torch
    import paper_2504_08860_b200 as H

    from paper_2504_08860_b200.stripes import (PowerIteration, Stripe, StripedOperator,
                                               plan_stripes, row_block_nnz)
    dist, rank, world, local = _dist()
    dev = torch.device("cuda", local)
    strong = args.config in STRONG
    iterated = args.config in ITERATED
    R = 512
    # strong configs: every rank generates the same global matrix (seed 0) and
    # keeps its nnz-balanced row stripe (stripes.plan_stripes); weak configs
    # (cfg1): an independent full instance per rank
    desc, rows_g, cols, rp, col, val, C, vdt = make_matrix_gpu(args.config, 0 if strong else rank,
                                                              device=dev)
    torch.cuda.synchronize()
    nnz_global = int(rp[-1].item())
    if strong:
        stripes = plan_stripes(row_block_nnz(rp, rows_g, R), rows_g, R, world)
        me = rank
    else:
        stripes, me = [Stripe(0, 0, -(-rows_g // R), 0, rows_g)], 0
    if args.col_width:
        C = int(args.col_width)  # geometry experiment (SURVEY §8(d) fixes C only for cfg1-4)
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=32, fixed_fraction=0.7)
    hot_arg = {"auto": None, "off": False, "on": True}.get(args.hot)
    if hot_arg is None and args.hot != "auto":
        hot_arg = int(args.hot)
    if args.hub is None and args.config == "cfg2d":
        args.hub = "auto"  # the fp64 R-MAT line is quoted with the hub-row path
    hub_arg = None if args.hub in (None, "off", "0") else (
        "auto" if args.hub == "auto" else int(args.hub))
    op_kwargs = dict(schedule=args.schedule, hot=hot_arg, workers=args.workers, hub_min=hub_arg)
    # cfg5 at N > 1: "fused" = the SpMV kernel stores y into every rank's next x
    # (CUDA IPC over NVLink, stripes.PowerIteration(fused=True)), no all-gather;
    # "gather" = NCCL all-gather, overlapped with the own-column split
    fused = iterated and world > 1 and args.collective == "fused"
    split = iterated and world > 1 and not args.no_overlap and not fused

    # ---- preprocessing (timed like cli.py:150-158, GPU stages; the global
    # hash-parameter draw is part of "sample" at N > 1)
    pre = {}
    for rep in range(2):  # first pass warms allocator / module load; report the second
        tm = {}
        t0 = time.perf_counter()
        sop = StripedOperator(rows_g, cols, rp, col, val, stripes, me, cfg,
                              x_layout="padded" if iterated else "global", split_own=split,
                              op_kwargs=op_kwargs, distributed=strong and world > 1, timings=tm)
        torch.cuda.synchronize()
        tm["total"] = (time.perf_counter() - t0) * 1e3
        pre = tm
        if rep == 0:
            del sop
    del col, val
    stripe = sop.stripe
    rows = stripe.rows
    nnz = sop.nnz
    hbp, op, grid, csr, params = sop.hbp, sop.op, sop.grid, sop.csr, sop.params
    # the paper's reordering comparison (Fig. 6/7 analogues): GPU time of
    # the sort2D reorder beside the hash reorder, and the mean per-group std of lane
    # counts (load imbalance) under no / hash / sort2D ordering
    reorder = {"hash_ms": round(pre.get("hash", 0.0), 3)}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sperm = H.sort_permutations(grid)
    torch.cuda.synchronize()
    reorder["sort2d_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    gpc = -(-rows // R) * (R // 32)
    if grid.num_col_blocks * gpc * 32 <= (1 << 27):
        perms = H.hash_permutations(grid, params)
        reorder["mean_group_std"] = {
            name: round(H.mean_group_std(H.group_stats(grid, pm), 32), 4)
            for name, pm in (("none", None), ("hash", perms), ("sort2d", sperm))}
        del perms
    del sperm
    esz = 4 if vdt == torch.float32 else 8
    x_host = np.random.default_rng(0).uniform(-1.0, 1.0, cols)  # cli.py:170-171
    stream = torch.cuda.current_stream()

    # ---- the step
    if iterated:
        # power iteration x <- A x / ||A x||_2 (config 5, stripes.PowerIteration):
        # the stripe SpMV with the normalisation folded into its y stores, hbp_sumsq,
        # an 8-byte all-reduce and an in-place all-gather of the y stripes into the
        # next x (padded layout); at N > 1 the gather overlaps the next step's
        # own-column part
        collective = None
        if fused:
            try:
                pit = PowerIteration(sop, torch.as_tensor(x_host, device=dev), fused=True)
                collective = "fused-p2p-stores"
            except Exception as e:  # no IPC between these processes: NCCL all-gather
                print(f"fused power iteration unavailable ({e}); all-gather instead",
                      file=sys.stderr)
        if collective is None:
            pit = PowerIteration(sop, torch.as_tensor(x_host, device=dev))
            collective = ("nccl-all-gather" + ("+own-column-overlap" if split else "")
                          if world > 1 else None)
        step = pit.step
        x_res = pit.x_global
    else:
        x = torch.as_tensor(x_host, device=dev).to(vdt)
        y = torch.empty(rows, dtype=vdt, device=dev)

        def step():
            sop(x, y)

    # algorithmic bytes of one step on this rank
    b_alg = nnz * (esz + 4) + cols * esz + rows * esz
    flush = b_alg < 2 * _l2_bytes()
    scratch = torch.empty(2 * _l2_bytes() // 4, dtype=torch.float32, device=dev) if flush else None

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(K):
        if flush:
            scratch.fill_(float(i))  # evict the working set from L2 (untimed)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kernel_ms = statistics.mean(step_ms)
    per_step_ms = kernel_ms if flush else start.elapsed_time(end) / K

    # the SpMV kernel alone (roofline): time the stripe SpMV by itself on this rank
    if iterated:
        pit.finish()
        xk = pit.xs[pit.cur]
        yk = torch.empty(rows, dtype=vdt, device=dev)
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K)]
        for a, b in kev:
            if flush:
                scratch.fill_(0.0)
            a.record(stream)
            sop(xk, yk)
            b.record(stream)
        torch.cuda.synchronize()
        spmv_ms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    else:
        spmv_ms = kernel_ms

    # ---- end to end through the public API with host buffers (HostPipeline:
    # x_i H2D, SpMV, y_i D2H on 2 rotating streams; every step moves its own
    # x in and y out).  With an L2 flush, steps run one at a time instead.
    depth = 1 if flush else int(os.environ.get("HBP_PIPE_DEPTH", "3"))
    x_len = sop.width
    pipe = H.HostPipeline(None, depth=depth, operator=sop, x_len=x_len)
    if iterated:  # x in the stripes' padded layout
        xpad = torch.zeros(x_len, dtype=torch.float64)
        for st in stripes:
            xpad[st.rank * sop.pad:st.rank * sop.pad + st.rows] = torch.as_tensor(
                x_host[st.row_lo:st.row_hi])
        xh = xpad.to(vdt).pin_memory()
    else:
        xh = torch.as_tensor(x_host).to(vdt).pin_memory()
    yhs = [torch.empty(rows, dtype=vdt).pin_memory() for _ in range(depth)]
    nw = max(depth, args.warmup)
    pipe.run([xh] * nw, [yhs[i % depth] for i in range(nw)])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    if flush:
        e2e_samples = []
        for i in range(K):
            scratch.fill_(float(i))
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pipe.run([xh], [yhs[0]])
            b.record(stream)
            torch.cuda.synchronize()
            e2e_samples.append(a.elapsed_time(b))
        e2e_ms = statistics.mean(e2e_samples)
    else:
        # three back-to-back runs of K steps, median (host-side jitter in the
        # pinned copies otherwise moves a single run by ~10 %)
        runs = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pipe.run([xh] * K, [yhs[i % depth] for i in range(K)])
            e1.record(stream)
            torch.cuda.synchronize()
            runs.append(e0.elapsed_time(e1) / K)
        e2e_ms = statistics.median(runs)
    xd = xh.to(dev)  # x in the operator's layout (global, or the stripes' padded one)
    ychk = torch.empty(rows, dtype=vdt, device=dev)
    sop(xd, ychk)
    e2e_ok = bool(torch.equal(yhs[(K - 1) % depth], ychk.cpu()))

    # ---- correctness check (not timed): componentwise vs cuSPARSE fp64
    A = torch.sparse_csr_tensor(csr.row_ptr, csr.col_idx.to(torch.int64),
                                csr.values.to(torch.float64), (rows, sop.width))
    Aabs = torch.sparse_csr_tensor(csr.row_ptr, csr.col_idx.to(torch.int64),
                                   csr.values.to(torch.float64).abs(), (rows, sop.width))
    x64 = xd.to(torch.float64)
    yref = A @ x64
    scale = Aabs @ x64.abs()
    err = (ychk.to(torch.float64) - yref).abs()
    live = scale > 0
    check = float((err[live] / scale[live]).max().item()) if bool(live.any()) else 0.0
    zero_ok = bool((err[~live] == 0).all().item())
    del A, Aabs, yref, scale, err, live, x64

    # ---- the paper's comparison kernels on the same matrix and device (not
    # part of `value`): CSR Alg. 1 (thread per row), plain 2D blocks (warp per
    # block, no reordering) and cuSPARSE (torch CSR @ x) as a library anchor
    baselines = None
    if not args.no_baselines:
        def _time(fn, iters=5):
            fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(iters):
                if flush:
                    scratch.fill_(1.0)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return statistics.mean(ts)
        Acs = torch.sparse_csr_tensor(csr.row_ptr, csr.col_idx.to(torch.int64), csr.values,
                                      (rows, sop.width))
        bl = {"csr_alg1_ms": _time(lambda: H.csr_spmv(csr, xd)),
              "block2d_ms": _time(lambda: H.block2d_spmv_baseline(csr, grid, xd)),
              "cusparse_ms": _time(lambda: Acs @ xd)}
        del Acs
        baselines = {k: round(v, 4) for k, v in bl.items()}
        baselines["hbp_ms"] = round(spmv_ms, 4)
        for k, name in (("csr_alg1_ms", "csr"), ("block2d_ms", "2d"), ("cusparse_ms", "cusparse")):
            baselines[f"speedup_vs_{name}"] = round(bl[k] / spmv_ms, 3)

    # ---- aggregate over ranks (max time, sum of work)
    vals = torch.tensor([per_step_ms, spmv_ms, e2e_ms, float(nnz)], dtype=torch.float64,
                        device=dev)
    if dist:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        per_step_ms, spmv_ms_max, e2e_ms = mx[0].item(), mx[1].item(), mx[2].item()
        total_nnz = sm[3].item()
    else:
        spmv_ms_max = spmv_ms
        total_nnz = float(nnz)
    if iterated:
        res = x_res()
        if not bool(torch.isfinite(res).all().item()):
            raise RuntimeError("power iteration produced non-finite values")

    # collectives alone (N > 1, cfg5): the step's 8-byte all-reduce + y all-gather,
    # device-timed on this rank, max over ranks
    comm_ms = None
    if dist and iterated:
        nxt = pit.xs[1 - pit.cur]
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        dist.barrier()
        c0.record(stream)
        for _ in range(K):
            dist.all_reduce(pit.sq)
            if not pit.fused:  # fused: the y exchange is inside the SpMV's stores
                dist.all_gather_into_tensor(nxt, nxt[rank * sop.pad:(rank + 1) * sop.pad])
        c1.record(stream)
        torch.cuda.synchronize()
        cm = torch.tensor([c0.elapsed_time(c1) / K], dtype=torch.float64, device=dev)
        dist.all_reduce(cm, op=dist.ReduceOp.MAX)
        comm_ms = round(float(cm.item()), 5)
    stripe_nnz = row_block_nnz(rp, rows_g, R) if strong else None
    stripe_info = ([{"rank": st.rank, "rows": [st.row_lo, st.row_hi],
                     "nnz": int(stripe_nnz[st.rb_lo:st.rb_hi].sum())} for st in stripes]
                   if strong else None)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None

    gflops = 2.0 * total_nnz / (per_step_ms * 1e-3) / 1e9
    peak, peak_src = _peaks()
    achieved = b_alg / (spmv_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get(args.config, {}).get("dram_bytes_per_launch")
    fmt_bytes = format_bytes(op, hbp, esz)
    launches_step = sop.launches_per_call + (2 if iterated else 0)  # + sumsq (2 launches)
    groof = None
    if hbp.num_col_blocks == 1:  # random columns over all of x: gather-bound, not HBM-bound
        groof = gather_roofline(
            nnz, op.hot.share if op.hot is not None else 0.0,
            op.hot.warm_share if op.hot is not None else 0.0,
            cols * esz <= 0.6 * _l2_bytes(), spmv_ms, clk.get("sm_mhz"),
            torch.cuda.get_device_properties(dev).multi_processor_count)
    out = {
        "metric": METRIC, "value": round(gflops, 3), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(per_step_ms, 5),
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "f32" if vdt == torch.float32 else "f64",
        "data": "synthetic (generated on device, seed = " + ("0" if strong else "rank") + ")",
        "config": {"workload": f"{args.config}: {desc}", "rows": rows_g if strong else rows,
                   "cols": cols, "nnz": nnz_global if strong else nnz,
                   "rows_per_rank": rows, "nnz_rank0": nnz,
                   "nonzero_blocks": hbp.nzb, "col_width": C, "row_height": R,
                   "warp_size": 32, "fixed_fraction": 0.7, "workers": op.workers,
                   "schedule": op.schedule,
                   "slice_cost": (list(op.slice_cost) if getattr(op, "slice_cost", None)
                                  else None),
                   "hub_min": getattr(op, "hub_min", 0),
                   "hub_groups": getattr(op, "hub_groups", 0),
                   "hub_element_share": round(getattr(op, "hub_share", 0.0), 4),
                   "hot_columns": op.hot.n_hot if op.hot is not None else 0,
                   "hot_share": round(op.hot.share, 4) if op.hot is not None else 0.0,
                   "warm_columns": op.hot.n_warm if op.hot is not None else 0,
                   "warm_share": round(op.hot.warm_share, 4) if op.hot is not None else 0.0,
                   "hash_params": [params.a, params.b, params.c, params.d],
                   "step": (("power iteration: SpMV storing y into every rank's next x "
                             "(CUDA IPC) + ||y|| all-reduce" if pit.fused else
                             "power iteration: SpMV + ||y|| all-reduce + y all-gather")
                            if iterated else "SpMV (+ combine when ncb > 1)"),
                   "parallelism": (f"row stripes x{world} of one matrix (strong)" if strong
                                   else f"independent instances x{world} (weak)"),
                   "stripes": stripe_info,
                   "own_column_split": sop.split,
                   "collective": collective if iterated else None,
                   "own_column_share_rank0": round(sop.own_share, 4),
                   "comm_ms_per_step": comm_ms,
                   "l2": ("working set < 2x L2: L2 flushed between timed steps" if flush
                          else "inputs larger than L2 (no flush); x reused from L2 by design")},
        "roofline": {"bound": "hbm", "binding": "l1_gather" if groof else "hbm",
                     "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes": b_alg, "format_bytes": fmt_bytes,
                     "peak_source": peak_src,
                     "kernel_ms": round(spmv_ms, 5),
                     "kernel": f"k_spmv_{op.schedule}" + (" (+ hot-column gather)" if op.hot is not None else "")
                     + ("" if op.launches_per_call == 1 + (op.hot is not None) else " (+ combine/zero launch)")},
        "gather_roofline": groof,
        "e2e": {"value": round(2.0 * total_nnz / (e2e_ms * 1e-3) / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": x_len * esz, "d2h_bytes_per_step": rows * esz,
                "ms_per_step": round(e2e_ms, 4),
                "how": ("HostPipeline (copy-in / compute / copy-out streams): pinned x H2D, SpMV, y D2H per step"
                        + (" (one step at a time, L2 flushed)" if flush
                           else f", {depth} buffers in flight"))},
        "gpu_launches": K * launches_step,
        "clocks": clk,
        "preprocess_ms": {k: round(v, 3) for k, v in pre.items()},
        "reorder": reorder,
        "check": {"max_componentwise_err_vs_cusparse_f64": check, "zero_rows_exact": zero_ok,
                  "e2e_y_equals_device_y": e2e_ok},
    }
    if baselines is not None:
        out["baselines_same_gpu"] = baselines
    if world == 1 and not args.no_cpu_baseline:
        # the reference package itself when baseline/_ref holds it (numba),
        # else (and alongside, for comparison) the oracle's C port
        port = cpu_reference(args.config, steps=5, warmup=1)
        nb = numba_reference(args.config, steps=3, warmup=1) \
            if args.config != "cfg1" or os.environ.get("HBP_REF_CFG1") else None
        cb = nb if nb is not None else port
        out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                   "gflops_by_workers")}
        out["cpu_baseline"]["preprocess_ms"] = {k: round(v, 1)
                                                for k, v in cb["preprocess_ms"].items()}
        out["cpu_baseline"]["cpu_model"] = _cpu_model()
        out["cpu_baseline"]["host_threads"] = os.cpu_count()
        if nb is not None:
            out["cpu_baseline"]["csr_spmv_gflops_1thread"] = nb["csr_spmv_gflops_1thread"]
            out["cpu_baseline"]["port"] = {k: port[k] for k in ("value", "cores",
                                                                "gflops_by_workers")}
        # SURVEY.md §8(d) gate: GPU preprocess vs one CPU reference SpMV of the
        # same sample, and the CPU preprocess on its sample
        out["preprocess_gate"] = {
            "gpu_preprocess_ms": round(pre["total"], 3),
            "cpu_reference_spmv_ms_on_sample": round(cb["ms_per_step"], 3),
            "cpu_reference_spmv_ms_scaled_to_workload": round(
                cb["ms_per_step"] * (nnz_global if strong else nnz) / cb["nnz"], 1),
            "cpu_reference_preprocess_ms_on_sample": round(cb["preprocess_ms"]["total"], 1),
            # linear in nnz (the reference's grid / hash / build passes are)
            "cpu_reference_preprocess_ms_scaled_to_workload": round(
                cb["preprocess_ms"]["total"] * (nnz_global if strong else nnz) / cb["nnz"], 1),
            "speedup_vs_cpu_reference_preprocess": round(
                cb["preprocess_ms"]["total"] * (nnz_global if strong else nnz) / cb["nnz"]
                / pre["total"], 1),
            "gpu_preprocess_in_gpu_spmvs": round(pre["total"] / per_step_ms, 2),
            "gpu_preprocess_faster_than_one_cpu_spmv":
                pre["total"] < cb["ms_per_step"] * (nnz_global if strong else nnz) / cb["nnz"]}
    if dist:
        dist.destroy_process_group()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    # the reference package on the benchmarked matrix itself where its dense
    # layout fits the host (REF_FULL; HBP_REF_SAMPLE=1: the bounded sample)
    full = os.environ.get("HBP_REF_SAMPLE", "0") != "1"
    nb = numba_reference(args.config, steps=args.steps, warmup=args.warmup, full=full)
    port = cpu_reference(args.config, steps=args.steps, warmup=args.warmup)
    cb = nb if nb is not None else port
    desc = CONFIGS[args.config][0]
    others = {"port": {"value": round(port["value"], 4), "cores": port["cores"],
                       "gflops_by_workers": port["gflops_by_workers"],
                       "what": "oracle/ C port of the same path (pthreads)"}}
    if nb is not None:
        others["reference_numba"] = {k: nb[k] for k in ("gflops_by_workers",
                                                         "csr_spmv_gflops_1thread")}
    return {
        "impl": "reference", "metric": METRIC, "value": round(cb["value"], 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(cb["ms_per_step"], 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (bounded CPU sample of the same workload)",
        "config": {"workload": f"{args.config}: {desc}", "sample": cb["sample"],
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": round(cb["value"], 4), "unit": UNIT, "cores": cb["cores"],
                         "kind": cb["kind"], "sample": cb["sample"]},
        "e2e": {"value": round(cb["value"], 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "preprocess_ms": {k: round(v, 1) for k, v in cb["preprocess_ms"].items()},
        "cpu_model": _cpu_model(), "host_threads": os.cpu_count(),
        "cpu_arms": others,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-baselines", action="store_true",
                    help="skip the CSR / 2D / cuSPARSE comparison timings")
    ap.add_argument("--schedule", default=None, choices=[None, "stream", "balanced", "plan", "rowblock", "rowstage", "seg"])
    ap.add_argument("--col-width", type=int, default=None,
                    help="override the config's column-block width C (geometry experiments)")
    ap.add_argument("--workers", type=int, default=None,
                    help="persistent warps of the SpMV (default: one per resident warp slot)")
    ap.add_argument("--collective", default="fused", choices=["fused", "gather"],
                    help="cfg5 at N > 1: y stored into the peers' x by the SpMV kernel "
                         "(CUDA IPC), or an NCCL all-gather")
    ap.add_argument("--no-overlap", action="store_true",
                    help="cfg5 at N > 1: no own-column split, all-gather then SpMV")
    ap.add_argument("--hub", default=None,
                    help="f64 hub-row path: off (exact everywhere), auto, or a group-length threshold")
    ap.add_argument("--hot", default="auto",
                    help="hot-column x staging: auto (>= 10%% of nnz), on, off, or a column count")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    out = run_reference(args) if args.impl == "reference" else run_gpu(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
