"""Load-balance analytics, the GFLOP/s formula and the timing harness.

Mirrors /root/reference/pkg/src/hbp_spmv/metrics.py:
``GroupStats`` (:26-50), ``group_stats`` (:53-75), ``mean_group_std``
(:82-90), ``reduction_summary`` (:93-107), ``group_stats_csv`` (:110-115),
``gflops`` (:118-122), ``Timing`` / ``time_kernel`` (:125-147) and
``BenchReport`` (:150-198).

``group_stats`` runs on the GPU (hbp_group_stats: one thread per lane group
of every nonzero block) and returns a ``GroupStatsTable`` -- a struct of
arrays in the reference's group order (bc, then br, then group) that
iterates, indexes and measures like the reference's ``list[GroupStats]``;
its mean / std_dev are bitwise equal to numpy's on the same lanes.
"""
from __future__ import annotations

import json
import statistics
import time
from dataclasses import dataclass, field
from typing import Iterator

import numpy as np
import torch

from . import _lib as L
from .partition import BlockGrid, PartitionConfig, groups_per_col_block

__all__ = ["GroupStats", "GroupStatsTable", "group_stats", "mean_group_std",
           "reduction_summary", "group_stats_csv", "gflops", "time_kernel", "Timing",
           "BenchReport"]


@dataclass(frozen=True)
class GroupStats:
    """Per-warp-group lane statistics of in-block row counts (metrics.py:26-50).

    utilization models lockstep lanes: W * max cycles of which sum(lane_nnz)
    do work; an all-zero group is vacuously fully utilized."""

    br: int
    bc: int
    group: int
    lane_nnz: np.ndarray
    mean: float
    std_dev: float
    max: int
    utilization: float

    @classmethod
    def from_lanes(cls, br: int, bc: int, group: int, lane_nnz: np.ndarray,
                   warp_size: int) -> "GroupStats":
        lane_nnz = np.asarray(lane_nnz)
        mx = int(lane_nnz.max()) if lane_nnz.size else 0
        util = float(lane_nnz.sum() / (warp_size * mx)) if mx > 0 else 1.0
        return cls(br, bc, group, lane_nnz, float(lane_nnz.mean()), float(lane_nnz.std()),
                   mx, util)


class GroupStatsTable:
    """Every lane group of a grid under one slot ordering, as host arrays
    (copied back from the device once): br, bc, group, lanes [G, W] with
    sizes [G], mean, std_dev, max, utilization."""

    def __init__(self, warp_size: int, br, bc, group, sizes, lanes, mean, std_dev, max_nnz,
                 utilization):
        self.warp_size = warp_size
        self.br, self.bc, self.group = br, bc, group
        self.sizes, self.lanes = sizes, lanes
        self.mean, self.std_dev, self.max, self.utilization = mean, std_dev, max_nnz, utilization

    def __len__(self) -> int:
        return int(self.br.size)

    def __getitem__(self, i: int) -> GroupStats:
        if i < 0:
            i += len(self)
        n = int(self.sizes[i])
        return GroupStats(int(self.br[i]), int(self.bc[i]), int(self.group[i]),
                          self.lanes[i, :n].astype(np.int64), float(self.mean[i]),
                          float(self.std_dev[i]), int(self.max[i]),
                          float(self.utilization[i]))

    def __iter__(self) -> Iterator[GroupStats]:
        for i in range(len(self)):
            yield self[i]

    def keys(self) -> np.ndarray:
        return np.stack([self.br, self.bc, self.group], 1)


def _compact_perm(grid: BlockGrid, permutations) -> torch.Tensor | None:
    """Compact slot -> local-row tables [nzb*R] (u32 bits in int32) or None."""
    if permutations is None:
        return None
    compact = getattr(permutations, "compact", None)
    if compact is not None:
        return compact
    dense = torch.as_tensor(np.asarray(permutations).astype(np.int64), device=grid.blk_br.device)
    R = grid.config.row_height
    s = torch.arange(R, device=dense.device)
    br = grid.blk_br.to(torch.int64)[:, None]
    src = grid.blk_bc.to(torch.int64)[:, None] * grid.rows + br * R + s[None, :]
    ok = (br * R + s[None, :]) < grid.rows
    out = torch.arange(R, device=dense.device).repeat(grid.nzb, 1)
    out[ok] = dense[src[ok]]
    return out.reshape(-1).to(torch.int32)


def group_stats(grid: BlockGrid, permutations=None,
                config: PartitionConfig | None = None) -> GroupStatsTable:
    """metrics.py:53-75: per-group lane statistics under a slot ordering
    (None = unordered), every block of every column block included."""
    if config is None:
        config = grid.config
    W, R = config.warp_size, config.row_height
    rows, nrb, ncb = grid.rows, grid.num_row_blocks, grid.num_col_blocks
    gpc = groups_per_col_block(rows, R, W)
    G = ncb * gpc
    dev = grid.blk_br.device
    lanes = torch.zeros(G * W, dtype=torch.int32, device=dev)
    mean = torch.zeros(G, dtype=torch.float64, device=dev)
    std = torch.zeros(G, dtype=torch.float64, device=dev)
    mx = torch.zeros(G, dtype=torch.int32, device=dev)
    util = torch.ones(G, dtype=torch.float64, device=dev)
    perm = _compact_perm(grid, permutations)
    L.call("hbp_group_stats", L.P(grid.blk_br), L.P(grid.blk_bc), L.c_i64(grid.nzb),
           L.P(grid.len_local), L.P(perm), L.c_i64(rows), L.c_i64(R), L.c_i64(W),
           L.c_i64(gpc), L.P(lanes), L.P(mean), L.P(std), L.P(mx), L.P(util), L.stream())
    # reference order: bc, br, group (== the flat group index g)
    gpb = R // W
    g = np.arange(G, dtype=np.int64)
    bc = g // gpc
    within = g - bc * gpc
    br = within // gpb
    grp = within - br * gpb
    last_rows = rows - (nrb - 1) * R
    n_block = np.where(br == nrb - 1, last_rows, R)
    sizes = np.minimum(W, n_block - grp * W)
    return GroupStatsTable(W, br, bc, grp, sizes, lanes.view(G, W).cpu().numpy(),
                           mean.cpu().numpy(), std.cpu().numpy(), mx.cpu().numpy(),
                           util.cpu().numpy())


def _arrays(stats) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(keys [G,3], sizes [G], std_dev [G]) of a table or a list of GroupStats."""
    if isinstance(stats, GroupStatsTable):
        return stats.keys(), stats.sizes, stats.std_dev
    stats = list(stats)
    keys = np.array([(s.br, s.bc, s.group) for s in stats], np.int64).reshape(-1, 3)
    sizes = np.array([s.lane_nnz.size for s in stats], np.int64)
    std = np.array([s.std_dev for s in stats], np.float64)
    return keys, sizes, std


def mean_group_std(stats, warp_size: int, full_only: bool = True) -> float:
    """metrics.py:82-90: mean per-group std, by default over full groups only."""
    _, sizes, std = _arrays(stats)
    pool = std[sizes == warp_size] if full_only else std
    if pool.size == 0:
        return 0.0
    return float(np.mean(pool))


def reduction_summary(stats_before, stats_after, warp_size: int) -> float:
    """metrics.py:93-107: 1 - mean(std after)/mean(std before) over full groups."""
    kb, _, _ = _arrays(stats_before)
    ka, _, _ = _arrays(stats_after)
    if kb.shape != ka.shape or not np.array_equal(kb, ka):
        raise ValueError("group coverage differs between orderings")
    before = mean_group_std(stats_before, warp_size)
    after = mean_group_std(stats_after, warp_size)
    if before == 0.0:
        return 0.0
    return 1.0 - after / before


def group_stats_csv(stats, ordering: str) -> str:
    """metrics.py:110-115."""
    lines = ["block_br,block_bc,group,ordering,mean,std_dev,utilization"]
    for s in stats:
        lines.append(f"{s.br},{s.bc},{s.group},{ordering},"
                     f"{s.mean:.6g},{s.std_dev:.6g},{s.utilization:.6g}")
    return "\n".join(lines) + "\n"


def gflops(nnz: int, seconds: float) -> float:
    """metrics.py:118-122: G = 2 * nnz / t."""
    if seconds <= 0:
        raise ValueError("seconds must be positive")
    return 2.0 * nnz / seconds / 1e9


@dataclass(frozen=True)
class Timing:
    median: float
    min: float
    max: float
    iterations: int


def time_kernel(fn, iterations: int = 20, warmup: int = 3, device: bool | None = None) -> Timing:
    """metrics.py:132-147: median time of fn() in seconds.  With a CUDA device
    (device=None -> auto) each sample is a pair of CUDA events on the current
    stream around fn(), so asynchronous kernels are timed on the device; on a
    host without CUDA, monotonic-clock samples as in the reference."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if device is None:
        device = torch.cuda.is_available()
    for _ in range(warmup):
        fn()
    samples: list[float] = []
    if device:
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(iterations)]
        for a, b in evs:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        samples = [a.elapsed_time(b) * 1e-3 for a, b in evs]
    else:
        for _ in range(iterations):
            t0 = time.perf_counter()
            fn()
            samples.append(time.perf_counter() - t0)
    return Timing(statistics.median(samples), min(samples), max(samples), iterations)


@dataclass
class BenchReport:
    """metrics.py:150-198: every kernel's gflops derives from its own median."""

    matrix: str
    rows: int
    cols: int
    nnz: int
    workers: int
    fixed_fraction: float
    config: dict = field(default_factory=dict)
    kernels: dict = field(default_factory=dict)
    preprocessing: dict = field(default_factory=dict)

    def add_kernel(self, name: str, timing: Timing, spmv_s: float | None = None,
                   combine_s: float | None = None) -> None:
        entry = {"time_s": timing.median, "min_s": timing.min, "max_s": timing.max,
                 "iterations": timing.iterations,
                 "gflops": gflops(self.nnz, timing.median) if self.nnz else 0.0}
        if spmv_s is not None:
            entry["spmv_s"] = spmv_s
        if combine_s is not None:
            entry["combine_s"] = combine_s
        self.kernels[name] = entry

    def to_dict(self) -> dict:
        return {"matrix": self.matrix, "rows": self.rows, "cols": self.cols, "nnz": self.nnz,
                "workers": self.workers, "fixed_fraction": self.fixed_fraction,
                "config": self.config, "kernels": self.kernels,
                "preprocessing": self.preprocessing}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2, sort_keys=True)
