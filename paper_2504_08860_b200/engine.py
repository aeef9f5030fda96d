"""Two-step SpMV execution on the GPU: scheduled block kernel, then combine.

Mirrors /root/reference/pkg/src/hbp_spmv/engine.py.  A worker is one
persistent GPU warp; the plan's fixed chunks and the atomic
ticket over the competitive pool are executed inside ``hbp_spmv_blocks``.
Each block writes a disjoint slice of the (compact) partial vector and every
row's sum is schedule-independent, so results are bitwise identical for any
worker count or fixed fraction (engine.py:1-8).

``SpmvOperator`` is the allocation-free hot path behind ``hbp_spmv``: it
owns the partial/ticket buffers and can capture SpMV + combine in a CUDA
graph.
"""
from __future__ import annotations

import ctypes
import os
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .hbp import HbpMatrix
from .partition import BlockGrid, PartitionConfig

__all__ = ["ExecutionPlan", "PartialVector", "ExecutionLog", "SpmvOperator", "plan_execution",
           "sumsq", "scale",
           "block_spmv", "run_spmv", "combine", "hbp_spmv", "KIND_FIXED", "KIND_COMPETITIVE"]

KIND_FIXED = 0
KIND_COMPETITIVE = 1


@dataclass(frozen=True)
class ExecutionPlan:
    """engine.py:38-56: nonzero blocks bc-major plus the fixed/competitive split."""

    block_order: np.ndarray
    fixed_count: int
    worker_ranges: tuple

    @property
    def competitive_start(self) -> int:
        return self.fixed_count

    @property
    def num_blocks(self) -> int:
        return len(self.block_order)

    @property
    def workers(self) -> int:
        return len(self.worker_ranges)


class PartialVector:
    """engine.py:59-68: per-(column block, row) partial sums.

    ``PartialVector(values, rows, num_col_blocks)`` is the reference's
    constructor: a caller-made dense [bc][global row] vector (numpy or a
    device tensor, float64), which block_spmv writes into and combine sums.
    The runtime path (run_spmv) makes ``PartialVector.from_compact(hbp, c)``:
    f64 [nzb * R] (block-major, original local row), with ``values`` /
    ``segment`` expanding to the dense layout on demand."""

    def __init__(self, values, rows: int, num_col_blocks: int):
        self.rows, self.num_col_blocks = int(rows), int(num_col_blocks)
        self.hbp = None
        self.compact = None
        self._dense = values

    @classmethod
    def from_compact(cls, hbp: HbpMatrix, compact: torch.Tensor) -> "PartialVector":
        pv = cls(None, hbp.rows, hbp.num_col_blocks)
        pv.hbp, pv.compact = hbp, compact
        return pv

    @property
    def values(self):
        if self._dense is None:
            d = torch.empty(self.num_col_blocks * self.rows, dtype=torch.float64,
                            device=self.compact.device)
            f = self.hbp.format_struct()
            L.call("hbp_expand_partial", ctypes.byref(f), L.P(self.compact), L.P(d), L.stream())
            self._dense = d
        return self._dense

    def segment(self, bc: int):
        return self.values[bc * self.rows:(bc + 1) * self.rows]


@dataclass
class ExecutionLog:
    """engine.py:71-83 (times from the GPU %globaltimer, ns)."""

    worker: np.ndarray
    kind: np.ndarray
    start_ns: np.ndarray
    end_ns: np.ndarray

    @classmethod
    def empty(cls, n: int) -> "ExecutionLog":
        return cls(np.full(n, -1, np.int32), np.full(n, -1, np.int8),
                   np.zeros(n, np.int64), np.zeros(n, np.int64))


def _block_order(source) -> np.ndarray:
    """engine.py:86-93: (br, bc) of nonzero blocks in bc-major order."""
    return np.ascontiguousarray(
        np.stack([source.blk_br.cpu().numpy(), source.blk_bc.cpu().numpy()], axis=1)
    ).astype(np.int32).reshape(-1, 2)


def default_workers(dtype=torch.float64, warp_size: int = 32) -> int:
    """Persistent warps that fill the device (all SMs x resident warps)."""
    return L.default_workers(dtype, warp_size)


def plan_execution(source, config: PartitionConfig, workers: int | None) -> ExecutionPlan:
    """engine.py:96-115.  source is a BlockGrid or an HbpMatrix; workers is the
    number of persistent GPU warps (None: fill the device)."""
    if workers is None:
        workers = default_workers(getattr(source, "dtype", torch.float64), config.warp_size)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if not isinstance(source, (BlockGrid, HbpMatrix)):
        raise TypeError("source must be a BlockGrid or an HbpMatrix")
    order = _block_order(source)
    n = len(order)
    fixed = int(config.fixed_fraction * n + 0.5)
    base, rem = divmod(fixed, workers)
    ranges, s = [], 0
    for w in range(workers):
        size = base + (1 if w < rem else 0)
        ranges.append((s, s + size))
        s += size
    return ExecutionPlan(order, fixed, tuple(ranges))


def _as_x(hbp: HbpMatrix, x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.as_tensor(np.asarray(x))
    if tuple(t.shape) != (hbp.cols,):
        raise ValueError(f"vector length {tuple(t.shape)} != cols {hbp.cols}")
    return t.to(device=hbp.data.device, dtype=hbp.data.dtype).contiguous()


class SpmvOperator:
    """Preallocated y = A x for one HbpMatrix (the bench / serving hot path).

    schedule="stream" (default when warp_size == 32): the element array is
    cut into equal slices, one per persistent warp, streamed through shared
    memory with TMA bulk copies (hbp_spmv_stream; exact reference order for
    f64, deterministic last-arriver combine of cut groups for f32).
    schedule="balanced": the same slices walked from global memory
    (hbp_spmv_balanced, step-aligned cuts).  schedule="plan": the reference's fixed + competitive
    block schedule (hbp_spmv_blocks) with this fixed_fraction.
    hub_min (f64, stream schedule): groups of more than hub_min elements --
    hub rows -- are cut across warps and summed in fast-mode order
    (deterministic, within ~1e-14 relative, not bitwise); every other row
    stays bitwise the reference.  0 / None: exact everywhere; "auto": twice
    the mean group length, at least 1024 (fp64 R-MAT 2^24: 1.54 ms vs 14.8
    exact everywhere; fp32 1.20).
    schedule="seg": one persistent CTA per worker runs whole nonzero blocks
    (its fixed chunk, then the atomic ticket), with the block's x-segment
    window staged in shared memory by TMA (hbp_spmv_seg).
    schedule="rowblock": one CTA per row block runs its nonzero blocks in
    ascending bc and folds them as the combine does (hbp_spmv_rowblock; one
    launch, no partial array -- for small matrices with several column blocks).
    direct mode (one column block): the kernel writes y itself; otherwise the
    partial (f64, compact) is combined in ascending bc."""

    ROWBLOCK_MAX_NNZ = 1 << 24  # auto: row-block owner below this size (f64) ...
    ROWBLOCK_MAX_NNZ_F32 = 1 << 28  # (f32: banded 138M nnz 0.32 vs 0.35 ms stream)
    ROWBLOCK_MAX_SKEW = 8.0     # ... when no row block holds > 8x the mean
    ROWBLOCK_MAX_BLOCKS = 4     # ... and row blocks average <= 4 nonzero blocks
    # auto: column-segment schedule for column-blocked matrices whose nonzero
    # blocks are large (cfg3: 16.9K elements per block, 2.18 vs 2.65 ms stream)
    SEG_MIN_BLOCK_NNZ = 4096
    SEG_MAX_WINDOW_BYTES = 64 << 10
    HOT_MIN_SHARE = 0.10  # stage hot columns when they hold >= 10 % of the nonzeros
    WARM_BYTES = 64 << 20  # warm tier: a 64 MB L2-resident copy of x at the next columns

    def __init__(self, hbp: HbpMatrix, workers: int | None = None,
                 fixed_fraction: float | None = None, schedule: str | None = None,
                 hot: bool | int | None = None, warm_bytes: int | None = None,
                 hub_min: int | str | None = None, ticket=None, slice_cost=None,
                 packed_x: bool | None = None, tail=None):
        self.hbp = hbp
        dev = hbp.data.device
        if schedule is None:
            schedule = os.environ.get("HBP_SCHEDULE") or self._auto_schedule(hbp, hot)
        if schedule in ("balanced", "stream", "seg") and hbp.config.warp_size != 32:
            raise ValueError(f"the {schedule} schedule needs warp_size == 32")
        self.schedule = schedule
        self.slice_cost = None
        self.tail = None
        if schedule == "stream":
            hbp.ensure_phases()
        # private descriptor: hot-column staging is a property of this operator
        f = self._fmt = L.FormatT.from_buffer_copy(hbp.format_struct())
        self.hot = None
        if schedule == "stream" and hot is not False and hbp.nnz and hbp.cols:
            n_hot = None if hot in (None, True) else int(hot)
            # x well inside L2 (cfg2: 64 MB of 126 MB) stays there with an
            # evict-last policy on every gather; a larger x (cfg5: 256 MB) gets
            # a warm tier, a compact evict-last copy of the next heaviest columns
            fits = hbp.cols * hbp.data.element_size() <= L.l2_bytes() * 0.6
            wb = (0 if fits else int(os.environ.get("HBP_WARM_BYTES", self.WARM_BYTES))) \
                if warm_bytes is None else int(warm_bytes)
            if packed_x is None:
                env = os.environ.get("HBP_PACKED_X")
                packed_x = (env == "1") if env is not None else (fits and wb == 0)
            cap = hbp.hot_capacity(warm=wb > 0 and hbp.cols <= (1 << 30), packed=bool(packed_x))
            n = min(cap if n_hot is None else min(n_hot, cap), hbp.cols) & ~3
            if hbp.cols >= (1 << 31):
                n = 0
            # packed x: the non-hot gathers read a compact copy of the USED
            # columns (cfg2: 29 MB instead of 64) when x fits the L2 budget;
            # past it the warm tier stays (cfg5 4.94 vs 5.23 ms packed; cfg2d,
            # f64: 1.52 vs 1.71 ms packed) -- DESIGN.md §4
            stage = n > 0 and (hot is not None or hbp.column_share(n) >= self.HOT_MIN_SHARE)
            if stage:
                if packed_x:
                    hc = hbp.hot_columns(n_hot, packed=True)
                else:
                    hc = hbp.hot_columns(n_hot, max(0, wb) // hbp.data.element_size())
                if hc.n_hot > 0:
                    self.hot = hc
                    hc.apply(f)
                f.cold_last = int(fits or hc.packed)
        if schedule in ("balanced", "stream"):
            if workers is None:
                w = L.c_i64(0)
                L.call(f"hbp_{schedule}_workers", ctypes.byref(f), ctypes.byref(w))
                workers = int(w.value)
            self.workers = max(1, workers)
            self.bal = L.BalancedT()
            self.bal.workers = self.workers
            self._scratch = []
            # f64 hub-row path (stream schedule): groups longer than hub_min
            # elements are split over warps and summed in fast-mode order
            if hub_min == "auto":  # groups longer than twice the mean (and >= 1024)
                ng = max(1, hbp.nzb * (hbp.config.row_height // 32))
                hub_min = max(1024, 2 * hbp.nnz // ng)
            self.hub_min = int(hub_min or 0) if (schedule == "stream" and f.exact) else 0
            if self.hub_min < 0:
                raise ValueError("hub_min must be >= 0")
            self.bal.hub_min = self.hub_min
            self.bal.warp_map = int(os.environ.get("HBP_WARP_MAP", "0"))
            # competitive pieces (stream schedule): (fixed fraction of the
            # elements as one static piece per warp, competitive pieces per
            # warp for the rest), e.g. "0.7:2"; off by default
            if ticket is None:
                ticket = os.environ.get("HBP_STREAM_TICKET") or None
            self.pieces = self.workers
            # tail pieces (stream schedule): "f:m" -- the first f of the cost as
            # one static slice per warp, the rest as m * workers pieces run by a
            # second, programmatically dependent launch whose CTAs fill the SMs
            # the first launch frees
            if tail is None:
                tail = os.environ.get("HBP_STREAM_TAIL") or None
            self.tail = None
            if tail and schedule == "stream" and hbp.nzb and not ticket:
                tf, tm = (tail.split(":") if isinstance(tail, str) else tail)
                tf, tm = float(tf), float(tm)
                if not (0.0 < tf <= 1.0 and tm > 0):
                    raise ValueError("tail needs a fixed fraction in (0, 1] and pieces > 0")
                self.tail = (tf, tm)
                self.pieces = self.workers + max(1, int(tm * self.workers + 0.5))
                self.bal.pieces = self.pieces
                self.bal.tail = 1
            if ticket and schedule == "stream" and hbp.nzb and not self.hub_min:
                ff, per = (ticket.split(":") if isinstance(ticket, str) else ticket)
                ff, per = float(ff), float(per)
                if not (0.0 <= ff <= 1.0 and per > 0):
                    raise ValueError("ticket needs a fixed fraction in [0, 1] and pieces > 0")
                self.pieces = self.workers + max(1, int(per * self.workers + 0.5))
                self.bal.pieces = self.pieces
                self.bal.fixed_elems = int(ff * hbp.nnz + 0.5)
                tk = torch.zeros(2, dtype=torch.int32, device=dev)
                self._ticket_buf = tk
                self.bal.ticket = tk.data_ptr()
            npc = self.pieces
            self.hub_groups, self.hub_share = 0, 0.0
            if self.hub_min:
                glen = hbp.group_start_c[1:] - hbp.group_start_c[:-1]
                big = glen > self.hub_min
                self.hub_groups = int(big.sum().item())
                self.hub_share = float(glen[big].sum().item()) / max(1, hbp.nnz)
            if not f.exact or self.hub_min:
                ph = torch.empty(npc * 32, dtype=torch.float64, device=dev)
                pt = torch.empty(npc * 32, dtype=torch.float64, device=dev)
                ce = torch.empty(self.workers, dtype=torch.int64, device=dev)
                cn = torch.zeros(max(1, hbp.nzb * (hbp.config.row_height // 32)),
                                 dtype=torch.int32, device=dev)
                self._scratch = [ph, pt, ce, cn]
                self.bal.part_head, self.bal.part_tail = ph.data_ptr(), pt.data_ptr()
                self.bal.cut_end, self.bal.counters = ce.data_ptr(), cn.data_ptr()
            if self.hot is not None:
                xh = torch.empty(self.hot.n_hot + self.hot.n_warm, dtype=hbp.dtype, device=dev)
                self._scratch.append(xh)
                self.bal.x_hot = xh.data_ptr()
            if schedule == "stream" and hbp.nzb:
                sl = torch.empty(npc + 1, dtype=torch.int64, device=dev)
                sg = torch.empty(npc, dtype=torch.int64, device=dev)
                self._scratch += [sl, sg]
                self.slice_lo_t = sl
                self.bal.slice_lo, self.bal.slice_g = sl.data_ptr(), sg.data_ptr()
                self.slice_cost = self._cost_weights(f, slice_cost)
                if self.slice_cost and (self.pieces == self.workers or self.tail):
                    ng = hbp.nzb * (hbp.config.row_height // 32)
                    cost = torch.empty(ng + 1, dtype=torch.int64, device=dev)
                    cost[ng] = 0
                    L.call("hbp_group_costs", ctypes.byref(f), *map(L.c_i64, self.slice_cost),
                           L.P(cost), L.stream())
                    cp = L.exclusive_sum(cost)
                    total = int(cp[-1].item())
                    if total // self.workers < (1 << 30):  # 32-bit slice offsets
                        self._scratch.append(cp)
                        self.bal.cost_prefix = cp.data_ptr()
                        if self.tail:  # the static part in cost units
                            self.bal.fixed_elems = int(self.tail[0] * total + 0.5)
                    else:
                        self.slice_cost = None
                if self.tail and not self.bal.cost_prefix:  # equal elements
                    self.bal.fixed_elems = int(self.tail[0] * hbp.nnz + 0.5)
                L.call("hbp_stream_slices", ctypes.byref(f), ctypes.byref(self.bal), L.stream())
        elif schedule == "seg":
            self.seg = self._seg_setup(hbp, f, workers)
            self.workers = int(self.seg.ctas)
        else:
            self.workers = workers or default_workers(hbp.dtype, hbp.config.warp_size)
        fr = hbp.config.fixed_fraction if fixed_fraction is None else fixed_fraction
        self.fixed_count = int(fr * hbp.nzb + 0.5)
        self.ticket = torch.zeros(2, dtype=torch.int32, device=dev)
        if schedule == "seg":
            self.seg.fixed_count = self.fixed_count
            self.seg.ticket = self.ticket.data_ptr()
        self.direct = hbp.num_col_blocks == 1
        R = hbp.config.row_height
        if schedule == "rowstage":
            self.rowstage_caps = self._rowstage_caps(hbp, f)
            if self.rowstage_caps is None:
                raise ValueError("the rowstage schedule needs warp_size == 32 and a row block "
                                 "whose staged elements fit one CTA's shared memory")
            self._rowstage_desc = hbp._ops["rowstage_desc"]
        self.partial = None if self.direct or schedule in ("rowblock", "rowstage") else torch.empty(hbp.nzb * R, dtype=torch.float64,
                                                            device=dev)
        self.has_empty_row_blocks = bool((hbp.rb_ptr[1:] == hbp.rb_ptr[:-1]).any())
        # stream schedule with several column blocks: optionally fuse the combine
        # into the SpMV kernel (last warp of each row block sums its partials).
        # Off by default: measured slower than the separate hbp_combine pass
        # (cfg3 3.56 vs 3.28 ms, cfg1 69 vs 61 us, same box)
        self.fused_combine = (not self.direct and schedule == "stream" and hbp.nzb > 0
                              and os.environ.get("HBP_FUSED_COMBINE", "0") == "1")
        if (not self.direct and schedule in ("stream", "seg") and not self.fused_combine
                and os.environ.get("HBP_DIRECT_SINGLE", "1") != "0"):
            f.reserved |= 4  # HBP_FLAG_DIRECT_SINGLE
        if self.fused_combine:
            rb = torch.zeros(max(1, hbp.num_row_blocks), dtype=torch.int32, device=dev)
            self._scratch.append(rb)
            self.bal.rb_done = rb.data_ptr()
        self.sched = L.ScheduleT()
        self.sched.workers = self.workers
        self.sched.fixed_count = self.fixed_count
        self.sched.ticket = self.ticket.data_ptr()
        self.launches_per_call = 1 if schedule in ("rowblock", "rowstage") else (1 + (1 if self.has_empty_row_blocks or not (
            self.direct or self.fused_combine) else 0) + (1 if self.hot is not None else 0))
        if self.tail:
            self.launches_per_call += 1  # the tail pieces' dependent launch
        self._graph = None
        self._gx = self._gy = None

    # Stream schedule, fast mode: warps get equal predicted COST, not equal
    # elements.  Per-group cost in element units = elements + 48 + 20 per phase
    # + 40 more per modular-pass phase: the per-warp model fitted to measured
    # warp times (tools/warp_cost.py; cfg2 R^2 0.97 on equal-element slices,
    # which ran 771..1181 us per warp on R-MAT -- short-row groups cost the
    # most).  A refit on its residual -- (49, 26, 33, 76) by phase kind and a
    # 17/64 discount per hot element -- narrowed the per-warp spread but not
    # the kernel time (cfg2 1.022 vs 1.024 ms, cfg5 +1 %): the end is set by
    # aggregate throughput once the gross imbalance is gone.
    SLICE_COST = (48, 20, 20, 60, 0)

    def _cost_weights(self, f, slice_cost):
        """(w_group, w_phase, w_modular) or None (equal elements).  Default:
        the fitted weights in fast mode and on the exact-mode hub-row path
        (cfg2d 1.519 -> 1.398 ms); plain exact mode keeps equal elements
        (its cuts round to group boundaries)."""
        if slice_cost is None:
            env = os.environ.get("HBP_SLICE_COST")
            if env is not None:
                slice_cost = env
            elif f.exact and not self.hub_min:
                return None
            else:
                return self.SLICE_COST
        if isinstance(slice_cost, str):
            slice_cost = None if slice_cost.strip() in ("", "0", "off") else \
                tuple(int(v) for v in slice_cost.split(","))
        if not slice_cost:
            return None
        w = tuple(int(v) for v in slice_cost)
        if len(w) == 3:  # (group, phase, modular extra): the first model's form
            w = (w[0], w[1], w[1], w[1] + w[2], 0)
        if len(w) != 5 or min(w) < 0 or w[4] > 64:
            raise ValueError("slice_cost needs 3 or 5 non-negative weights "
                             "(group, short, step, modular phase, hot/64)")
        return w

    ROWSTAGE_SMEM = 200 * 1024  # one CTA's staged elements + partials (+ x windows) at most
    ROWSTAGE_AUTO_SMEM = 64 * 1024  # auto choice only where >= 3 CTAs fit an SM (cfg1: 44 KB)
    ROWSTAGE_X_SMEM = 72 * 1024  # x windows staged only while the CTA stays this small

    @classmethod
    def _rowstage_caps(cls, hbp: HbpMatrix, f):
        """(ecap, kmax, xcap) of the TMA-staged row-block schedule
        (hbp_rowstage_plan over hbp_seg_windows' column windows), cached on
        the matrix; xcap = 0 (x gathered from global memory) when staging
        the windows would grow the CTA past ROWSTAGE_X_SMEM; None when
        W != 32 or a row block exceeds ROWSTAGE_SMEM."""
        if hbp.config.warp_size != 32:
            return None
        if "rowstage_caps" not in hbp._ops:
            dev = hbp.data.device
            lo = hi = None
            if hbp.nzb:
                lo = torch.empty(hbp.nzb, dtype=torch.int32, device=dev)
                hi = torch.empty(hbp.nzb, dtype=torch.int32, device=dev)
                cap = torch.zeros(1, dtype=torch.int64, device=dev)
                L.call("hbp_seg_windows", ctypes.byref(f), L.P(lo), L.P(hi), L.P(cap),
                       L.stream())
            caps = torch.zeros(3, dtype=torch.int64, device=dev)
            desc = torch.zeros(max(1, 4 * hbp.nzb), dtype=torch.int64, device=dev)
            L.call("hbp_rowstage_plan", ctypes.byref(f), L.P(lo) if lo is not None else None,
                   L.P(hi) if hi is not None else None, L.P(desc), L.P(caps), L.stream())
            ecap, kmax, xcap = (int(v) for v in caps.cpu())
            hbp._ops["rowstage_caps"] = (max(4, ecap), max(1, kmax), xcap)
            hbp._ops["rowstage_desc"] = desc
        ecap, kmax, xcap = hbp._ops["rowstage_caps"]
        esz = hbp.data.element_size()
        need = ecap * (4 + esz) + kmax * hbp.config.row_height * 8
        if kmax > 32 or need > cls.ROWSTAGE_SMEM:
            return None
        # x windows staged too: measured slower on cfg1 (27.4 vs 24.1 us: the
        # windows hold 2.5x the columns the walk reads and cost CTAs per SM),
        # so opt-in (HBP_ROWSTAGE_X=1)
        if os.environ.get("HBP_ROWSTAGE_X", "0") != "1" or need + xcap * esz > cls.ROWSTAGE_X_SMEM:
            xcap = 0
        return ecap, kmax, xcap

    def _seg_setup(self, hbp: HbpMatrix, f, workers) -> "L.SegT":
        """Column windows of the nonzero blocks (hbp_seg_windows, cached on
        the matrix) and the CTA count of the column-segment schedule."""
        dev = hbp.data.device
        if "seg_win" not in hbp._ops:
            lo = torch.empty(max(1, hbp.nzb), dtype=torch.int32, device=dev)
            hi = torch.empty(max(1, hbp.nzb), dtype=torch.int32, device=dev)
            cap = torch.zeros(1, dtype=torch.int64, device=dev)
            L.call("hbp_seg_windows", ctypes.byref(f), L.P(lo), L.P(hi), L.P(cap), L.stream())
            hbp._ops["seg_win"] = (lo, hi, int(cap.item()))
        lo, hi, cap = hbp._ops["seg_win"]
        sg = L.SegT()
        sg.win_lo, sg.win_hi, sg.win_cap = lo.data_ptr(), hi.data_ptr(), cap
        if workers is None:
            n = L.c_i64(0)
            L.call("hbp_seg_workers", ctypes.byref(f), L.c_i64(cap), ctypes.byref(n))
            workers = int(n.value)
        sg.ctas = max(1, int(workers))
        self._seg_keep = (lo, hi)
        return sg

    @classmethod
    def _auto_schedule(cls, hbp: HbpMatrix, hot=None) -> str:
        """stream for W = 32, plan otherwise; seg (x-segment staged per
        block, CTA per block) for column-blocked matrices with large nonzero
        blocks (>= 4096 elements on average) and x-segments of <= 64 KB;
        rowblock for small, evenly
        spread matrices with several column blocks and few nonzero blocks
        per row block (one launch instead of SpMV + combine; cfg1: 38.7 vs
        61 us) -- rowstage (its TMA-staged form) for f64 when a row block's
        elements fit one CTA (cfg1 28.7 us) -- unless hot staging was asked about (a stream-schedule
        feature).  With many small blocks per row block (uniform columns,
        C << cols) the stream schedule wins: 0.19 vs 0.30 ms at 4M nnz,
        64 blocks per row block (tools/prof_sched.py)."""
        R = hbp.config.row_height
        cap = cls.ROWBLOCK_MAX_NNZ_F32 if hbp.dtype == torch.float32 else cls.ROWBLOCK_MAX_NNZ
        if (hot is None and hbp.num_col_blocks > 1 and 0 < hbp.nnz <= cap
                and R <= 3072 and hbp.nzb <= cls.ROWBLOCK_MAX_BLOCKS * hbp.num_row_blocks):
            gpb = R // hbp.config.warp_size
            gs = hbp.group_start_c.view(-1)
            blk_nnz = gs[gpb::gpb] - gs[:-1:gpb]
            rb = torch.zeros(hbp.num_row_blocks, dtype=torch.int64, device=gs.device)
            rb.index_add_(0, hbp.blk_br.long(), blk_nnz)
            if float(rb.max()) <= cls.ROWBLOCK_MAX_SKEW * hbp.nnz / hbp.num_row_blocks:
                # f64 with W = 32: the TMA-staged form when a row block's
                # elements fit a CTA (cfg1 28.7 vs 36.9 us); f32 banded
                # matrices keep rowblock (0.101 vs 0.109 ms at 35M nnz)
                caps = (cls._rowstage_caps(hbp, L.FormatT.from_buffer_copy(hbp.format_struct()))
                        if hbp.dtype == torch.float64 else None)
                if caps is not None and (caps[0] * 12 + caps[1] * R * 8 <= cls.ROWSTAGE_AUTO_SMEM):
                    return "rowstage"
                return "rowblock"
        if (hbp.config.warp_size == 32 and hbp.num_col_blocks > 1 and hbp.nzb
                and hbp.nnz >= cls.SEG_MIN_BLOCK_NNZ * hbp.nzb
                and hbp.config.col_width * hbp.data.element_size() <= cls.SEG_MAX_WINDOW_BYTES):
            return "seg"
        return "stream" if hbp.config.warp_size == 32 else "plan"

    def _blocks(self, f, x, partial, y, s):
        if self.schedule == "seg":
            L.call("hbp_spmv_seg", ctypes.byref(f), ctypes.byref(self.seg), L.P(x), L.P(y),
                   L.P(partial), s)
        elif self.schedule in ("balanced", "stream"):
            L.call(f"hbp_spmv_{self.schedule}", ctypes.byref(f), ctypes.byref(self.bal), L.P(x), L.P(y),
                   L.P(partial), s)
        else:
            L.call("hbp_spmv_blocks", ctypes.byref(f), ctypes.byref(self.sched), L.P(x),
                   L.P(partial), L.P(y), s)

    def __call__(self, x: torch.Tensor, y: torch.Tensor | None = None,
                 x_sumsq: torch.Tensor | None = None,
                 y_peers: Sequence[int] = ()) -> torch.Tensor:
        """y = A x, or y = A (x / sqrt(x_sumsq[0])) when x_sumsq (a float64
        device scalar) is given -- the power-iteration step without a separate
        scaling pass (stream schedule, one column block).  y_peers: device
        addresses (e.g. other GPUs' buffers mapped by hbp_ipc_open) that get
        a copy of y from the same stores."""
        hbp = self.hbp
        self._check_vec(x, hbp.cols, "x")
        if y is None:
            y = torch.empty(hbp.rows, dtype=hbp.dtype, device=hbp.data.device)
        else:
            self._check_vec(y, hbp.rows, "y")
        f = self._fmt
        s = L.stream()
        if (x_sumsq is not None or y_peers) and (self.schedule != "stream" or not self.direct):
            raise ValueError("x_sumsq / y_peers need the stream schedule and one column block")
        if len(y_peers) > L.MAX_PEERS:
            raise ValueError(f"at most {L.MAX_PEERS} y_peers")
        if self.schedule == "stream":
            self.bal.y_sumsq = x_sumsq.data_ptr() if x_sumsq is not None else None
            self.bal.n_peers = len(y_peers)
            for i, a in enumerate(y_peers):
                self.bal.y_peer[i] = int(a)
        if self.schedule == "rowblock":
            L.call("hbp_spmv_rowblock", ctypes.byref(f), L.P(x), L.P(y), s)
            return y
        if self.schedule == "rowstage":
            ecap, kmax, xcap = self.rowstage_caps
            if x.data_ptr() % 16:
                xcap = 0  # the x windows' bulk copies need a 16-byte aligned x
            L.call("hbp_spmv_rowstage", ctypes.byref(f), L.P(self._rowstage_desc), L.P(x),
                   L.P(y), L.c_i64(ecap), L.c_i64(kmax), L.c_i64(xcap), s)
            return y
        if self.direct:
            self._blocks(f, x, None, y, s)
            if self.has_empty_row_blocks:
                for a in (y.data_ptr(), *y_peers):
                    L.call("hbp_zero_empty_rows", ctypes.byref(f), L.c_vp(a), s)
        elif self.fused_combine:
            self._blocks(f, x, self.partial, y, s)
            if self.has_empty_row_blocks:
                L.call("hbp_zero_empty_rows", ctypes.byref(f), L.P(y), s)
        else:
            # stream / seg schedule: single-block row blocks go straight to y
            self._blocks(f, x, self.partial, y if f.reserved & 4 else None, s)
            L.call("hbp_combine", ctypes.byref(f), L.P(self.partial), L.P(y), s)
        return y

    def _check_vec(self, v, n: int, name: str) -> None:
        """Device, dtype, contiguity and length of a caller vector (the
        kernels take raw pointers)."""
        d = self.hbp.data
        if not isinstance(v, torch.Tensor) or not v.is_cuda or v.device != d.device:
            raise ValueError(f"{name} must be a CUDA tensor on {d.device}")
        if v.dtype != d.dtype:
            raise ValueError(f"{name} dtype {v.dtype} != matrix dtype {d.dtype}")
        if not v.is_contiguous() or v.numel() != n:
            raise ValueError(f"{name} length {v.numel()} != {n} (or not contiguous)")

    def warp_clock(self) -> torch.Tensor:
        """Stream schedule diagnostics: from now on every launch records each
        persistent warp's %globaltimer at start and end into the returned
        int64 [workers, 2] tensor (load balance: the spread of the end times)."""
        if self.schedule != "stream":
            raise ValueError("warp_clock needs the stream schedule")
        t = torch.zeros(self.workers, 2, dtype=torch.int64, device=self.hbp.data.device)
        self._warp_ns = t
        self.bal.warp_ns = t.data_ptr()
        return t

    def capture(self, x: torch.Tensor, y: torch.Tensor) -> "torch.cuda.CUDAGraph":
        """Capture one SpMV (+combine) on fixed x / y buffers in a CUDA graph."""
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self(x, y)  # warm (library calls have no lazy init, but keep it symmetric)
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            self(x, y)
        self._graph, self._gx, self._gy = g, x, y
        return g


class HostPipeline:
    """End-to-end y_i = A x_i for a sequence of HOST vectors (pinned memory).

    Three streams: copy-in (H2D of x_i into device buffer i mod depth),
    compute (the SpMV, one SpmvOperator) and copy-out (D2H of y_i), ordered
    by events, so H2D(x_{i+1}), SpMV_i and D2H(y_{i-1}) run concurrently on
    the two copy engines and the SMs.  A buffer is rewritten only after the
    work that read it finished (SpMV_{i-depth} for x, D2H_{i-depth} for y)."""

    def __init__(self, hbp: HbpMatrix | None, depth: int = 2, operator=None,
                 x_len: int | None = None, chunks: int | None = None, **op_kwargs):
        """operator: any y = op(x, y) callable on device buffers (e.g. a
        StripedOperator) instead of a SpmvOperator of hbp; x_len its x
        length (default hbp.cols)."""
        src = hbp if hbp is not None else operator.hbp
        dev = src.data.device
        self.hbp = src
        self.depth = max(1, depth)
        self.s_in = torch.cuda.Stream(device=dev)
        self.s_comp = torch.cuda.Stream(device=dev)
        self.s_out = torch.cuda.Stream(device=dev)
        self.op = operator if operator is not None else SpmvOperator(hbp, **op_kwargs)
        nx = x_len if x_len is not None else src.cols
        self.xd = [torch.empty(nx, dtype=src.dtype, device=dev) for _ in range(self.depth)]
        # each copy as `chunks` consecutive pieces (the two directions interleave
        # at piece granularity instead of whole vectors)
        self.chunks = max(1, int(os.environ.get("HBP_PIPE_CHUNKS", "1")) if chunks is None
                          else int(chunks))
        self.yd = [torch.empty(src.rows, dtype=src.dtype, device=dev) for _ in range(self.depth)]

    @property
    def launches_per_call(self) -> int:
        return getattr(self.op, "launches_per_call", 1)

    def _pieces(self, n: int):
        k = min(self.chunks, max(1, n))
        step = -(-n // k)
        return [(a, min(n, a + step)) for a in range(0, n, step)]

    def run(self, xs_host, ys_host) -> None:
        """Enqueue every (x_i -> y_i); ordered after the current stream's work.
        The caller synchronizes (or waits on the current stream)."""
        cur = torch.cuda.current_stream()
        D = self.depth
        for s in (self.s_in, self.s_comp, self.s_out):
            s.wait_stream(cur)
        x_free = [None] * D   # event: SpMV that last read xd[j] finished
        y_free = [None] * D   # event: D2H that last read yd[j] finished
        for i, (xh, yh) in enumerate(zip(xs_host, ys_host)):
            j = i % D
            if x_free[j] is not None:
                self.s_in.wait_event(x_free[j])
            with torch.cuda.stream(self.s_in):
                for a, b in self._pieces(xh.numel()):
                    self.xd[j][a:b].copy_(xh[a:b], non_blocking=True)
            x_ready = torch.cuda.Event()
            x_ready.record(self.s_in)
            self.s_comp.wait_event(x_ready)
            if y_free[j] is not None:
                self.s_comp.wait_event(y_free[j])
            with torch.cuda.stream(self.s_comp):
                self.op(self.xd[j], self.yd[j])
            done = torch.cuda.Event()
            done.record(self.s_comp)
            x_free[j] = done
            self.s_out.wait_event(done)
            with torch.cuda.stream(self.s_out):
                for a, b in self._pieces(yh.numel()):
                    yh[a:b].copy_(self.yd[j][a:b], non_blocking=True)
            out = torch.cuda.Event()
            out.record(self.s_out)
            y_free[j] = out
        for s in (self.s_in, self.s_comp, self.s_out):
            cur.wait_stream(s)


def block_spmv(hbp: HbpMatrix, block, x, partial: PartialVector) -> None:
    """engine.py:123-134: run one block (the reference's lane-per-row chain
    walk, hbp_spmv_blocks with one worker) into the partial vector: entry
    bc*rows + br*R + output_hash[slot] of a dense PartialVector (numpy
    arrays are updated in place, like the reference), or the block's compact
    slice of a runtime one.  Every row of the block is written (+0.0 for
    empty rows, which a pre-zeroed partial holds already)."""
    br, bc = int(block[0]), int(block[1])
    keys = (hbp.blk_bc.to(torch.int64) * hbp.num_row_blocks + hbp.blk_br).cpu().numpy()
    k = bc * hbp.num_row_blocks + br
    i = int(np.searchsorted(keys, k))
    if i >= keys.size or keys[i] != k:
        return  # an empty block contributes nothing
    xd = _as_x(hbp, x)
    R, gpb = hbp.config.row_height, hbp.config.row_height // hbp.config.warp_size
    f = L.FormatT.from_buffer_copy(hbp.format_struct())
    esz4, esz8 = 4, 8
    f.nzb = 1
    f.blk_br = hbp.blk_br.data_ptr() + i * esz4
    f.blk_bc = hbp.blk_bc.data_ptr() + i * esz4
    f.slot_len = hbp.slot_len.data_ptr() + i * R * esz4
    f.perm = hbp.perm.data_ptr() + i * R * esz4
    f.group_start = hbp.group_start_c.data_ptr() + i * gpb * esz8
    sched = L.ScheduleT()
    sched.workers, sched.fixed_count = 1, 0
    ticket = torch.zeros(1, dtype=torch.int32, device=xd.device)
    sched.ticket = ticket.data_ptr()
    n = min(R, hbp.rows - br * R)
    if partial.compact is not None:
        if partial.hbp is not hbp:
            raise ValueError("partial belongs to another HbpMatrix")
        out = torch.empty(R, dtype=torch.float64, device=xd.device)
    else:
        if (partial.rows, partial.num_col_blocks) != (hbp.rows, hbp.num_col_blocks):
            raise ValueError("partial length disagrees with the matrix")
        out = torch.empty(R, dtype=torch.float64, device=xd.device)
    L.call("hbp_spmv_blocks", ctypes.byref(f), ctypes.byref(sched), L.P(xd), L.P(out),
           L.P(None), L.stream())
    if partial.compact is not None:
        partial.compact[i * R:i * R + n] = out[:n]
        partial._dense = None
        return
    base = bc * hbp.rows + br * R
    vals = partial.values
    if isinstance(vals, torch.Tensor):
        vals[base:base + n] = out[:n].to(device=vals.device, dtype=vals.dtype)
    else:
        vals[base:base + n] = out[:n].cpu().numpy()


def run_spmv(hbp: HbpMatrix, x, plan: ExecutionPlan, workers: int):
    """engine.py:179-193: every planned block once (GPU persistent warps);
    returns (PartialVector, ExecutionLog)."""
    if workers != plan.workers:
        raise ValueError("plan was built for a different worker count")
    xd = _as_x(hbp, x)
    dev = xd.device
    n = plan.num_blocks
    R = hbp.config.row_height
    compact = torch.zeros(hbp.nzb * R, dtype=torch.float64, device=dev)
    lw = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
    lk = torch.full((max(n, 1),), -1, dtype=torch.int8, device=dev)
    ls = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
    le = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
    ticket = torch.zeros(1, dtype=torch.int32, device=dev)
    sched = L.ScheduleT()
    sched.workers, sched.fixed_count = workers, plan.fixed_count
    sched.ticket = ticket.data_ptr()
    sched.log_worker, sched.log_kind = lw.data_ptr(), lk.data_ptr()
    sched.log_start_ns, sched.log_end_ns = ls.data_ptr(), le.data_ptr()
    f = hbp.format_struct()
    L.call("hbp_spmv_blocks", ctypes.byref(f), ctypes.byref(sched), L.P(xd), L.P(compact),
           L.P(None), L.stream())
    log = ExecutionLog(lw[:n].cpu().numpy(), lk[:n].cpu().numpy(), ls[:n].cpu().numpy(),
                       le[:n].cpu().numpy())
    return PartialVector.from_compact(hbp, compact), log


def combine(partial: PartialVector) -> torch.Tensor:
    """engine.py:196-201: sum partials over column blocks, ascending bc
    (f64 device tensor for a caller-made dense PartialVector, the matrix's
    dtype for a runtime one)."""
    if partial.compact is None:
        v = partial.values
        dev = L.require_cuda()
        vd = (v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v, np.float64)))
        vd = vd.to(device=dev, dtype=torch.float64).contiguous()
        if vd.numel() != partial.rows * partial.num_col_blocks:
            raise ValueError("partial length disagrees with rows * num_col_blocks")
        y = torch.empty(partial.rows, dtype=torch.float64, device=dev)
        L.call("hbp_combine_dense", L.P(vd), L.c_i64(partial.rows),
               L.c_i64(partial.num_col_blocks), L.P(y), L.stream())
        return y
    hbp = partial.hbp
    y = torch.empty(hbp.rows, dtype=hbp.dtype, device=partial.compact.device)
    f = hbp.format_struct()
    L.call("hbp_combine", ctypes.byref(f), L.P(partial.compact), L.P(y), L.stream())
    return y


def block2d_spmv_baseline(csr, grid: BlockGrid, x, workers: int = 1) -> torch.Tensor:
    """engine.py:204-225: plain 2D-partitioned SpMV (no reordering, no
    interleaving) through the same partial + combine machinery; a warp per
    nonzero block, a lane per row (hbp_block2d_spmv + hbp_combine).
    `workers` is accepted for signature parity (the GPU grid fills the device)."""
    from .hbp import row_block_lists
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if isinstance(x, torch.Tensor):
        xt = x
    else:
        xt = torch.as_tensor(np.asarray(x))
    if tuple(xt.shape) != (csr.cols,):
        raise ValueError(f"vector length {tuple(xt.shape)} != cols {csr.cols}")
    dev = csr.values.device
    xt = xt.to(device=dev, dtype=csr.values.dtype).contiguous()
    R = grid.config.row_height
    partial = torch.empty(max(1, grid.nzb * R), dtype=torch.float64, device=dev)
    L.call("hbp_block2d_spmv", L.P(grid.len_local), L.P(grid.start_local), L.P(grid.blk_br),
           L.c_i64(grid.nzb), L.c_i64(grid.rows), L.c_i64(R), L.P(csr.col_idx),
           L.P(csr.values), L.c_int(L.dtype_code(csr.values.dtype)), L.P(xt), L.P(partial),
           L.stream())
    key = "rb_lists"
    if key not in grid._cache:
        grid._cache[key] = row_block_lists(grid.blk_br, grid.num_row_blocks)
    rb_ptr, rb_blk = grid._cache[key]
    f = L.FormatT()
    f.rows, f.cols, f.col_width, f.row_height = grid.rows, grid.cols, grid.config.col_width, R
    f.warp_size, f.nrb, f.ncb, f.nzb = grid.config.warp_size, grid.num_row_blocks, \
        grid.num_col_blocks, grid.nzb
    f.dtype = L.dtype_code(csr.values.dtype)
    f.rb_ptr, f.rb_blk = rb_ptr.data_ptr(), (rb_blk.data_ptr() if rb_blk.numel() else 0)
    y = torch.empty(grid.rows, dtype=csr.values.dtype, device=dev)
    L.call("hbp_combine", ctypes.byref(f), L.P(partial), L.P(y), L.stream())
    return y


def hbp_spmv(hbp: HbpMatrix, x, workers: int = 1, *, gpu_workers: int | None = None
             ) -> torch.Tensor:
    """engine.py:228-232: plan, run and combine in one call (device tensor y).

    ``workers`` keeps the reference's signature, default and validation
    (plan_execution: ValueError for < 1).  The result does not depend on it
    (engine.py:1-8: bitwise identical for any worker count), so the GPU
    operator always fills the device; ``gpu_workers`` pins the number of
    persistent warps instead.  The operator (and its partial / ticket
    scratch) is cached per (gpu_workers, CUDA stream): calls on different
    streams never share scratch."""
    if int(workers) < 1:
        raise ValueError("workers must be >= 1")
    xd = _as_x(hbp, x)
    key = ("op", gpu_workers, torch.cuda.current_stream(xd.device).cuda_stream)
    op = hbp._ops.get(key)
    if op is None:
        op = SpmvOperator(hbp, gpu_workers)
        hbp._ops[key] = op
    return op(xd)


# ---- iterated SpMV helpers (config 5 power iteration; include/hbp.h hbp_sumsq / hbp_scale)
def sumsq(y: torch.Tensor, out: torch.Tensor, scratch: torch.Tensor | None = None) -> torch.Tensor:
    """out[0] = sum(y**2) in float64 on the device, deterministic."""
    n = L.c_i64(0)
    L.call("hbp_sumsq_scratch", ctypes.byref(n))
    if scratch is None or scratch.numel() < n.value:
        scratch = torch.empty(n.value, dtype=torch.float64, device=y.device)
    L.call("hbp_sumsq", L.P(y), L.c_int(L.dtype_code(y.dtype)), L.c_i64(y.numel()), L.P(scratch),
           L.P(out), L.stream())
    return out


def scale(y: torch.Tensor, sq: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out = y / sqrt(sq[0]) (sq read on the device; out may be y)."""
    L.call("hbp_scale", L.P(y), L.c_int(L.dtype_code(y.dtype)), L.c_i64(y.numel()), L.P(sq),
           L.P(out), L.stream())
    return out
