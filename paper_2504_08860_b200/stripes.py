"""Row-stripe sharding of the HBP path over several GPUs.

Every block's permutation and layout depend only on its own rows and the
global hash constants (a, c), so whole row blocks are independent: a rank
that owns rows [row_lo, row_hi) (multiples of row_height) builds exactly the
blocks the single-GPU build would, once (a, c) are global.  x is replicated;
each rank writes its slice of y; a single SpMV needs no collective.  The
iterated SpMV (power iteration, config 5) all-reduces ||y||^2 (8 bytes) and
all-gathers the y slices into the next x.

Compute is injected (callables) so the orchestration is testable with the
gloo backend on CPU; the default callables use the GPU path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from .reorder import BUCKET_MAX, HashParams

__all__ = ["Stripe", "plan_stripes", "sample_hash_params_global", "gather_rows",
           "power_iteration", "row_block_nnz", "padded_columns", "StripedOperator",
           "PowerIteration"]


@dataclass(frozen=True)
class Stripe:
    rank: int
    rb_lo: int   # first row block
    rb_hi: int   # one past the last row block
    row_lo: int
    row_hi: int

    @property
    def rows(self) -> int:
        return self.row_hi - self.row_lo


def plan_stripes(row_block_nnz: Sequence[int], rows: int, row_height: int,
                 world: int) -> list[Stripe]:
    """Contiguous row-block ranges with balanced nnz: stripe r ends at the
    first row block where the nnz prefix reaches (r+1)/world of the total
    (every stripe non-empty while there are enough row blocks)."""
    w = np.asarray(row_block_nnz, dtype=np.int64)
    nrb = w.size
    if world < 1:
        raise ValueError("world must be >= 1")
    pref = np.concatenate(([0], np.cumsum(w)))
    total = int(pref[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        c = int(np.searchsorted(pref, target, side="left"))
        if c > 0 and abs(pref[c - 1] - target) <= abs(pref[min(c, nrb)] - target):
            c -= 1  # the nearer prefix
        c = max(c, cuts[-1] + (1 if cuts[-1] < nrb else 0))
        cuts.append(min(c, nrb))
    cuts.append(nrb)
    out = []
    for r in range(world):
        lo, hi = cuts[r], max(cuts[r], cuts[r + 1])
        out.append(Stripe(r, lo, hi, min(lo * row_height, rows), min(hi * row_height, rows)))
    return out


def _params_from_sample(sample: np.ndarray, row_height: int, quantile: float) -> HashParams:
    """reorder.py:87-103 on the gathered sample (same numpy calls)."""
    b = max(1, row_height // (BUCKET_MAX + 1))
    a = 0
    if sample.size:
        while np.quantile(sample >> a, quantile, method="inverted_cdf") > BUCKET_MAX:
            a += 1
        modal = int(np.bincount(np.minimum(sample >> a, BUCKET_MAX),
                                minlength=BUCKET_MAX + 1).max())
    else:
        modal = 0
    c = max(1, -(-modal // b))
    while math.gcd(c, b) != 1:
        c += 1
    return HashParams(a=a, b=b, c=c, d=b)


def sample_hash_params_global(counts_fn: Callable[[np.ndarray], np.ndarray], stripe: Stripe,
                              rows: int, num_col_blocks: int, row_height: int, group=None,
                              sample_size: int = 4096, seed: int = 0, quantile: float = 0.9,
                              device=None) -> HashParams:
    """sample_hash_params (reorder.py:69-103) over the GLOBAL grid when the
    rows are spread over ranks: rank 0 draws the flat indices with the
    reference's numpy call, every rank answers the indices whose row it owns
    (counts_fn(local_flat_indices) -> counts), a SUM all-reduce assembles the
    sample, and every rank derives the same (a, c)."""
    import torch.distributed as dist
    pop = num_col_blocks * rows
    if sample_size < pop:
        flat = np.random.default_rng(seed).choice(pop, sample_size, replace=False)
    else:
        flat = np.arange(pop, dtype=np.int64)
    flat = np.asarray(flat, dtype=np.int64)
    if group is not None or (dist.is_available() and dist.is_initialized()):
        t = torch.as_tensor(flat, device=device)
        dist.broadcast(t, src=0, group=group)
        flat = t.cpu().numpy()
    bc, r = np.divmod(flat, rows)
    mine = (r >= stripe.row_lo) & (r < stripe.row_hi)
    counts = np.zeros(flat.size, dtype=np.int64)
    if mine.any():
        local = bc[mine] * stripe.rows + (r[mine] - stripe.row_lo)
        counts[mine] = np.asarray(counts_fn(local), dtype=np.int64)
    if group is not None or (dist.is_available() and dist.is_initialized()):
        t = torch.as_tensor(counts, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        counts = t.cpu().numpy()
    return _params_from_sample(counts, row_height, quantile)


def gather_rows(y_local: torch.Tensor, stripes: Sequence[Stripe], group=None) -> torch.Tensor:
    """All-gather of the y slices (padded to the largest stripe) into the
    full vector, in row order."""
    import torch.distributed as dist
    world = len(stripes)
    m = max(s.rows for s in stripes)
    buf = torch.zeros(m, dtype=y_local.dtype, device=y_local.device)
    buf[:y_local.numel()] = y_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[s.rank][:s.rows] for s in stripes])


def power_iteration(spmv_local: Callable[[torch.Tensor], torch.Tensor], x0: torch.Tensor,
                    stripes: Sequence[Stripe], iters: int, group=None) -> torch.Tensor:
    """x <- A x / ||A x||_2 (config 5): per iteration one all-reduce of
    ||y_local||^2 and one all-gather of the y slices (the only collectives)."""
    import torch.distributed as dist
    x = x0
    for _ in range(iters):
        y = spmv_local(x)
        sq = (y.to(torch.float64) ** 2).sum().reshape(1)
        dist.all_reduce(sq, op=dist.ReduceOp.SUM, group=group)
        y = y / torch.sqrt(sq).to(y.dtype)
        x = gather_rows(y, stripes, group)
    return x


# ------------------------------------------------------------- GPU striping
def row_block_nnz(row_ptr: torch.Tensor, rows: int, row_height: int) -> np.ndarray:
    """nnz per row block from a CSR row_ptr (the weights of plan_stripes)."""
    nrb = -(-rows // row_height)
    idx = torch.clamp(torch.arange(nrb + 1, device=row_ptr.device) * row_height, max=rows)
    return torch.diff(row_ptr[idx]).cpu().numpy()


def padded_columns(col_idx: torch.Tensor, stripes: Sequence[Stripe], pad: int) -> torch.Tensor:
    """Global column c of a square matrix whose x is distributed like y ->
    its slot in the all-gather buffer [world * pad]: owner * pad + (c -
    row_lo(owner)).  Monotone in c, so every row keeps its column order (and
    the HBP layout its element order)."""
    lo = torch.tensor([st.row_lo for st in stripes], dtype=torch.int64, device=col_idx.device)
    c = col_idx.to(torch.int64)
    owner = torch.searchsorted(lo, c, right=True) - 1
    return (owner * pad + (c - lo[owner])).to(torch.int32)


class StripedOperator:
    """This rank's row stripe of a global CSR matrix as HBP SpMV operators
    (SURVEY.md §8e): rows [row_lo, row_hi) of whole row blocks, hash
    parameters from the global sample (sample_hash_params_global), so every
    block's permutation and layout equal the single-GPU build's.

    x_layout="global": x is the full global vector (a single SpMV, x
    replicated).  x_layout="padded": x lives in the all-gather buffer
    [world * pad] (padded_columns), the iterated SpMV's layout; with
    split_own the stripe is built as two operators, the columns this rank
    owns (usable before the all-gather lands) and the rest.

    Compute is the CUDA path (build_hbp, SpmvOperator); the collectives are
    torch.distributed (NCCL on B200; gloo works for tests)."""

    def __init__(self, rows: int, cols: int, row_ptr: torch.Tensor, col_idx: torch.Tensor,
                 values: torch.Tensor, stripes: Sequence[Stripe], rank: int, config,
                 x_layout: str = "global", split_own: bool = False, group=None,
                 op_kwargs: dict | None = None, seed: int = 0,
                 distributed: bool | None = None, timings: dict | None = None):
        from .formats import CsrMatrix
        from .hbp import build_hbp
        from .partition import PartitionConfig, make_grid
        from .reorder import _grid_counts_at, hash_permutations
        from .engine import SpmvOperator
        import torch.distributed as dist

        if x_layout not in ("global", "padded"):
            raise ValueError("x_layout must be 'global' or 'padded'")
        if x_layout == "padded" and rows != cols:
            raise ValueError("the padded (iterated) layout needs a square matrix")
        self.stripes, self.rank, self.world = list(stripes), rank, len(stripes)
        self.stripe = st = self.stripes[rank]
        self.pad = max(x.rows for x in self.stripes)
        self.rows_global, self.cols_global = rows, cols
        self.x_layout = x_layout
        self.dtype = values.dtype
        dev = values.device
        e0, e1 = int(row_ptr[st.row_lo].item()), int(row_ptr[st.row_hi].item())
        rp = (row_ptr[st.row_lo:st.row_hi + 1] - e0).contiguous()
        ci = col_idx[e0:e1]
        vals = values[e0:e1].contiguous()
        if x_layout == "padded":
            ci = padded_columns(ci, self.stripes, self.pad)
            width = self.world * self.pad
        else:
            ci = ci.contiguous()
            width = cols
        # C = cols configs keep one column block over the (padded) width
        C = width if config.col_width >= cols else config.col_width
        cfg = PartitionConfig(col_width=C, row_height=config.row_height,
                              warp_size=config.warp_size, fixed_fraction=config.fixed_fraction)
        self.config = cfg
        self.width = width
        self.nnz = e1 - e0
        import time

        def mark(name):
            # stage times (cli.py:150-158 analogue) when asked for: synchronised
            if timings is not None:
                torch.cuda.synchronize(dev)
                now = time.perf_counter()
                timings[name] = (now - mark.t) * 1e3
                mark.t = now
        if timings is not None:
            torch.cuda.synchronize(dev)
        mark.t = time.perf_counter()
        csr = CsrMatrix(st.rows, width, rp, ci, vals)
        grid = make_grid(csr, cfg)
        mark("grid")
        ncb = -(-width // C)
        if distributed is None:
            distributed = self.world > 1
        if distributed:
            self.params = sample_hash_params_global(lambda flat: _grid_counts_at(grid, flat), st,
                                                    rows, ncb, cfg.row_height, group=group,
                                                    seed=seed, device=dev if dev.type == "cuda"
                                                    and dist.get_backend(group) == "nccl" else None)
        else:
            from .reorder import sample_hash_params
            self.params = sample_hash_params(grid, cfg, seed=seed)
        mark("sample")
        kw = dict(op_kwargs or {})
        own_lo, own_hi = rank * self.pad, rank * self.pad + st.rows
        self.split = bool(split_own and x_layout == "padded" and self.world > 1)
        self.csr, self.grid = csr, grid

        def build(csr_part, g=None):
            g = make_grid(csr_part, cfg) if g is None else g
            perms = hash_permutations(g, self.params)
            mark("hash")
            h = build_hbp(csr_part, g, perms, with_add_sign=False, with_zero_row=False)
            mark("build")
            o = SpmvOperator(h, **kw)
            mark("operator")
            return h, o

        if self.split:
            # entries of own columns vs the rest, each as its own CSR stripe
            own = (ci >= own_lo) & (ci < own_hi)
            row_of = torch.repeat_interleave(torch.arange(st.rows, device=dev), torch.diff(rp))
            parts = []
            for m in (own, ~own):
                cnt = torch.zeros(st.rows, dtype=torch.int64, device=dev)
                cnt.index_add_(0, row_of[m], torch.ones_like(row_of[m]))
                rpm = torch.zeros(st.rows + 1, dtype=torch.int64, device=dev)
                rpm[1:] = torch.cumsum(cnt, 0)
                parts.append(CsrMatrix(st.rows, width, rpm, ci[m].contiguous(),
                                       vals[m].contiguous()))
            del row_of, own
            (self.hbp_own, self.op_own), (self.hbp, self.op) = build(parts[0]), build(parts[1])
            self.y_own = torch.empty(st.rows, dtype=self.dtype, device=dev)
        else:
            self.hbp, self.op = build(csr, grid)
            self.hbp_own = self.op_own = None
        self.own_share = (self.hbp_own.nnz / max(1, self.nnz)) if self.split else 0.0

    @property
    def ops(self):
        return [o for o in (self.op_own, self.op) if o is not None]

    @property
    def launches_per_call(self) -> int:
        return sum(o.launches_per_call for o in self.ops) + (1 if self.split else 0)

    def __call__(self, x: torch.Tensor, y: torch.Tensor, x_sumsq: torch.Tensor | None = None,
                 before_remote=None, y_peers=()) -> torch.Tensor:
        """y (this stripe's rows) = A_stripe x.  With the own-column split,
        before_remote() (e.g. waiting for the all-gather) runs between the
        own-column part and the rest.  y_peers: addresses that receive a copy
        of y from the kernel's own stores (unsplit operator only)."""
        if y_peers and self.split:
            raise ValueError("y_peers needs an operator without the own-column split")
        if self.split:
            self.op_own(x, self.y_own, x_sumsq=x_sumsq)
            if before_remote is not None:
                before_remote()
            self.op(x, y, x_sumsq=x_sumsq)
            from . import _lib as L
            L.call("hbp_add", L.P(y), L.P(self.y_own), L.c_int(L.dtype_code(self.dtype)),
                   L.c_i64(y.numel()), L.stream())
            return y
        if before_remote is not None:
            before_remote()
        return self.op(x, y, x_sumsq=x_sumsq, y_peers=y_peers)


class PowerIteration:
    """Config 5 over row stripes: x <- A x / ||A x||_2.  A step is the
    stripe SpMV (normalisation folded into its y stores), hbp_sumsq, an
    8-byte all-reduce of ||y||^2 and an in-place all-gather of the y
    stripes straight into the next x buffer (padded layout, no copy).  With
    overlap, the gather runs asynchronously and the next step's own-column
    part (StripedOperator split_own) computes while it is in flight.

    fused=True (SURVEY §8(e)'s fused variant): there is no all-gather.  The
    ranks map each other's two x buffers once (CUDA IPC, handles exchanged
    through torch.distributed), and the SpMV kernel stores every y row into
    its own next-x buffer AND into every peer's at the same offset, over
    NVLink, as the rows finish -- the transfer overlaps the SpMV row by row.
    The 8-byte all-reduce that follows orders the steps: a rank's next SpMV
    starts after every rank's current one has finished (and fenced its peer
    stores), so x is complete, and no rank writes a peer's x while the peer
    still reads it (the two buffers alternate)."""

    def __init__(self, op: StripedOperator, x0: torch.Tensor, group=None, overlap: bool = True,
                 fused: bool = False):
        import torch.distributed as dist
        from . import engine as E
        if op.x_layout != "padded":
            raise ValueError("PowerIteration needs a padded-layout StripedOperator")
        if fused and op.split:
            raise ValueError("the fused power iteration needs an operator without split_own")
        self.op, self.group = op, group
        self.dist = dist if op.world > 1 else None
        self.fused = bool(fused and op.world > 1)
        self.overlap = overlap and op.world > 1 and not self.fused
        dev = x0.device
        n = op.world * op.pad
        self.xs = [torch.zeros(n, dtype=op.dtype, device=dev) for _ in range(2)]
        for st in op.stripes:
            self.xs[0][st.rank * op.pad:st.rank * op.pad + st.rows] = x0[st.row_lo:st.row_hi].to(
                op.dtype)
        self.sq = torch.ones(1, dtype=torch.float64, device=dev)
        n_scr = E.L.c_i64(0)
        E.L.call("hbp_sumsq_scratch", E.ctypes.byref(n_scr))
        self.scratch = torch.empty(n_scr.value, dtype=torch.float64, device=dev)
        self.cur = 0
        self.pending = None
        self._sumsq = E.sumsq
        self._mapped = []            # (base address) of every peer mapping opened here
        self.peer_x = [[], []]       # peer_x[k]: the other ranks' xs[k] addresses
        if self.fused:
            self._map_peers()
        self.sync_host = self.dist is not None and dist.get_backend(group) != "nccl"

    def _map_peers(self) -> None:
        from . import _lib as L
        import ctypes
        mine = []
        for buf in self.xs:
            h = (ctypes.c_char * L.IPC_HANDLE_BYTES)()
            off = L.c_i64(0)
            L.call("hbp_ipc_export", L.P(buf), h, ctypes.byref(off))
            mine.append((bytes(h), off.value))
        allh = [None] * self.op.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        for p in range(self.op.world):
            if p == self.op.rank:
                continue
            for k in range(2):
                hb, off = allh[p][k]
                ptr = L.c_vp()
                L.call("hbp_ipc_open", ctypes.create_string_buffer(hb, len(hb)), L.c_i64(off),
                       ctypes.byref(ptr))
                self._mapped.append(ptr.value - off)
                self.peer_x[k].append(ptr.value)

    def close(self) -> None:
        """Unmap the peers' buffers (fused); the object is unusable after."""
        from . import _lib as L
        self.finish()
        if self._mapped:
            torch.cuda.synchronize()
            for base in self._mapped:
                L.call("hbp_ipc_close", L.c_vp(base))
            self._mapped = []
            self.peer_x = [[], []]

    def _own(self, buf: torch.Tensor) -> torch.Tensor:
        o = self.op
        return buf[o.rank * o.pad:(o.rank + 1) * o.pad]

    def step(self) -> None:
        o = self.op
        x, nxt = self.xs[self.cur], self.xs[1 - self.cur]
        y = self._own(nxt)[:o.stripe.rows]
        if self.fused:
            off = o.rank * o.pad * nxt.element_size()
            o(x, y, x_sumsq=self.sq, y_peers=[a + off for a in self.peer_x[1 - self.cur]])
            self._sumsq(y, self.sq, self.scratch)
            if self.sync_host:
                torch.cuda.synchronize()  # gloo: the peer stores are done before we meet
            self.dist.all_reduce(self.sq, group=self.group)
            self.cur = 1 - self.cur
            return

        def wait_gather():
            if self.pending is not None:
                self.pending.wait()
                self.pending = None

        o(x, y, x_sumsq=self.sq, before_remote=wait_gather)
        wait_gather()
        self._sumsq(y, self.sq, self.scratch)
        if self.dist is not None:
            self.dist.all_reduce(self.sq, group=self.group)
            work = self.dist.all_gather_into_tensor(nxt, self._own(nxt), group=self.group,
                                                    async_op=True)
            if self.overlap:
                self.pending = work
            else:
                work.wait()
        self.cur = 1 - self.cur

    def finish(self) -> None:
        if self.pending is not None:
            self.pending.wait()
            self.pending = None

    def x_global(self) -> torch.Tensor:
        """The current iterate x_k / ||x_k|| in the global row order."""
        self.finish()
        o = self.op
        x = self.xs[self.cur]
        parts = [x[st.rank * o.pad:st.rank * o.pad + st.rows] for st in o.stripes]
        v = torch.cat(parts).to(torch.float64)
        return v / torch.sqrt((v * v).sum())
