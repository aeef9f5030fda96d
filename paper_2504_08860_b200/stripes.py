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
           "power_iteration"]


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
