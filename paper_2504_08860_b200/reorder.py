"""Nonlinear-hash row reordering (and the identity / sort orderings) on the GPU.

Mirrors /root/reference/pkg/src/hbp_spmv/reorder.py.  The hash constants
(a, b, c, d) are chosen on the host with the reference's own numpy calls
(reorder.py:69-103) from 4096 counts the GPU looks up; every nonzero block's
permutation is then built by ``hbp_hash_perm`` (FCFS linear probing, one warp
per block over a register-resident occupancy bitmap, bit-exact with _kernels.py:62-92).

Permutations are returned as ``BlockPermutations``: compact per nonzero block
on the device, array-like (``.size``, ``np.asarray``, slicing) over the
reference's dense flat [ncb * rows] table so ``perm_for_block`` and direct
indexing behave as in the reference.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .partition import BlockGrid, PartitionConfig

__all__ = ["HashParams", "OpCounter", "BlockPermutations", "sample_hash_params", "hash_slot",
           "build_block_permutation", "hash_permutations", "sort_permutation",
           "sort_permutations", "identity_permutations", "perm_for_block", "BUCKET_MAX"]

BUCKET_MAX = 8  # reorder.py:37


@dataclass(frozen=True)
class HashParams:
    """reorder.py:40-58."""

    a: int
    b: int
    c: int
    d: int
    bucket_max: int = BUCKET_MAX

    def __post_init__(self):
        if self.a < 0:
            raise ValueError("shift a must be >= 0")
        if self.b < 1:
            raise ValueError("bucket stride b must be >= 1")
        if self.d != self.b:
            raise ValueError("d must equal b")
        if math.gcd(self.c, self.d) != 1:
            raise ValueError("c must be co-prime with d")


@dataclass
class OpCounter:
    """reorder.py:61-66."""

    probes: int = 0
    comparisons: int = 0


class BlockPermutations:
    """Slot -> local-row tables of every block (execution slot order).

    ``compact`` is u32 [nzb * R] on the device (nonzero blocks only); empty
    blocks' tables are implied (``empty_kind``): the hash of an all-zero
    block (a pure function of its height), the
    identity, or the stable sort of zeros (= identity)."""

    def __init__(self, grid: BlockGrid, compact: torch.Tensor, kind: str,
                 params: HashParams | None = None):
        self.grid = grid
        self.compact = compact
        self.kind = kind
        self.params = params
        self._dense = None

    @property
    def size(self) -> int:
        return self.grid.num_col_blocks * self.grid.rows

    def __len__(self) -> int:
        return self.size

    def empty_block_perm(self, n: int) -> np.ndarray:
        if self.kind != "hash":
            return np.arange(n, dtype=np.uint32)
        p = self.params
        out = torch.empty(n, dtype=torch.int32, device=self.compact.device)
        L.call("hbp_hash_perm_empty", L.c_i64(n), L.c_i64(p.a), L.c_i64(p.b), L.c_i64(p.c),
               L.c_i64(p.d), L.c_i64(p.bucket_max), L.P(out), L.stream())
        return out.cpu().numpy().view(np.uint32)

    def dense_device(self) -> torch.Tensor:
        """The reference's flat [ncb * rows] table as an int32 (u32 bits) device tensor."""
        if self._dense is None:
            g = self.grid
            R = g.config.row_height
            nrb = g.num_row_blocks
            last = g.rows - (nrb - 1) * R
            full = torch.as_tensor(self.empty_block_perm(R).view(np.int32))
            lastp = torch.as_tensor(self.empty_block_perm(last).view(np.int32))
            one = torch.cat([full.repeat(nrb - 1), lastp]).to(self.compact.device)
            dense = one.repeat(g.num_col_blocks)
            if g.nzb:
                s = torch.arange(R, device=dense.device)
                br = g.blk_br.to(torch.int64)[:, None]
                dst = g.blk_bc.to(torch.int64)[:, None] * g.rows + br * R + s[None, :]
                ok = (br * R + s[None, :]) < g.rows
                dense[dst[ok]] = self.compact.view(g.nzb, R)[ok]
            self._dense = dense
        return self._dense

    def __array__(self, dtype=None, copy=None):
        a = self.dense_device().cpu().numpy().view(np.uint32)
        return a.astype(dtype) if dtype is not None else a

    def __getitem__(self, item):
        return np.asarray(self)[item]


def _grid_counts_at(grid: BlockGrid, flat: np.ndarray) -> np.ndarray:
    """row_counts.reshape(-1)[flat] via the GPU (binary search in CSR rows)."""
    if grid.csr is None:
        raise ValueError("sample_hash_params needs the grid's CSR")
    dev = grid.blk_br.device
    idx = torch.as_tensor(np.ascontiguousarray(flat, np.int64), device=dev)
    out = torch.empty(idx.numel(), dtype=torch.int32, device=dev)
    L.call("hbp_sample_counts", L.P(grid.csr.row_ptr), L.P(grid.csr.col_idx),
           L.c_i64(grid.rows), L.c_i64(grid.config.col_width), L.P(idx), L.c_i64(idx.numel()),
           L.P(out), L.stream())
    return out.cpu().numpy()


def sample_hash_params(grid: BlockGrid, config: PartitionConfig, sample_size: int = 4096,
                       seed: int = 0, quantile: float = 0.9) -> HashParams:
    """reorder.py:69-103.  The index draw is numpy's default_rng(seed).choice
    over the dense (bc, row) population (independent of its contents, so it
    needs no dense grid); the GPU supplies the counts at those indices; the
    (a, c) arithmetic is the reference's, on the host."""
    pop = grid.num_col_blocks * grid.rows
    if sample_size < pop:
        rng = np.random.default_rng(seed)
        flat = rng.choice(pop, sample_size, replace=False)
    else:
        flat = np.arange(pop, dtype=np.int64)
    sample = _grid_counts_at(grid, flat).astype(np.int64)

    b = max(1, config.row_height // (BUCKET_MAX + 1))
    a = 0
    if sample.size:
        while np.quantile(sample >> a, quantile, method="inverted_cdf") > BUCKET_MAX:
            a += 1
    if sample.size:
        buckets = np.minimum(sample >> a, BUCKET_MAX)
        modal = int(np.bincount(buckets, minlength=BUCKET_MAX + 1).max())
    else:
        modal = 0
    c = max(1, -(-modal // b))
    while math.gcd(c, b) != 1:
        c += 1
    return HashParams(a=a, b=b, c=c, d=b)


def hash_slot(nnz: int, local_row: int, params: HashParams) -> int:
    """reorder.py:106-109: preliminary slot before collision resolution."""
    g = min(nnz >> params.a, params.bucket_max)
    return g * params.b + (local_row * params.c) % params.d


def _hash_compact(len_local, blk_br, nzb, rows, R, params, counter):
    dev = len_local.device
    perm = torch.empty(nzb * R, dtype=torch.int32, device=dev)
    probes = torch.zeros(1, dtype=torch.int64, device=dev)
    L.call("hbp_hash_perm", L.P(len_local), L.P(blk_br), L.c_i64(nzb), L.c_i64(rows), L.c_i64(R),
           L.c_i64(params.a), L.c_i64(params.b), L.c_i64(params.c), L.c_i64(params.d),
           L.c_i64(params.bucket_max), L.P(perm), L.P(probes), L.stream())
    if counter is not None:
        counter.probes += int(probes.item())
    return perm


def build_block_permutation(row_nnz, params: HashParams,
                            counter: OpCounter | None = None) -> np.ndarray:
    """reorder.py:112-136 for one block (runs the same GPU kernel)."""
    dev = L.require_cuda()
    lens = torch.as_tensor(np.asarray(row_nnz, dtype=np.int64).astype(np.int32), device=dev)
    n = lens.numel()
    if n == 0:
        return np.empty(0, np.uint32)
    br = torch.zeros(1, dtype=torch.int32, device=dev)
    perm = _hash_compact(lens, br, 1, n, n, params, counter)
    return perm.cpu().numpy().view(np.uint32)


def hash_permutations(grid: BlockGrid, params: HashParams,
                      counter: OpCounter | None = None) -> BlockPermutations:
    """reorder.py:174-184: every nonzero block's hash permutation (one GPU
    warp per block, the block's occupancy bitmap in the warp's registers).  The probe count covers nonzero blocks plus the
    implied empty blocks, so it equals the reference's OpCounter.probes."""
    R = grid.config.row_height
    perm = _hash_compact(grid.len_local, grid.blk_br, grid.nzb, grid.rows, R, params, counter)
    if counter is not None:
        counter.probes += _empty_block_probes(grid, params)
    return BlockPermutations(grid, perm, "hash", params)


def _empty_block_probes(grid: BlockGrid, params: HashParams) -> int:
    """Probes the reference spends on empty blocks: (count of empty blocks of
    each height) x (probes of one all-zero block of that height)."""
    R = grid.config.row_height
    nrb, ncb = grid.num_row_blocks, grid.num_col_blocks
    last = grid.rows - (nrb - 1) * R
    br = grid.blk_br.cpu().numpy()
    nz_last = int((br == nrb - 1).sum())
    nz_full = grid.nzb - nz_last
    total = 0
    if last == R:
        groups = [(R, ncb * nrb - grid.nzb)]
    else:
        groups = [(R, ncb * (nrb - 1) - nz_full), (last, ncb - nz_last)]
    for n, empties in groups:
        if empties <= 0:
            continue
        ctr = OpCounter()
        build_block_permutation(np.zeros(n, np.int64), params, ctr)
        total += empties * ctr.probes
    return total


def sort_permutation(row_nnz, counter: OpCounter | None = None) -> np.ndarray:
    """reorder.py:160-171: ascending nnz, ties by ascending local row (GPU
    stable block radix sort).  With a counter attached, ``hbp_merge_comparisons``
    adds the comparisons the reference's instrumented merge sort
    (reorder.py:139-157) makes on the same keys; the permutation is the same
    either way, as in the reference."""
    dev = L.require_cuda()
    keys = np.asarray(row_nnz, dtype=np.int64)
    if keys.size and (keys.min() < 0 or keys.max() >= 2**31):
        raise ValueError("row nnz counts must lie in [0, 2^31)")
    lens = torch.as_tensor(keys.astype(np.int32), device=dev)
    n = lens.numel()
    if counter is not None and n > 1:
        k64 = torch.as_tensor(keys, device=dev)
        cmp = torch.zeros(1, dtype=torch.int64, device=dev)
        L.call("hbp_merge_comparisons", L.P(k64), L.c_i64(n), L.P(cmp), L.stream())
        counter.comparisons += int(cmp.item())
    if n == 0:
        return np.empty(0, np.uint32)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    br = torch.zeros(1, dtype=torch.int32, device=dev)
    L.call("hbp_sort_perm", L.P(lens), L.P(br), L.c_i64(1), L.c_i64(n), L.c_i64(n), L.P(perm),
           L.stream())
    return perm.cpu().numpy().view(np.uint32)


def sort_permutations(grid: BlockGrid) -> BlockPermutations:
    """reorder.py:187-219: per block stable sort by nnz (the sort2D baseline)."""
    R = grid.config.row_height
    perm = torch.empty(grid.nzb * R, dtype=torch.int32, device=grid.blk_br.device)
    L.call("hbp_sort_perm", L.P(grid.len_local), L.P(grid.blk_br), L.c_i64(grid.nzb),
           L.c_i64(grid.rows), L.c_i64(R), L.P(perm), L.stream())
    return BlockPermutations(grid, perm, "sort")


def identity_permutations(grid: BlockGrid) -> BlockPermutations:
    """reorder.py:222-225."""
    R = grid.config.row_height
    perm = torch.arange(R, dtype=torch.int32, device=grid.blk_br.device).repeat(grid.nzb)
    return BlockPermutations(grid, perm, "identity")


def perm_for_block(perm_flat, grid: BlockGrid, br: int, bc: int) -> np.ndarray:
    """reorder.py:228-231."""
    base = grid.slot_base(br, bc)
    return np.asarray(perm_flat)[base:base + grid.rows_in_block(br)]
