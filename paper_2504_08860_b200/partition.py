"""2D partitioning into row_height x col_width blocks, compact on the GPU.

Mirrors /root/reference/pkg/src/hbp_spmv/partition.py.  The reference's
BlockGrid holds dense [ncb, rows] arrays (:58-97) that do not fit at the
benchmark scales; here the grid is the list of NONZERO
blocks in bc-major order plus compact per-block slot arrays:

    blk_br, blk_bc   int32[nzb]       nonzero block directory (bc-major)
    len_local        u32[nzb * R]     in-block count of each local row
    start_local      int64[nzb * R]   CSR offset where that run begins
    nz_block_nnz     int64[nzb]

The reference attributes (row_counts, row_starts, block_nnz,
block_elem_start) are still available as dense views built on demand.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .formats import CsrMatrix

__all__ = ["PartitionConfig", "BlockGrid", "make_grid", "block_rows_of",
           "rows_in_row_block", "groups_in_row_block", "groups_per_col_block"]


@dataclass(frozen=True)
class PartitionConfig:
    """partition.py:19-40: column width, row height, lane-group width and the
    scheduler's fixed fraction.  The GPU kernels support warp_size <= 32."""

    col_width: int = 4096
    row_height: int = 512
    warp_size: int = 32
    fixed_fraction: float = 0.7

    def __post_init__(self):
        if self.col_width < 1 or self.row_height < 1 or self.warp_size < 1:
            raise ValueError("partition sizes must be >= 1")
        if self.row_height % self.warp_size != 0:
            raise ValueError("row_height must be a multiple of warp_size")
        if not 0.0 <= self.fixed_fraction <= 1.0:
            raise ValueError("fixed_fraction must be in [0, 1]")


def rows_in_row_block(rows: int, row_height: int, br: int) -> int:
    """partition.py:43-44."""
    return min(row_height, rows - br * row_height)


def groups_in_row_block(rows: int, row_height: int, warp_size: int, br: int) -> int:
    """partition.py:47-49."""
    n = rows_in_row_block(rows, row_height, br)
    return -(-n // warp_size)


def groups_per_col_block(rows: int, row_height: int, warp_size: int) -> int:
    """partition.py:52-55."""
    nrb = -(-rows // row_height)
    full = (nrb - 1) * (row_height // warp_size)
    return full + groups_in_row_block(rows, row_height, warp_size, nrb - 1)


def _check_gpu_geometry(config: PartitionConfig):
    if config.warp_size > 32:
        raise ValueError("warp_size > 32 is not supported by the GPU kernels "
                         "(one lane group must fit in a hardware warp)")


@dataclass(eq=False)
class BlockGrid:
    """Compact block grid (see module docstring)."""

    rows: int
    cols: int
    config: PartitionConfig
    num_row_blocks: int
    num_col_blocks: int
    nnz: int
    blk_br: torch.Tensor
    blk_bc: torch.Tensor
    len_local: torch.Tensor
    start_local: torch.Tensor
    nz_block_nnz: torch.Tensor
    csr: CsrMatrix | None = None
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def nzb(self) -> int:
        return self.blk_br.numel()

    # ---- addressing (partition.py:79-97)
    def rows_in_block(self, br: int) -> int:
        return rows_in_row_block(self.rows, self.config.row_height, br)

    def groups_in_block(self, br: int) -> int:
        return groups_in_row_block(self.rows, self.config.row_height, self.config.warp_size, br)

    def slot_base(self, br: int, bc: int) -> int:
        return bc * self.rows + br * self.config.row_height

    def group_base(self, br: int, bc: int) -> int:
        per_col = groups_per_col_block(self.rows, self.config.row_height, self.config.warp_size)
        return bc * per_col + br * (self.config.row_height // self.config.warp_size)

    def block_index(self, br: int, bc: int) -> int:
        """Position of (br, bc) in the nonzero-block list, or -1."""
        keys = self._cache.get("keys")
        if keys is None:
            keys = (self.blk_bc.to(torch.int64) * self.num_row_blocks + self.blk_br).cpu().numpy()
            self._cache["keys"] = keys
        k = bc * self.num_row_blocks + br
        i = int(np.searchsorted(keys, k))
        return i if i < keys.size and keys[i] == k else -1

    def nnz_per_row(self, br: int, bc: int) -> torch.Tensor:
        """In-block nonzero count per local row of block (br, bc) (partition.py:94-97)."""
        n = self.rows_in_block(br)
        i = self.block_index(br, bc)
        R = self.config.row_height
        if i < 0:
            return torch.zeros(n, dtype=torch.int32, device=self.blk_br.device)
        return self.len_local[i * R:i * R + n].clone()

    # ---- dense reference views (partition.py:73-77), built on demand
    @property
    def block_nnz(self) -> np.ndarray:
        """int64 [nrb, ncb] (partition.py:118-120)."""
        if "block_nnz" not in self._cache:
            out = np.zeros((self.num_row_blocks, self.num_col_blocks), np.int64)
            out[self.blk_br.cpu().numpy(), self.blk_bc.cpu().numpy()] = \
                self.nz_block_nnz.cpu().numpy()
            self._cache["block_nnz"] = out
        return self._cache["block_nnz"]

    @property
    def block_elem_start(self) -> np.ndarray:
        """int64 [nrb, ncb], exclusive bc-major prefix of block_nnz (partition.py:122-124)."""
        flat = self.block_nnz.T.ravel()
        starts = np.concatenate(([0], np.cumsum(flat)[:-1])).astype(np.int64)
        return np.ascontiguousarray(starts.reshape(self.num_col_blocks, self.num_row_blocks).T)

    def _dense_slots(self, src: torch.Tensor, dtype) -> torch.Tensor:
        R = self.config.row_height
        out = torch.zeros(self.num_col_blocks * self.rows, dtype=dtype, device=src.device)
        if self.nzb:
            s = torch.arange(R, device=src.device)
            br = self.blk_br.to(torch.int64)[:, None]
            dst = self.blk_bc.to(torch.int64)[:, None] * self.rows + br * R + s[None, :]
            ok = (br * R + s[None, :]) < self.rows
            out[dst[ok]] = src.view(self.nzb, R)[ok].to(dtype)
        return out

    @property
    def row_counts(self) -> np.ndarray:
        """int32 [ncb, rows] dense view (partition.py:110-112)."""
        return self._dense_slots(self.len_local, torch.int32).view(
            self.num_col_blocks, self.rows).cpu().numpy()

    @property
    def row_starts(self) -> np.ndarray:
        """int64 [ncb, rows] dense view (partition.py:114-116); for (bc, row)
        with no elements the reference's value is row_ptr[row] + elements of
        that row in lower column blocks, which equals the next run's start."""
        ncb, rows = self.num_col_blocks, self.rows
        counts = self.row_counts.astype(np.int64)
        before = np.cumsum(counts, axis=0) - counts
        rp = self.csr.row_ptr.cpu().numpy() if self.csr is not None else None
        if rp is None:
            raise ValueError("row_starts needs the CSR the grid was built from")
        return rp[:-1][None, :] + before

    def to_reference(self) -> dict:
        return dict(row_counts=self.row_counts, row_starts=self.row_starts,
                    block_nnz=self.block_nnz, block_elem_start=self.block_elem_start)


def make_grid(csr: CsrMatrix, config: PartitionConfig) -> BlockGrid:
    """partition.py:100-127 on the GPU: split each CSR row run at multiples of
    col_width; keep only nonzero blocks (compact)."""
    if csr.rows < 1 or csr.cols < 1:
        raise ValueError("matrix must have nonempty dimensions")
    _check_gpu_geometry(config)
    dev = L.require_cuda()
    rows, cols = csr.rows, csr.cols
    R, C = config.row_height, config.col_width
    nrb, ncb = -(-rows // R), -(-cols // C)
    i64 = lambda n: torch.empty(n, dtype=torch.int64, device=dev)  # noqa: E731
    i32 = lambda n: torch.empty(n, dtype=torch.int32, device=dev)  # noqa: E731
    s = L.stream()

    runs_per_row = i64(rows + 1)
    runs_per_row[rows:] = 0
    L.call("hbp_grid_count_runs", L.P(csr.row_ptr), L.P(csr.col_idx), L.c_i64(rows),
           L.c_i64(cols), L.c_i64(C), L.P(runs_per_row), s)
    run_offset = L.exclusive_sum(runs_per_row)
    nruns = int(run_offset[rows].item())
    run_bc, run_row, run_cnt = i32(nruns), i32(nruns), i32(nruns)
    run_start = i64(nruns)
    L.call("hbp_grid_emit_runs", L.P(csr.row_ptr), L.P(csr.col_idx), L.c_i64(rows), L.c_i64(cols),
           L.c_i64(C), L.P(run_offset), L.c_i64(nruns), L.P(run_bc), L.P(run_row),
           L.P(run_start), L.P(run_cnt), s)
    if ncb > 1 and nruns:
        idx = torch.arange(nruns, dtype=torch.int32, device=dev)
        sbc, order = L.sort_pairs_u32(run_bc, idx, max(1, int(ncb - 1).bit_length()))
    else:
        sbc, order = None, None
    head = i64(nruns)
    L.call("hbp_grid_block_heads", L.P(sbc), L.P(order), L.P(run_row), L.c_i64(nruns),
           L.c_i64(R), L.P(head), s)
    incl = L.inclusive_sum(head)
    nzb = int(incl[-1].item()) if nruns else 0
    blk_br, blk_bc = i32(nzb), i32(nzb)
    len_local = torch.zeros(nzb * R, dtype=torch.int32, device=dev)
    start_local = torch.zeros(nzb * R, dtype=torch.int64, device=dev)
    L.call("hbp_grid_fill_slots", L.P(sbc), L.P(order), L.P(run_row), L.P(run_start),
           L.P(run_cnt), L.P(incl), L.c_i64(nruns), L.c_i64(R), L.P(blk_br), L.P(blk_bc),
           L.P(len_local), L.P(start_local), s)
    nz_block_nnz = i64(nzb)
    L.call("hbp_block_nnz", L.P(len_local), L.c_i64(nzb), L.c_i64(R), L.P(nz_block_nnz), s)
    return BlockGrid(rows, cols, config, nrb, ncb, csr.nnz, blk_br, blk_bc, len_local,
                     start_local, nz_block_nnz, csr)


def block_rows_of(csr: CsrMatrix, grid: BlockGrid, br: int, bc: int):
    """partition.py:130-143: each local row's (global columns, values) in block (br, bc)."""
    if not (0 <= br < grid.num_row_blocks and 0 <= bc < grid.num_col_blocks):
        raise IndexError(f"block ({br}, {bc}) out of range")
    R = grid.config.row_height
    i = grid.block_index(br, bc)
    n = grid.rows_in_block(br)
    lens = grid.len_local[i * R:i * R + n].cpu().numpy() if i >= 0 else np.zeros(n, np.int64)
    starts = grid.start_local[i * R:i * R + n].cpu().numpy() if i >= 0 else np.zeros(n, np.int64)
    col = csr.col_idx
    for r in range(n):
        j, k = int(starts[r]), int(lens[r])
        yield col[j:j + k].to(torch.int64), csr.values[j:j + k]
