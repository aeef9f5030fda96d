"""The HBP format on the GPU: build, reference-layout views, validation, inverse.

Mirrors /root/reference/pkg/src/hbp_spmv/hbp.py.  Element arrays (col, data,
add_sign) have exactly the reference's layout (bc-major blocks, groups,
column-major steps within a group).  The slot and group arrays are kept
compact over nonzero blocks for the kernels; ``zero_row``, ``output_hash``
and ``group_start`` expose the reference's dense layout (hbp.py:51-62) as
device tensors built on first access (``hbp_expand_reference``).

Runtime layout (HBM) used by the SpMV kernel:
    col u32[nnz], data f32|f64[nnz]              streamed once per SpMV
    slot_len u32[nzb*R], perm u32[nzb*R]         per-slot length / output row
    group_start_c int64[nzb*gpb + 1]             per-group element base
    blk_br, blk_bc int32[nzb]                    nonzero block directory
    rb_ptr int64[nrb+1], rb_blk int32[nzb]       combine lists (ascending bc)
add_sign is produced for the reference view and the .hbp codec; the kernel
derives addresses from slot lengths instead of chasing it.
"""
from __future__ import annotations

import ctypes
import os
import io
import struct

import numpy as np
import torch

from . import _lib as L
from .formats import CsrMatrix, TripletMatrix
from .partition import (BlockGrid, PartitionConfig, _check_gpu_geometry, groups_in_row_block,
                        groups_per_col_block, rows_in_row_block)
from .reorder import BlockPermutations

__all__ = ["HbpMatrix", "HbpFormatError", "build_hbp", "hbp_to_triplets", "serialize_hbp",
           "deserialize_hbp", "save_hbp", "load_hbp", "validate_reference_arrays"]

MAGIC = b"HBP1"
VERSION = 1


def _padded(t: torch.Tensor, pad: int = 16) -> torch.Tensor:
    """Copy of a 1-D tensor whose storage extends `pad` elements past its end
    (the streaming kernel's 16-byte bulk copies may read past the last element)."""
    out = torch.zeros(t.numel() + pad, dtype=t.dtype, device=t.device)
    out[:t.numel()] = t
    return out[:t.numel()]


class HotColumns:
    """x staging of the heaviest columns (hbp_spmv_stream): hot_cols[s] is
    the column of hot slot s (then of warm slot w at n_hot + w), scol the
    element stream with hot columns as HBP_HOT_FLAG | s and warm ones as
    HBP_WARM_FLAG | w, share / warm_share the fractions of nonzeros."""

    def __init__(self, n_hot: int, hot_cols: torch.Tensor, scol: torch.Tensor, share: float,
                 n_warm: int = 0, warm_share: float = 0.0):
        self.n_hot, self.hot_cols, self.scol, self.share = n_hot, hot_cols, scol, share
        self.n_warm, self.warm_share = n_warm, warm_share

    packed = False  # HBP_FLAG_PACKED_X: n_warm counts the packed copy of x

    def refresh_order(self):
        """(cols, slots): the staged slots in ascending column order, for the
        per-SpMV refresh of x_hot (reads x in column order).  Cached."""
        if self._refresh is None:
            n = self.hot_cols.numel()
            slots = torch.arange(n, dtype=torch.int32, device=self.hot_cols.device)
            cols, slots = L.sort_pairs_u32(self.hot_cols.contiguous(), slots, 32)
            self._refresh = (cols, slots)
        return self._refresh

    _refresh = None

    def apply(self, f: "L.FormatT") -> None:
        f.scol, f.hot_cols = self.scol.data_ptr(), self.hot_cols.data_ptr()
        f.n_hot, f.n_warm = self.n_hot, self.n_warm
        if os.environ.get("HBP_HOT_REFRESH", "1") != "0" and self.hot_cols.numel():
            cols, slots = self.refresh_order()
            f.refresh_cols, f.refresh_slots = cols.data_ptr(), slots.data_ptr()
        if self.packed:
            f.reserved |= 8  # HBP_FLAG_PACKED_X
            f.cold_last = 1


class HbpFormatError(ValueError):
    """hbp.py:47-48: malformed .hbp streams or structurally invalid matrices."""


class HbpMatrix:
    """Device-resident HBP matrix (hbp.py:51-135)."""

    def __init__(self, rows: int, cols: int, config: PartitionConfig, grid_shape, *,
                 col: torch.Tensor, data: torch.Tensor, add_sign: torch.Tensor | None,
                 blk_br: torch.Tensor, blk_bc: torch.Tensor, slot_len: torch.Tensor,
                 perm: torch.Tensor, group_start_c: torch.Tensor,
                 zero_row_c: torch.Tensor | None, rb_ptr: torch.Tensor, rb_blk: torch.Tensor,
                 permutations=None):
        self.rows, self.cols, self.config = rows, cols, config
        self.grid_shape = tuple(grid_shape)
        self.col, self.data, self._add_sign = col, data, add_sign
        self.blk_br, self.blk_bc = blk_br, blk_bc
        self.slot_len, self.perm = slot_len, perm
        self.group_start_c, self.zero_row_c = group_start_c, zero_row_c
        self.rb_ptr, self.rb_blk = rb_ptr, rb_blk
        self.permutations = permutations
        self.phase_ptr = None
        self.phases = None
        self._views: dict = {}
        self._fmt = None
        self._ops: dict = {}

    def ensure_phases(self) -> None:
        """Build the phase stream (runtime index of hbp_spmv_stream, W = 32):
        per group its (live mask, element offset) phases, ~9 per group on
        R-MAT, 8 bytes each (include/hbp.h hbp_phase_counts/emit)."""
        if self.phases is not None:
            return
        if self.config.warp_size != 32:
            raise ValueError("the phase stream needs warp_size == 32")
        dev = self.data.device
        ng = self.nzb * (self.config.row_height // 32)
        nph = torch.empty(ng + 1, dtype=torch.int64, device=dev)
        L.call("hbp_phase_counts", L.P(self.slot_len), L.c_i64(ng), L.P(nph), L.stream())
        ptr = L.exclusive_sum(nph)
        total = int(ptr[-1].item())
        if total + 32 >= (1 << 31):  # the stream kernel keeps phase offsets in 32 bits
            raise ValueError(f"phase stream of {total} entries exceeds the 32-bit kernel index")
        # + 32 entries: the stream kernel reads a whole warp's worth of phases
        # per group without waiting for the group's phase count
        phases = torch.zeros((total + 32) * 2, dtype=torch.int32, device=dev)
        L.call("hbp_phase_emit", L.P(self.slot_len), L.c_i64(ng), L.P(ptr), L.P(phases),
               L.stream())
        self.phase_ptr, self.phases = ptr, phases
        if self._fmt is not None:
            self._fmt.phase_ptr = ptr.data_ptr()
            self._fmt.phases = phases.data_ptr()

    def hot_capacity(self, warm: bool = False, packed: bool = False) -> int:
        """Largest hot set the stream kernel can stage for this dtype (with or
        without a warm tier in the same launch)."""
        cap = L.c_i64(0)
        L.call("hbp_hot_capacity", L.c_int(L.dtype_code(self.data.dtype)),
               L.c_int(2 if packed else int(warm)),
               ctypes.byref(cap))
        return int(cap.value)

    RANK_SAMPLE = 1 << 28  # column degrees from at most ~256M sampled elements

    def column_ranking(self):
        """(degree, order): nonzeros per column and the columns by descending
        degree, ties by ascending column (hbp_col_degree + stable radix sort).
        Above RANK_SAMPLE elements the degrees count every stride-th element
        (a power of two): the ranking only picks which columns are staged.
        Cached."""
        if "rank" not in self._ops:
            dev = self.data.device
            stride = 1
            while self.nnz // stride > self.RANK_SAMPLE:
                stride *= 2
            deg = torch.zeros(self.cols, dtype=torch.int32, device=dev)
            L.call("hbp_col_degree", L.P(self.col), L.c_i64(self.nnz), L.c_i64(stride), L.P(deg),
                   L.stream())
            keys = (torch.iinfo(torch.int32).max - deg).contiguous()
            vals = torch.arange(self.cols, dtype=torch.int32, device=dev)
            _, order = L.sort_pairs_u32(keys, vals, 32)
            self._ops["rank"] = (deg, order)
            self._ops["rank_stride"] = stride
        return self._ops["rank"]

    def used_columns(self):
        """(used bool[cols], n_used): the columns the matrix touches, exact even
        when the ranking was sampled (then one full degree pass).  Cached."""
        if "used_cols" not in self._ops:
            deg, _ = self.column_ranking()
            if self._ops["rank_stride"] != 1:
                deg = torch.zeros(self.cols, dtype=torch.int32, device=self.data.device)
                L.call("hbp_col_degree", L.P(self.col), L.c_i64(self.nnz), L.c_i64(1),
                       L.P(deg), L.stream())
            used = deg > 0
            self._ops["used_cols"] = (used, int(used.sum().item()))
        return self._ops["used_cols"]

    def column_share(self, n: int) -> float:
        """Fraction of the (sampled) nonzeros in the n heaviest columns."""
        if n <= 0 or not self.nnz:
            return 0.0
        deg, order = self.column_ranking()
        return float(deg[order[:n].long()].to(torch.int64).sum().item()) / max(
            1, int(deg.to(torch.int64).sum().item()))

    def hot_columns(self, n_hot: int | None = None, n_warm: int = 0,
                    packed: bool = False) -> "HotColumns":
        """Hot-column staging metadata for hbp_spmv_stream (include/hbp.h
        hbp_col_degree .. hbp_hot_remap): the n_hot heaviest columns (capped
        by the kernel's shared-memory capacity), then the n_warm next ones
        (warm tier), and the staged column stream.  packed: every used column
        after the hot ones goes to the packed copy of x (HBP_FLAG_PACKED_X;
        n_warm is ignored).  Cached."""
        if packed:
            return self._packed_columns(n_hot)
        cap = self.hot_capacity(warm=n_warm > 0)
        n = cap if n_hot is None else min(int(n_hot), cap)
        n = max(0, min(n, self.cols)) & ~3
        if self.cols >= (1 << 31):  # the staged stream flags hot columns with bit 31
            n = 0
        nw = max(0, min(int(n_warm), self.cols - n)) if self.cols <= (1 << 30) else 0
        key = ("hot", n, nw)
        if key in self._ops:
            return self._ops[key]
        dev = self.data.device
        deg, order = self.column_ranking()
        hot_cols = order[:n + nw].contiguous()
        dsum = torch.cumsum(deg[hot_cols.long()].to(torch.int64), 0)
        total = max(1, int(deg.to(torch.int64).sum().item()))
        share = float(dsum[n - 1].item()) / total if n else 0.0
        warm_share = (float(dsum[-1].item()) / total - share) if nw else 0.0
        slot_of = torch.full((self.cols,), -1, dtype=torch.int32, device=dev)
        L.call("hbp_hot_slots", L.P(hot_cols), L.c_i64(n + nw), L.P(slot_of), L.stream())
        scol = _padded(torch.empty(self.nnz, dtype=self.col.dtype, device=dev))
        L.call("hbp_hot_remap", L.P(self.col), L.c_i64(self.nnz), L.P(slot_of), L.c_i64(n),
               L.P(scol), L.stream())
        hc = HotColumns(n, hot_cols, scol, share, nw, warm_share)
        self._ops[key] = hc
        return hc

    def _packed_columns(self, n_hot: int | None) -> "HotColumns":
        """Packed x: the n_hot heaviest columns (staged in shared memory), then
        every other used column in ascending column order.  The copy holds
        only the columns the matrix touches (cfg2: 7.36M of 16.8M, 29 MB), so
        it stays L2-resident where x thrashed; ascending order makes the
        per-SpMV refresh one coalesced sweep over x."""
        cap = self.hot_capacity(packed=True)
        n = cap if n_hot is None else min(int(n_hot), cap)
        used, n_used = self.used_columns()
        deg, order = self.column_ranking()
        n = max(0, min(n, n_used)) & ~3
        key = ("packed", n)
        if key in self._ops:
            return self._ops[key]
        dev = self.data.device
        hot = order[:n]
        rest = used.clone()
        rest[hot.long()] = False
        hot_cols = torch.cat([hot, rest.nonzero().view(-1).to(torch.int32)]).contiguous()
        total = max(1, int(deg.to(torch.int64).sum().item()))
        share = float(deg[hot.long()].to(torch.int64).sum().item()) / total if n else 0.0
        slot_of = torch.full((self.cols,), -1, dtype=torch.int32, device=dev)
        L.call("hbp_hot_slots", L.P(hot_cols), L.c_i64(n_used), L.P(slot_of), L.stream())
        scol = _padded(torch.empty(self.nnz, dtype=self.col.dtype, device=dev))
        L.call("hbp_hot_remap_packed", L.P(self.col), L.c_i64(self.nnz), L.P(slot_of),
               L.c_i64(n), L.P(scol), L.stream())
        hc = HotColumns(n, hot_cols, scol, share, n_used - n, 1.0 - share)
        hc.packed = True
        self._ops[key] = hc
        return hc

    # ---- reference attributes
    @property
    def nnz(self) -> int:
        return self.data.numel()

    @property
    def nzb(self) -> int:
        return self.blk_br.numel()

    @property
    def dtype(self) -> torch.dtype:
        return self.data.dtype

    @property
    def num_row_blocks(self) -> int:
        return self.grid_shape[0]

    @property
    def num_col_blocks(self) -> int:
        return self.grid_shape[1]

    def rows_in_block(self, br: int) -> int:
        return rows_in_row_block(self.rows, self.config.row_height, br)

    def groups_in_block(self, br: int) -> int:
        return groups_in_row_block(self.rows, self.config.row_height, self.config.warp_size, br)

    def slot_base(self, br: int, bc: int) -> int:
        return bc * self.rows + br * self.config.row_height

    def group_base(self, br: int, bc: int) -> int:
        per_col = groups_per_col_block(self.rows, self.config.row_height, self.config.warp_size)
        return bc * per_col + br * (self.config.row_height // self.config.warp_size)

    @property
    def add_sign(self) -> torch.Tensor:
        if self._add_sign is None:
            raise ValueError("this HbpMatrix was built without add_sign")
        return self._add_sign

    def _expand(self):
        if "zero_row" in self._views:
            return
        R, W, C = self.config.row_height, self.config.warp_size, self.config.col_width
        nrb, ncb = self.grid_shape
        dev = self.data.device
        gpc = groups_per_col_block(self.rows, R, W)
        zr = torch.empty(ncb * self.rows, dtype=torch.int32, device=dev)
        oh = torch.empty(ncb * self.rows, dtype=torch.int32, device=dev)
        gs = torch.empty(ncb * gpc + 1, dtype=torch.int64, device=dev)
        last = self.rows - (nrb - 1) * R
        if isinstance(self.permutations, BlockPermutations):
            ef = torch.as_tensor(self.permutations.empty_block_perm(R).view(np.int32), device=dev)
            el = torch.as_tensor(self.permutations.empty_block_perm(last).view(np.int32),
                                 device=dev)
        else:
            ef = torch.arange(R, dtype=torch.int32, device=dev)
            el = torch.arange(last, dtype=torch.int32, device=dev)
        zrc = self.zero_row_c
        if zrc is None:
            raise ValueError("this HbpMatrix was built without zero_row")
        L.call("hbp_expand_reference", L.P(self.blk_br), L.P(self.blk_bc), L.c_i64(self.nzb),
               L.c_i64(self.rows), L.c_i64(self.cols), L.c_i64(self.nnz), L.c_i64(C), L.c_i64(R),
               L.c_i64(W), L.P(self.perm), L.P(zrc), L.P(self.group_start_c), L.P(ef), L.P(el),
               L.P(zr), L.P(oh), L.P(gs), L.stream())
        if self.permutations is not None and not isinstance(self.permutations, BlockPermutations):
            oh = self.permutations  # the caller's dense table, copied like hbp.py:237
        self._views.update(zero_row=zr, output_hash=oh, group_start=gs)

    @property
    def zero_row(self) -> torch.Tensor:
        """int32 [ncb * rows] (reference layout)."""
        self._expand()
        return self._views["zero_row"]

    @property
    def output_hash(self) -> torch.Tensor:
        """u32 bits in int32 [ncb * rows] (reference layout)."""
        self._expand()
        return self._views["output_hash"]

    @property
    def group_start(self) -> torch.Tensor:
        """int64 [ncb * gpc + 1] (reference layout)."""
        self._expand()
        return self._views["group_start"]

    def block_nnz_matrix(self) -> np.ndarray:
        """hbp.py:91-100: element count per block, from the compact group starts."""
        R, W = self.config.row_height, self.config.warp_size
        gpb = R // W
        gs = self.group_start_c.view(-1)
        per = (gs[gpb::gpb] - gs[:-1:gpb])[: self.nzb] if self.nzb else gs[:0]
        out = np.zeros(self.grid_shape, np.int64)
        out[self.blk_br.cpu().numpy(), self.blk_bc.cpu().numpy()] = per.cpu().numpy()
        return out

    def to_reference(self) -> dict:
        """The six reference arrays as numpy with the reference dtypes."""
        out = dict(col=self.col.cpu().numpy().view(np.uint32),
                   data=self.data.to(torch.float64).cpu().numpy(),
                   zero_row=self.zero_row.cpu().numpy(),
                   group_start=self.group_start.cpu().numpy(),
                   output_hash=self.output_hash.cpu().numpy().view(np.uint32))
        out["add_sign"] = self.add_sign.cpu().numpy() if self._add_sign is not None else None
        return out

    # ---- kernel descriptor
    def format_struct(self) -> L.FormatT:
        if self._fmt is None:
            f = L.FormatT()
            f.rows, f.cols = self.rows, self.cols
            f.col_width, f.row_height = self.config.col_width, self.config.row_height
            f.warp_size = self.config.warp_size
            f.nrb, f.ncb = self.grid_shape
            f.nzb, f.nnz = self.nzb, self.nnz
            f.dtype = L.dtype_code(self.data.dtype)
            f.exact = 1 if self.data.dtype == torch.float64 else 0
            for name, t in (("blk_br", self.blk_br), ("blk_bc", self.blk_bc),
                            ("slot_len", self.slot_len), ("perm", self.perm),
                            ("group_start", self.group_start_c), ("col", self.col),
                            ("data", self.data), ("rb_ptr", self.rb_ptr),
                            ("rb_blk", self.rb_blk)):
                setattr(f, name, t.data_ptr() if t.numel() else 0)
            if self.phases is not None:
                f.phase_ptr = self.phase_ptr.data_ptr()
                f.phases = self.phases.data_ptr()
            self._fmt = f
        return self._fmt

    def astype(self, dtype: torch.dtype) -> "HbpMatrix":
        """Same structure with values in another precision (f64 <-> f32)."""
        m = HbpMatrix(self.rows, self.cols, self.config, self.grid_shape, col=self.col,
                      data=_padded(self.data.to(dtype)), add_sign=self._add_sign, blk_br=self.blk_br,
                      blk_bc=self.blk_bc, slot_len=self.slot_len, perm=self.perm,
                      group_start_c=self.group_start_c, zero_row_c=self.zero_row_c,
                      rb_ptr=self.rb_ptr, rb_blk=self.rb_blk, permutations=self.permutations)
        m._views = self._views
        return m

    # ---- validation (hbp.py:102-135) on the reference-layout views
    def validate_structure(self) -> None:
        validate_reference_arrays(self.rows, self.cols, self.config, self.grid_shape,
                                  col=self.col, data=self.data, add_sign=self._add_sign,
                                  zero_row=self.zero_row, group_start=self.group_start,
                                  output_hash=self.output_hash)


def validate_reference_arrays(rows: int, cols: int, config: PartitionConfig, grid_shape, *,
                              col, data, add_sign, zero_row, group_start, output_hash) -> None:
    """hbp.py:102-135 validate_structure on the six reference-layout arrays
    (device tensors; add_sign may be None), in the reference's order: grid
    shape, element lengths, slot lengths, group_start length / span /
    monotonicity, add_sign domain, then block by block in bc-major order
    output_hash bijection before zero_row lane counts."""
    nrb, ncb = grid_shape
    R, W = config.row_height, config.warp_size
    if nrb != -(-rows // R) or ncb != -(-cols // config.col_width):
        raise HbpFormatError("grid shape inconsistent with dimensions")
    nnz = data.numel()
    if not (col.numel() == nnz and (add_sign is None or add_sign.numel() == nnz)):
        raise HbpFormatError("element array lengths differ")
    n_slots = ncb * rows
    if zero_row.numel() != n_slots or output_hash.numel() != n_slots:
        raise HbpFormatError("slot array length mismatch")
    n_groups = ncb * groups_per_col_block(rows, R, W)
    gs = group_start
    if gs.numel() != n_groups + 1:
        raise HbpFormatError("group_start length mismatch")
    ends = gs[[0, -1]].cpu().tolist()
    if ends[0] != 0 or ends[1] != nnz:
        raise HbpFormatError("group_start must span [0, nnz]")
    if bool((gs[1:] < gs[:-1]).any()):
        raise HbpFormatError("group_start must be non-decreasing")
    if add_sign is not None and nnz and bool(((add_sign < 1) & (add_sign != -1)).any()):
        raise HbpFormatError("add_sign entries must be >= 1 or -1")
    if not n_slots:
        return
    dev = zero_row.device
    # first block (bc-major key bc*nrb + br) whose output_hash is not a bijection
    bad = torch.full((1,), L.LLONG_MAX, dtype=torch.int64, device=dev)
    L.call("hbp_gather_dense_perm", L.P(output_hash), L.c_i64(rows), L.c_i64(ncb), L.c_i64(R),
           L.P(None), L.P(None), L.c_i64(0), L.P(None), L.P(bad), L.stream())
    b_perm = int(bad.item())
    # first block whose zero_row disagrees with its empty-slot mask, per W-lane group
    i = torch.arange(n_slots, device=dev)
    q = (i % rows) % R % W
    is_zero = (zero_row == -1).to(torch.int64)
    cs = torch.cumsum(is_zero, 0)
    g0 = i - q
    before = cs - is_zero - (cs[g0] - is_zero[g0])
    expected = torch.where(is_zero.bool(), torch.full_like(before, -1), before)
    wrong = torch.nonzero(expected != zero_row.to(torch.int64))
    b_zr = L.LLONG_MAX
    if wrong.numel():
        bc, r = divmod(int(wrong[0, 0]), rows)
        b_zr = bc * nrb + r // R
    if b_perm != L.LLONG_MAX and b_perm <= b_zr:
        bc, br = divmod(b_perm, nrb)
        raise HbpFormatError(f"output_hash of block ({br}, {bc}) is not a permutation")
    if b_zr != L.LLONG_MAX:
        bc, br = divmod(b_zr, nrb)
        raise HbpFormatError(f"zero_row of block ({br}, {bc}) has wrong lane counts")


def _bad_block_message(grid_or_hbp, idx: int, dense: bool, nrb: int) -> str:
    if dense:
        bc, br = divmod(idx, nrb)
    else:
        br = int(grid_or_hbp.blk_br[idx])
        bc = int(grid_or_hbp.blk_bc[idx])
    return f"permutation of block ({br}, {bc}) is not a bijection"


def build_hbp(csr: CsrMatrix, grid: BlockGrid, permutations, config: PartitionConfig | None = None,
              *, with_add_sign: bool = True, with_zero_row: bool = True) -> HbpMatrix:
    """hbp.py:150-238 on the GPU.

    permutations: a ``BlockPermutations`` (from hash_/sort_/identity_permutations)
    or any dense flat [ncb * rows] slot -> local-row table (numpy or tensor),
    validated block by block like hbp.py:179-181."""
    if config is None:
        config = grid.config
    elif config != grid.config:
        raise ValueError("config disagrees with the grid's config")
    if grid.rows != csr.rows or grid.cols != csr.cols or grid.nnz != csr.nnz:
        raise ValueError("grid does not describe this matrix")
    _check_gpu_geometry(config)
    dev = L.require_cuda()
    R, W = config.row_height, config.warp_size
    nrb, ncb, nzb = grid.num_row_blocks, grid.num_col_blocks, grid.nzb
    gpb = R // W
    s = L.stream()
    bad = torch.full((1,), L.LLONG_MAX, dtype=torch.int64, device=dev)

    keep = permutations
    if isinstance(permutations, BlockPermutations):
        if permutations.grid is not grid:
            permutations = np.asarray(permutations)
        else:
            perm = permutations.compact
    if not isinstance(permutations, BlockPermutations):
        dense = permutations
        if not isinstance(dense, torch.Tensor):
            dense = torch.as_tensor(np.ascontiguousarray(np.asarray(dense, np.uint32)).view(np.int32))
        dense = dense.to(device=dev, dtype=torch.int32).contiguous()
        if dense.numel() != ncb * grid.rows:
            raise ValueError("permutation table length mismatch")
        perm = torch.empty(nzb * R, dtype=torch.int32, device=dev)
        L.call("hbp_gather_dense_perm", L.P(dense), L.c_i64(grid.rows), L.c_i64(ncb), L.c_i64(R),
               L.P(grid.blk_br), L.P(grid.blk_bc), L.c_i64(nzb), L.P(perm), L.P(bad), s)
        b = int(bad.item())
        if b != L.LLONG_MAX:
            raise ValueError(_bad_block_message(grid, b, True, nrb))
        keep = dense

    slot_len = torch.empty(nzb * R, dtype=torch.int32, device=dev)
    zero_row_c = torch.empty(nzb * R, dtype=torch.int32, device=dev) if with_zero_row else None
    group_nnz = torch.empty(nzb * gpb + 1, dtype=torch.int64, device=dev)
    L.call("hbp_slot_lengths", L.P(grid.len_local), L.P(perm), L.P(grid.blk_br), L.c_i64(nzb),
           L.c_i64(grid.rows), L.c_i64(R), L.c_i64(W), L.P(slot_len), L.P(zero_row_c),
           L.P(group_nnz), L.P(bad), s)
    b = int(bad.item())
    if b != L.LLONG_MAX:
        raise ValueError(_bad_block_message(grid, b, False, nrb))
    group_start_c = L.exclusive_sum(group_nnz)
    if int(group_start_c[-1].item()) != csr.nnz:
        raise ValueError("emitted element count disagrees with matrix nnz")

    vdt = csr.values.dtype
    # padded by 16 elements: the streaming kernel's bulk copies may read up
    # to 15 bytes past the last element
    col = torch.zeros(csr.nnz + 16, dtype=torch.int32, device=dev)[:csr.nnz]
    data = torch.zeros(csr.nnz + 16, dtype=vdt, device=dev)[:csr.nnz]
    add = torch.empty(csr.nnz, dtype=torch.int32, device=dev) if with_add_sign else None
    L.call("hbp_emit", L.P(slot_len), L.P(perm), L.P(grid.start_local), L.P(group_start_c),
           L.P(grid.blk_br), L.c_i64(nzb), L.c_i64(grid.rows), L.c_i64(R), L.c_i64(W),
           L.P(csr.col_idx), L.P(csr.values), L.c_int(L.dtype_code(vdt)), L.P(col), L.P(data),
           L.P(add), s)

    rb_ptr, rb_blk = row_block_lists(grid.blk_br, nrb)
    return HbpMatrix(csr.rows, csr.cols, config, (nrb, ncb), col=col, data=data, add_sign=add,
                     blk_br=grid.blk_br, blk_bc=grid.blk_bc, slot_len=slot_len, perm=perm,
                     group_start_c=group_start_c, zero_row_c=zero_row_c, rb_ptr=rb_ptr,
                     rb_blk=rb_blk, permutations=keep)


def row_block_lists(blk_br: torch.Tensor, nrb: int):
    """Combine lists: rb_ptr[br] .. rb_ptr[br+1] index rb_blk, the nonzero
    blocks of row block br in ascending bc (stable sort of the bc-major
    directory by br)."""
    dev = blk_br.device
    nzb = blk_br.numel()
    rb_count = torch.zeros(nrb + 1, dtype=torch.int64, device=dev)
    L.call("hbp_row_block_counts", L.P(blk_br), L.c_i64(nzb), L.P(rb_count), L.stream())
    rb_ptr = L.exclusive_sum(rb_count)
    idx = torch.arange(nzb, dtype=torch.int32, device=dev)
    _, rb_blk = L.sort_pairs_u32(blk_br, idx, max(1, int(nrb - 1).bit_length()))
    return rb_ptr, rb_blk


def hbp_to_triplets(hbp: HbpMatrix) -> TripletMatrix:
    """hbp.py:241-315: invert the layout by walking every add_sign chain on
    the GPU (over the reference-layout arrays, so corruption is detected the
    way the reference detects it)."""
    dev = hbp.data.device
    nnz = hbp.nnz
    row = torch.full((nnz,), -1, dtype=torch.int64, device=dev)
    seen = torch.zeros(max(1, nnz), dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    c = hbp.config
    L.call("hbp_walk_chains", L.c_i64(hbp.rows), L.c_i64(hbp.cols), L.c_i64(c.col_width),
           L.c_i64(c.row_height), L.c_i64(c.warp_size), L.P(hbp.zero_row), L.P(hbp.output_hash),
           L.P(hbp.group_start), L.P(hbp.col), L.P(hbp.add_sign), L.c_i64(nnz), L.P(row),
           L.P(seen), L.P(err), L.stream())
    e = int(err.item())
    if e & 1:
        raise HbpFormatError("lane start offset outside its group region")
    if e & 2:
        raise HbpFormatError("element column outside its block's range")
    if e & 4:
        raise HbpFormatError("invalid add_sign stride")
    if e & 8:
        raise HbpFormatError("stride chain escapes its group region")
    if nnz:
        if int(seen.max().item()) > 1:
            raise HbpFormatError("element visited more than once")
        if int(seen[:nnz].sum().item()) != nnz:
            raise HbpFormatError("stride chains do not cover every element")
    return TripletMatrix(hbp.rows, hbp.cols, row, hbp.col.to(torch.int64) & 0xFFFFFFFF,
                         hbp.data.clone())


# ------------------------------------------------------------ .hbp codec
_ARRAY_SPECS = (("group_start", "<u8"), ("col", "<u4"), ("data", "<f8"), ("add_sign", "<i4"),
                ("zero_row", "<i4"), ("output_hash", "<u4"))


def serialize_hbp(hbp: HbpMatrix, stream) -> None:
    """hbp.py:328-339: the .hbp binary layout (little-endian, length-prefixed)."""
    ref = hbp.to_reference()
    stream.write(MAGIC)
    stream.write(struct.pack("<I", VERSION))
    stream.write(struct.pack("<8Q", hbp.rows, hbp.cols, hbp.nnz, hbp.config.col_width,
                             hbp.config.row_height, hbp.config.warp_size, hbp.num_row_blocks,
                             hbp.num_col_blocks))
    for name, dt in _ARRAY_SPECS:
        arr = np.ascontiguousarray(ref[name], dtype=dt)
        stream.write(struct.pack("<Q", arr.size))
        stream.write(arr.tobytes())


def _read_exact(stream, n: int) -> bytes:
    buf = stream.read(n)
    if len(buf) != n:
        raise HbpFormatError(f"truncated stream: wanted {n} bytes, got {len(buf)}")
    return buf


_TORCH_OF = {"<u8": torch.int64, "<u4": torch.int32, "<f8": torch.float64, "<i4": torch.int32}


def _dev_array(a, dt: str) -> torch.Tensor:
    """A reference array (numpy of codec type `dt`, or a tensor) as a
    contiguous device tensor of the same bits (u32 -> int32, u64 -> int64)."""
    tt = _TORCH_OF[dt]
    if isinstance(a, torch.Tensor):
        a = a.to(device=L.require_cuda())
        if a.dtype != tt:
            a = a.view(tt) if a.element_size() == torch.empty(0, dtype=tt).element_size() \
                and not a.is_floating_point() else a.to(tt)
        return a.contiguous()
    h = np.array(np.asarray(a, dt), copy=True)  # writable (frombuffer arrays are read-only)
    return torch.as_tensor(h.view({"<u8": np.int64, "<u4": np.int32}.get(dt, h.dtype)),
                           device=L.require_cuda()).contiguous()


def deserialize_hbp(stream) -> HbpMatrix:
    """hbp.py:349-381: read a .hbp stream into a device HbpMatrix.  The raw
    reference-layout arrays are validated first (hbp.py:102-135, same order
    and messages), then the compact runtime arrays are derived from them on
    the device."""
    if _read_exact(stream, 4) != MAGIC:
        raise HbpFormatError("bad magic; not an .hbp stream")
    (version,) = struct.unpack("<I", _read_exact(stream, 4))
    if version != VERSION:
        raise HbpFormatError(f"unsupported version {version}")
    rows, cols, nnz, C, R, W, nrb, ncb = struct.unpack("<8Q", _read_exact(stream, 64))
    arrays = {}
    for name, dt in _ARRAY_SPECS:
        (count,) = struct.unpack("<Q", _read_exact(stream, 8))
        arrays[name] = np.frombuffer(_read_exact(stream, count * np.dtype(dt).itemsize), dtype=dt)
    try:
        config = PartitionConfig(col_width=C, row_height=R, warp_size=W)
    except ValueError as exc:
        raise HbpFormatError(f"invalid partition config in header: {exc}") from exc
    if arrays["data"].size != nnz:
        raise HbpFormatError("element array length disagrees with header nnz")
    _check_gpu_geometry(config)
    t = {name: _dev_array(arrays[name], dt) for name, dt in _ARRAY_SPECS}
    rows, cols, grid_shape = int(rows), int(cols), (int(nrb), int(ncb))
    validate_reference_arrays(rows, cols, config, grid_shape, **t)
    return from_reference(rows, cols, config, grid_shape, **t)


def from_reference(rows, cols, config: PartitionConfig, grid_shape, *, col, data, add_sign,
                   zero_row, group_start, output_hash, dtype=torch.float64) -> HbpMatrix:
    """Build the device HbpMatrix from the reference's six dense arrays
    (numpy or device tensors; structure assumed valid -- see
    validate_reference_arrays).  Everything is derived on the device:
    nonzero blocks from group_start, the compact slot tables by gathers,
    slot lengths by walking the add_sign chains (hbp_chain_lengths)."""
    _check_gpu_geometry(config)
    dev = L.require_cuda()
    col, add_sign = _dev_array(col, "<u4"), _dev_array(add_sign, "<i4")
    zr, gs = _dev_array(zero_row, "<i4"), _dev_array(group_start, "<u8")
    oh = _dev_array(output_hash, "<u4")
    data = (data if isinstance(data, torch.Tensor) else torch.as_tensor(
        np.asarray(data, np.float64))).to(device=dev, dtype=dtype).contiguous()
    R, W, C = config.row_height, config.warp_size, config.col_width
    nrb, ncb = grid_shape
    gpb = R // W
    gpc = groups_per_col_block(rows, R, W)
    nnz = data.numel()
    # nonzero blocks (bc-major): their group range spans at least one element
    bc_i = torch.arange(ncb, device=dev).repeat_interleave(nrb)
    br_i = torch.arange(nrb, device=dev).repeat(ncb)
    first = bc_i * gpc + br_i * gpb
    n_b = torch.clamp(rows - br_i * R, max=R)
    ng_b = (n_b + W - 1) // W
    last = gs.numel() - 1
    nnz_b = gs[torch.clamp(first + ng_b, max=last)] - gs[torch.clamp(first, max=last)]
    nzmask = nnz_b > 0
    blk_bc = bc_i[nzmask].to(torch.int32)
    blk_br = br_i[nzmask].to(torch.int32)
    nzb = blk_br.numel()
    # compact slot tables: slot s of nonzero block i is dense slot bc*rows + br*R + s
    s_loc = torch.arange(R, device=dev)
    base = (blk_bc.to(torch.int64) * rows + blk_br.to(torch.int64) * R)[:, None] + s_loc
    valid = (blk_br.to(torch.int64)[:, None] * R + s_loc) < rows
    base_c = torch.where(valid, base, torch.zeros_like(base))
    dense_len = torch.empty(ncb * rows, dtype=torch.int32, device=dev)
    L.call("hbp_chain_lengths", L.c_i64(rows), L.c_i64(cols), L.c_i64(C), L.c_i64(R),
           L.c_i64(W), L.P(zr), L.P(gs), L.P(add_sign), L.c_i64(nnz), L.P(dense_len), L.stream())
    zero_i = torch.zeros((), dtype=torch.int32, device=dev)
    perm = torch.where(valid, oh[base_c], zero_i).reshape(-1).contiguous()
    zrc = torch.where(valid, zr[base_c], torch.full((), -1, dtype=torch.int32,
                                                     device=dev)).reshape(-1).contiguous()
    slot_len = torch.where(valid, dense_len[base_c], zero_i).reshape(-1).contiguous()
    # compact group starts: group g of block i is dense group bc*gpc + br*gpb + g;
    # groups past the block's last one repeat its end
    g_loc = torch.arange(gpb, device=dev)
    g0 = (blk_bc.to(torch.int64) * gpc + blk_br.to(torch.int64) * gpb)[:, None]
    ngi = ((torch.clamp(rows - blk_br.to(torch.int64) * R, max=R) + W - 1) // W)[:, None]
    gsc = torch.empty(nzb * gpb + 1, dtype=torch.int64, device=dev)
    gsc[:-1] = gs[g0 + torch.minimum(g_loc, ngi)].reshape(-1)
    gsc[-1] = nnz
    rb_ptr, rb_blk = row_block_lists(blk_br, nrb)
    return HbpMatrix(rows, cols, config, grid_shape,
                     col=_padded(col), data=_padded(data), add_sign=add_sign,
                     blk_br=blk_br, blk_bc=blk_bc, slot_len=slot_len, perm=perm,
                     group_start_c=gsc, zero_row_c=zrc, rb_ptr=rb_ptr, rb_blk=rb_blk,
                     permutations=oh)


def save_hbp(hbp: HbpMatrix, path) -> None:
    with open(path, "wb") as fh:
        serialize_hbp(hbp, fh)


def load_hbp(path) -> HbpMatrix:
    with open(path, "rb") as fh:
        return deserialize_hbp(fh)


def serialize_bytes(hbp: HbpMatrix) -> bytes:
    buf = io.BytesIO()
    serialize_hbp(hbp, buf)
    return buf.getvalue()
