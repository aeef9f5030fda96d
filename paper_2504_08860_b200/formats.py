"""COO / CSR containers and the GPU COO -> CSR conversion.

Mirrors the reference's formats (/root/reference/pkg/src/hbp_spmv/formats.py):
``TripletMatrix`` (:52-97), ``CsrMatrix`` (:100-121), ``coo_to_csr``
(:243-258), ``csr_to_triplets`` (:261-263).  Arrays live on the CUDA device as
torch tensors.  Values keep float32 when given float32 (the B200 fp32 path);
anything else is coerced to float64 like the reference (:67-70, :114-117).
Column indices are stored as int32 on the device (the HBP ``col`` array is
u32 in the reference too, hbp.py:57).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np
import torch

from . import _lib as L

__all__ = ["TripletMatrix", "CsrMatrix", "coo_to_csr", "csr_to_triplets", "as_device_values",
           "csr_spmv", "dense_oracle_spmv", "to_dense"]


def _dev(a, dtype: torch.dtype) -> torch.Tensor:
    dev = L.require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), device=dev).to(dtype)


def _value_dtype(a) -> torch.dtype:
    if isinstance(a, torch.Tensor):
        return torch.float32 if a.dtype == torch.float32 else torch.float64
    return torch.float32 if np.asarray(a).dtype == np.float32 else torch.float64


def as_device_values(a, dtype: torch.dtype | None = None) -> torch.Tensor:
    return _dev(a, dtype or _value_dtype(a))


@dataclass(frozen=True)
class TripletMatrix:
    """Coordinate-format sparse matrix (formats.py:52-97), device-resident."""

    rows: int
    cols: int
    row: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor

    def __post_init__(self):
        vdt = _value_dtype(self.val)
        object.__setattr__(self, "row", _dev(self.row, torch.int64))
        object.__setattr__(self, "col", _dev(self.col, torch.int64))
        object.__setattr__(self, "val", _dev(self.val, vdt))
        if not (self.row.shape == self.col.shape == self.val.shape) or self.row.dim() != 1:
            raise ValueError("entry arrays must have equal length")
        if self.row.numel():
            lo = torch.stack([self.row.min(), self.col.min()]).cpu()
            hi = torch.stack([self.row.max(), self.col.max()]).cpu()
            if lo[0] < 0 or hi[0] >= self.rows:
                raise ValueError("row index out of bounds")
            if lo[1] < 0 or hi[1] >= self.cols:
                raise ValueError("column index out of bounds")

    @property
    def nnz(self) -> int:
        return self.val.numel()

    def entries(self) -> Iterator[tuple[int, int, float]]:
        for r, c, v in zip(self.row.tolist(), self.col.tolist(), self.val.tolist()):
            yield int(r), int(c), float(v)

    def _sorted_keys(self):
        """Stable sort of key = row*cols + col (np.lexsort((col, row)) order)."""
        keys = self.row * self.cols + self.col
        order = torch.arange(self.nnz, dtype=torch.int64, device=keys.device)
        bits = max(1, int(self.rows * self.cols - 1).bit_length())
        return L.sort_pairs_u64(keys, order, bits)

    def canonicalized(self) -> "TripletMatrix":
        """formats.py:87-97: sort by (row, col), duplicates summed like
        np.add.reduceat (first element + numpy pairwise sum of the rest)."""
        if self.nnz == 0:
            return self
        skeys, order = self._sorted_keys()
        head = torch.empty(self.nnz, dtype=torch.int64, device=skeys.device)
        L.call("hbp_coo_run_heads", L.P(skeys), L.c_i64(self.nnz), L.P(head), L.stream())
        incl = L.inclusive_sum(head)
        m = int(incl[-1].item())
        dev = skeys.device
        r = torch.empty(m, dtype=torch.int64, device=dev)
        c = torch.empty(m, dtype=torch.int64, device=dev)
        v = torch.empty(m, dtype=torch.float64, device=dev)
        v64 = self.val.to(torch.float64).contiguous()
        L.call("hbp_coo_reduce_runs", L.P(skeys), L.P(order), L.P(v64), L.P(incl),
               L.c_i64(self.nnz), L.c_i64(self.cols), L.P(r), L.P(c), L.P(v), L.stream())
        return TripletMatrix(self.rows, self.cols, r, c, v.to(self.val.dtype))

    def to_numpy(self):
        return (self.row.cpu().numpy(), self.col.cpu().numpy(),
                self.val.to(torch.float64).cpu().numpy())


@dataclass(frozen=True)
class CsrMatrix:
    """Compressed sparse row matrix (formats.py:100-121), device-resident:
    row_ptr int64[rows+1], col_idx int32[nnz], values float32/float64[nnz]."""

    rows: int
    cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    values: torch.Tensor

    def __post_init__(self):
        vdt = _value_dtype(self.values)
        object.__setattr__(self, "row_ptr", _dev(self.row_ptr, torch.int64))
        object.__setattr__(self, "col_idx", _dev(self.col_idx, torch.int32))
        object.__setattr__(self, "values", _dev(self.values, vdt))
        if self.cols >= 2 ** 31:
            raise ValueError("cols must fit in int32 on the GPU path")

    @property
    def nnz(self) -> int:
        return self.values.numel()

    @property
    def dtype(self) -> torch.dtype:
        return self.values.dtype

    def astype(self, dtype: torch.dtype) -> "CsrMatrix":
        return CsrMatrix(self.rows, self.cols, self.row_ptr, self.col_idx, self.values.to(dtype))


def coo_to_csr(matrix: TripletMatrix) -> CsrMatrix:
    """formats.py:243-258: lexsort (row, col) on the GPU (stable radix sort of
    row*cols + col), reject duplicates, row_ptr by binary search."""
    dev = L.require_cuda()
    nnz = matrix.nnz
    vdt = matrix.val.dtype
    row_ptr = torch.empty(matrix.rows + 1, dtype=torch.int64, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=vdt, device=dev)
    dup = torch.zeros(1, dtype=torch.int32, device=dev)
    if nnz:
        skeys, order = matrix._sorted_keys()
    else:
        skeys = order = torch.empty(0, dtype=torch.int64, device=dev)
    L.call("hbp_coo_finish_csr", L.P(skeys), L.P(order), L.P(matrix.val), L.c_i64(nnz),
           L.c_i64(matrix.rows), L.c_i64(matrix.cols), L.c_int(L.dtype_code(vdt)), L.P(row_ptr),
           L.P(col), L.P(val), L.P(dup), L.stream())
    if int(dup.item()):
        raise ValueError("duplicate (row, col) entries; canonicalize first")
    return CsrMatrix(matrix.rows, matrix.cols, row_ptr, col, val)


def csr_spmv(csr: CsrMatrix, x) -> torch.Tensor:
    """formats.py:266-273 / _kernels.py:13-19 (PAPER Alg. 1) on the GPU: one
    thread per row, left to right in storage order (hbp_csr_spmv)."""
    if isinstance(x, torch.Tensor):
        xt = x
    else:
        xt = torch.as_tensor(np.asarray(x))
    if tuple(xt.shape) != (csr.cols,):
        raise ValueError(f"vector length {tuple(xt.shape)} != cols {csr.cols}")
    xt = xt.to(device=csr.values.device, dtype=csr.values.dtype).contiguous()
    y = torch.empty(csr.rows, dtype=csr.values.dtype, device=csr.values.device)
    L.call("hbp_csr_spmv", L.P(csr.row_ptr), L.P(csr.col_idx), L.P(csr.values),
           L.c_int(L.dtype_code(csr.values.dtype)), L.c_i64(csr.rows), L.P(xt), L.P(y),
           L.stream())
    return y


def csr_to_triplets(csr: CsrMatrix) -> TripletMatrix:
    """formats.py:261-263."""
    counts = csr.row_ptr[1:] - csr.row_ptr[:-1]
    row = torch.repeat_interleave(torch.arange(csr.rows, device=counts.device), counts)
    return TripletMatrix(csr.rows, csr.cols, row, csr.col_idx.to(torch.int64), csr.values.clone())


def _host_triplets(matrix):
    if isinstance(matrix, TripletMatrix):
        return matrix.to_numpy()
    return (np.asarray(matrix.row, np.int64), np.asarray(matrix.col, np.int64),
            np.asarray(matrix.val, np.float64))


def dense_oracle_spmv(matrix: TripletMatrix, x) -> np.ndarray:
    """formats.py:276-284: brute-force y = A x in entry order (np.add.at),
    independent of every kernel; a host verification utility like the
    reference's, not an SpMV path of this package."""
    x = np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x, dtype=np.float64)
    if x.shape != (matrix.cols,):
        raise ValueError(f"vector length {x.shape} != cols {matrix.cols}")
    r, c, v = _host_triplets(matrix)
    y = np.zeros(matrix.rows, dtype=np.float64)
    np.add.at(y, r, v * x[c])
    return y


def to_dense(matrix: TripletMatrix) -> np.ndarray:
    """formats.py:287-290 (host array, duplicates summed in entry order)."""
    r, c, v = _host_triplets(matrix)
    dense = np.zeros((matrix.rows, matrix.cols), dtype=np.float64)
    np.add.at(dense, (r, c), v)
    return dense
