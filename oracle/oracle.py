"""CPU oracle for the HBP SpMV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker or the timed CPU baseline.  The product package
``paper_2504_08860_b200`` never imports it and has no CPU fallback.

It restates the reference package (``/root/reference/pkg/src/hbp_spmv``) in
numpy plus the plain-C loops in ``hbp_oracle.c`` and works in the reference's
DENSE layout (rows x column-blocks slot arrays).  Each function cites the
reference file:line it follows.  Parity of this restatement with the reference
itself is pinned by ``tests/test_oracle_golden.py`` against the golden vectors
in ``tests/golden/`` that ``tests/golden/make_golden.py`` produced by running
the reference in the build container.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
BUCKET_MAX = 8  # reorder.py:37

_lib = None


def build(force: bool = False) -> str:
    """Compile hbp_oracle.c -> oracle/build/liboracle.so (gcc, -ffp-contract=off)."""
    src = os.path.join(HERE, "hbp_oracle.c")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= os.path.getmtime(src)):
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.orc_hash_perm.restype = ctypes.c_uint64
        _lib.orc_hash_perm_block.restype = ctypes.c_uint64
        _lib.orc_build_hbp.restype = ctypes.c_int
        _lib.orc_run_spmv.restype = ctypes.c_int
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


I64 = ctypes.c_int64


# --------------------------------------------------------------- formats
def coo_to_csr(rows, cols, row, col, val):
    """formats.py:243-258: lexsort (row, col); reject duplicates; bincount row_ptr."""
    row = np.asarray(row, np.int64)
    col = np.asarray(col, np.int64)
    val = np.asarray(val, np.float64)
    order = np.lexsort((col, row))
    row, col, val = row[order], col[order], val[order]
    if row.size and ((row[1:] == row[:-1]) & (col[1:] == col[:-1])).any():
        raise ValueError("duplicate (row, col) entries; canonicalize first")
    counts = np.bincount(row, minlength=rows)
    row_ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    return row_ptr, col, val


def canonicalize(rows, cols, row, col, val):
    """formats.py:87-97: sort by (row, col), sum duplicates."""
    row = np.asarray(row, np.int64)
    col = np.asarray(col, np.int64)
    val = np.asarray(val, np.float64)
    if row.size == 0:
        return row, col, val
    order = np.lexsort((col, row))
    r, c, v = row[order], col[order], val[order]
    key = r * cols + c
    first = np.concatenate(([True], key[1:] != key[:-1]))
    starts = np.flatnonzero(first)
    return r[starts], c[starts], np.add.reduceat(v, starts)


def csr_spmv(row_ptr, col_idx, values, x):
    """formats.py:266-273 -> _kernels.py:13-19 (C restatement)."""
    rows = row_ptr.size - 1
    out = np.zeros(rows)
    lib().orc_csr_kernel(_p(np.ascontiguousarray(row_ptr, np.int64)),
                         _p(np.ascontiguousarray(col_idx, np.int64)),
                         _p(np.ascontiguousarray(values, np.float64)),
                         _p(np.ascontiguousarray(x, np.float64)), _p(out), I64(rows))
    return out


def rows_blocked(row_ptr, col_idx, values, x, C, rows_sel):
    """y[rows_sel] as the reference computes it (hbp_block_kernel per column
    block, _kernels.py:22-47, then combine in ascending bc, engine.py:196-201)
    without the dense layout: CSR rows with C-wide column blocks (C
    restatement, orc_rows_blocked).  row_ptr / col_idx / values may be the
    CSR of just the selected rows' neighbourhood as long as rows_sel indexes
    into row_ptr."""
    sel = np.ascontiguousarray(rows_sel, np.int64)
    out = np.zeros(sel.size)
    lib().orc_rows_blocked(_p(np.ascontiguousarray(row_ptr, np.int64)),
                           _p(np.ascontiguousarray(col_idx, np.int64)),
                           _p(np.ascontiguousarray(values, np.float64)),
                           _p(np.ascontiguousarray(x, np.float64)), I64(C), _p(sel),
                           I64(sel.size), _p(out))
    return out


def dense_oracle_spmv(rows, row, col, val, x):
    """formats.py:276-283: np.add.at brute force."""
    y = np.zeros(rows)
    np.add.at(y, np.asarray(row, np.int64), np.asarray(val) * np.asarray(x)[col])
    return y


def componentwise_error(rows, row, col, val, x, y):
    """test_acceptance.py:112-123: |y - o| / (|A||x|)_i, exact zero where scale is 0."""
    o = dense_oracle_spmv(rows, row, col, val, x)
    scale = dense_oracle_spmv(rows, row, col, np.abs(val), np.abs(x))
    err = np.abs(np.asarray(y, np.float64) - o)
    if np.any(err[scale == 0.0] != 0.0):
        return np.inf
    live = scale > 0
    return float((err[live] / scale[live]).max()) if live.any() else 0.0


# ------------------------------------------------------------- partition
def geometry(rows, cols, C, R, W):
    """partition.py:43-55."""
    nrb = -(-rows // R)
    ncb = -(-cols // C)
    last = rows - (nrb - 1) * R
    gpc = (nrb - 1) * (R // W) + -(-last // W)
    return nrb, ncb, gpc


@dataclass
class DenseGrid:
    rows: int
    cols: int
    C: int
    R: int
    W: int
    nrb: int
    ncb: int
    row_counts: np.ndarray      # i32 [ncb, rows]
    row_starts: np.ndarray      # i64 [ncb, rows]
    block_nnz: np.ndarray       # i64 [nrb, ncb]
    block_elem_start: np.ndarray  # i64 [nrb, ncb]
    nnz: int


def make_grid(row_ptr, col_idx, rows, cols, C, R, W) -> DenseGrid:
    """partition.py:100-127: split each row run at multiples of C."""
    if rows < 1 or cols < 1:
        raise ValueError("matrix must have nonempty dimensions")
    nrb, ncb, _ = geometry(rows, cols, C, R, W)
    row_of = np.repeat(np.arange(rows, dtype=np.int64), np.diff(row_ptr))
    counts = np.bincount((col_idx // C) * rows + row_of, minlength=ncb * rows)
    row_counts = counts.reshape(ncb, rows).astype(np.int32)
    row_starts = row_ptr[:-1][None, :] + (
        np.cumsum(row_counts, axis=0, dtype=np.int64) - row_counts)
    padded = np.zeros((ncb, nrb * R), np.int64)
    padded[:, :rows] = row_counts
    block_nnz = padded.reshape(ncb, nrb, R).sum(axis=2).T
    flat = block_nnz.T.ravel()
    starts = np.concatenate(([0], np.cumsum(flat)[:-1])).astype(np.int64)
    return DenseGrid(rows, cols, C, R, W, nrb, ncb, row_counts, row_starts,
                     np.ascontiguousarray(block_nnz),
                     np.ascontiguousarray(starts.reshape(ncb, nrb).T),
                     int(row_ptr[-1]))


# --------------------------------------------------------------- reorder
def quantile_inverted_cdf(v, q):
    """np.quantile(..., method='inverted_cdf') == sorted(v)[ceil(q n) - 1]."""
    s = np.sort(np.asarray(v))
    k = max(1, math.ceil(q * s.size))
    return s[k - 1]


def params_from_sample(sample, R, quantile=0.9):
    """reorder.py:87-103: a = smallest shift with quantile(sample >> a) <= 8;
    b = d = max(1, R // 9); c = smallest value >= ceil(modal / b), >= 1,
    co-prime with b."""
    sample = np.asarray(sample, np.int64)
    b = max(1, R // (BUCKET_MAX + 1))
    a = 0
    if sample.size:
        while quantile_inverted_cdf(sample >> a, quantile) > BUCKET_MAX:
            a += 1
        modal = int(np.bincount(np.minimum(sample >> a, BUCKET_MAX),
                                minlength=BUCKET_MAX + 1).max())
    else:
        modal = 0
    c = max(1, -(-modal // b))
    while math.gcd(c, b) != 1:
        c += 1
    return a, b, c, b


def sample_indices(population, sample_size=4096, seed=0):
    """reorder.py:80-85: indices drawn by default_rng(seed).choice(..., replace=False);
    None means 'the whole population'."""
    if sample_size < population:
        return np.random.default_rng(seed).choice(population, sample_size, replace=False)
    return None


def sample_hash_params(grid: DenseGrid, sample_size=4096, seed=0, quantile=0.9):
    pop = grid.row_counts.reshape(-1)
    idx = sample_indices(pop.size, sample_size, seed)
    sample = pop if idx is None else pop[idx]
    return params_from_sample(sample, grid.R, quantile)


def hash_slot(nnz, r, a, b, c, d, bmax=BUCKET_MAX):
    """reorder.py:106-109."""
    return min(nnz >> a, bmax) * b + (r * c) % d


def hash_perm_block(row_nnz, a, b, c, d, bmax=BUCKET_MAX):
    """reorder.py:112-136 (C restatement). Returns (perm u32[n], probes)."""
    row_nnz = np.ascontiguousarray(row_nnz, np.int32)
    out = np.empty(row_nnz.size, np.uint32)
    probes = lib().orc_hash_perm_block(_p(row_nnz), I64(row_nnz.size), I64(a), I64(b),
                                       I64(c), I64(d), I64(bmax), _p(out))
    return out, int(probes)


def hash_permutations(grid: DenseGrid, params):
    """reorder.py:174-184 -> _kernels.py:62-92 (C restatement). Returns (perms, probes)."""
    a, b, c, d = params
    out = np.empty(grid.ncb * grid.rows, np.uint32)
    rc = np.ascontiguousarray(grid.row_counts.reshape(-1), np.int32)
    probes = lib().orc_hash_perm(_p(rc), I64(grid.rows), I64(grid.R), I64(grid.nrb),
                                 I64(grid.ncb), I64(a), I64(b), I64(c), I64(d),
                                 I64(BUCKET_MAX), _p(out))
    return out, int(probes)


def identity_permutations(grid: DenseGrid):
    """reorder.py:222-225."""
    return np.tile((np.arange(grid.rows, dtype=np.uint32) % grid.R), grid.ncb)


def sort_permutation(row_nnz):
    """reorder.py:160-171 fast path: stable ascending-nnz order."""
    return np.argsort(np.asarray(row_nnz), kind="stable").astype(np.uint32)


def counting_merge_sort(row_nnz):
    """reorder.py:139-171 counter path: top-down merge sort split at len//2,
    merged with `key[left] <= key[right]`, one comparison per step of the
    merge loop.  Returns (perm u32[n], comparisons)."""
    key = np.asarray(row_nnz)
    count = [0]

    def msort(idx):
        if len(idx) <= 1:
            return idx
        mid = len(idx) // 2
        left, right = msort(idx[:mid]), msort(idx[mid:])
        out, i, j = [], 0, 0
        while i < len(left) and j < len(right):
            count[0] += 1
            if key[left[i]] <= key[right[j]]:
                out.append(left[i])
                i += 1
            else:
                out.append(right[j])
                j += 1
        return out + left[i:] + right[j:]

    order = msort(list(range(key.size)))
    return np.asarray(order, dtype=np.uint32), count[0]


def sort_permutations(grid: DenseGrid):
    """reorder.py:187-219: per block stable sort by nnz."""
    out = np.empty(grid.ncb * grid.rows, np.uint32)
    for bc in range(grid.ncb):
        for br in range(grid.nrb):
            r0 = br * grid.R
            n = min(grid.R, grid.rows - r0)
            out[bc * grid.rows + r0: bc * grid.rows + r0 + n] = sort_permutation(
                grid.row_counts[bc, r0:r0 + n])
    return out


# ------------------------------------------------------------------- hbp
def zero_row_for(is_zero, W):
    """hbp.py:138-147."""
    is_zero = np.asarray(is_zero, bool)
    n = is_zero.size
    ng = -(-n // W) if n else 0
    padded = np.zeros(ng * W, np.int64)
    padded[:n] = is_zero
    within = (np.cumsum(padded.reshape(ng, W), axis=1) - padded.reshape(ng, W)).reshape(-1)[:n]
    return np.where(is_zero, -1, within).astype(np.int32)


@dataclass
class DenseHbp:
    rows: int
    cols: int
    C: int
    R: int
    W: int
    nrb: int
    ncb: int
    col: np.ndarray
    data: np.ndarray
    add_sign: np.ndarray
    zero_row: np.ndarray
    group_start: np.ndarray
    output_hash: np.ndarray

    @property
    def nnz(self):
        return self.data.size

    def block_nnz_matrix(self):
        """hbp.py:91-100."""
        _, _, gpc = geometry(self.rows, self.cols, self.C, self.R, self.W)
        out = np.empty((self.nrb, self.ncb), np.int64)
        for bc in range(self.ncb):
            for br in range(self.nrb):
                gb = bc * gpc + br * (self.R // self.W)
                ng = -(-min(self.R, self.rows - br * self.R) // self.W)
                out[br, bc] = self.group_start[gb + ng] - self.group_start[gb]
        return out


def build_hbp(row_ptr, col_idx, values, grid: DenseGrid, perms) -> DenseHbp:
    """hbp.py:150-238 (per-block loop restated in C)."""
    nnz = grid.nnz
    perms = np.ascontiguousarray(perms, np.uint32)
    if perms.size != grid.ncb * grid.rows:
        raise ValueError("permutation table length mismatch")
    _, _, gpc = geometry(grid.rows, grid.cols, grid.C, grid.R, grid.W)
    col = np.empty(nnz, np.uint32)
    data = np.empty(nnz, np.float64)
    add = np.empty(nnz, np.int32)
    zr = np.empty(grid.ncb * grid.rows, np.int32)
    gs = np.empty(grid.ncb * gpc + 1, np.int64)
    bad = np.zeros(2, np.int64)
    rc = lib().orc_build_hbp(
        _p(np.ascontiguousarray(col_idx, np.int64)), _p(np.ascontiguousarray(values, np.float64)),
        _p(np.ascontiguousarray(grid.row_counts, np.int32)),
        _p(np.ascontiguousarray(grid.row_starts, np.int64)),
        _p(np.ascontiguousarray(grid.block_elem_start, np.int64)), _p(perms),
        I64(grid.rows), I64(nnz), I64(grid.R), I64(grid.W), I64(grid.nrb), I64(grid.ncb),
        _p(col), _p(data), _p(add), _p(zr), _p(gs), _p(bad))
    if rc == 1:
        raise ValueError(f"permutation of block ({bad[0]}, {bad[1]}) is not a bijection")
    if rc == 2:
        raise ValueError("emitted element count disagrees with matrix nnz")
    if rc != 0:
        raise MemoryError("oracle build failed")
    return DenseHbp(grid.rows, grid.cols, grid.C, grid.R, grid.W, grid.nrb, grid.ncb,
                    col, data, add, zr, gs, perms.copy())


def hbp_to_triplets(h: DenseHbp):
    """hbp.py:241-315: walk every stride chain; returns (row, col, val) in walk order."""
    _, _, gpc = geometry(h.rows, h.cols, h.C, h.R, h.W)
    rows_out, cols_out, vals_out = [], [], []
    seen = np.zeros(h.nnz, np.int32)
    for bc in range(h.ncb):
        for br in range(h.nrb):
            n = min(h.R, h.rows - br * h.R)
            base = bc * h.rows + br * h.R
            gb = bc * gpc + br * (h.R // h.W)
            for s in range(n):
                zr = int(h.zero_row[base + s])
                if zr < 0:
                    continue
                g, q = divmod(s, h.W)
                end = h.group_start[gb + g + 1]
                j = int(h.group_start[gb + g]) + q - zr
                r = br * h.R + int(h.output_hash[base + s])
                while True:
                    if not (bc * h.C <= h.col[j] < min((bc + 1) * h.C, h.cols)):
                        raise ValueError("element column outside its block's range")
                    seen[j] += 1
                    rows_out.append(r)
                    cols_out.append(int(h.col[j]))
                    vals_out.append(h.data[j])
                    step = int(h.add_sign[j])
                    if step == 0 or (step < 0 and step != -1):
                        raise ValueError("invalid add_sign stride")
                    if step < 0:
                        break
                    j += step
                    if j >= end:
                        raise ValueError("stride chain escapes its group region")
    if (seen != 1).any():
        raise ValueError("stride chains do not cover every element exactly once")
    return (np.asarray(rows_out, np.int64), np.asarray(cols_out, np.int64),
            np.asarray(vals_out, np.float64))


# ---------------------------------------------------------------- engine
def nonzero_blocks(block_nnz):
    """engine.py:86-93: (br, bc) of nonzero blocks in bc-major order."""
    pairs = np.argwhere(np.asarray(block_nnz).T > 0)
    return np.ascontiguousarray(pairs[:, ::-1]).astype(np.int32)


def plan_execution(block_nnz, fixed_fraction, workers):
    """engine.py:96-115. Returns (block_order, fixed_count, worker_ranges)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    order = nonzero_blocks(block_nnz)
    fixed = int(fixed_fraction * len(order) + 0.5)
    base, rem = divmod(fixed, workers)
    ranges, s = [], 0
    for w in range(workers):
        size = base + (1 if w < rem else 0)
        ranges.append((s, s + size))
        s += size
    return order, fixed, tuple(ranges)


def run_spmv(h: DenseHbp, x, plan, workers, with_log=False):
    """engine.py:179-193 + _run_plan (engine.py:137-176), C restatement with
    pthreads. Returns (partial f64[ncb*rows], log or None)."""
    order, fixed, ranges = plan
    if workers != len(ranges):
        raise ValueError("plan was built for a different worker count")
    x = np.ascontiguousarray(x, np.float64)
    if x.shape != (h.cols,):
        raise ValueError(f"vector length {x.shape} != cols {h.cols}")
    partial = np.empty(h.ncb * h.rows)
    n = len(order)
    log = None
    if with_log:
        log = dict(worker=np.full(n, -1, np.int32), kind=np.full(n, -1, np.int8),
                   start_ns=np.zeros(n, np.int64), end_ns=np.zeros(n, np.int64))
    rng = np.ascontiguousarray(np.asarray(ranges, np.int64).reshape(-1, 2))
    rc = lib().orc_run_spmv(
        _p(h.col), _p(h.data), _p(h.add_sign), _p(h.zero_row), _p(h.output_hash),
        _p(h.group_start), I64(h.rows), I64(h.cols), I64(h.C), I64(h.R), I64(h.W),
        I64(h.nrb), I64(h.ncb), _p(np.ascontiguousarray(order, np.int32)), I64(n),
        I64(fixed), _p(rng), I64(workers), _p(x), _p(partial),
        _p(log["worker"] if log else None), _p(log["kind"] if log else None),
        _p(log["start_ns"] if log else None), _p(log["end_ns"] if log else None))
    if rc != 0:
        raise ValueError("workers must be >= 1")
    return partial, log


def combine(partial, rows, ncb):
    """engine.py:196-201."""
    out = np.empty(rows)
    lib().orc_combine(_p(np.ascontiguousarray(partial, np.float64)), I64(rows), I64(ncb), _p(out))
    return out


def hbp_spmv(h: DenseHbp, x, workers=1, fixed_fraction=0.7):
    """engine.py:228-232."""
    plan = plan_execution(h.block_nnz_matrix(), fixed_fraction, workers)
    partial, _ = run_spmv(h, x, plan, workers)
    return combine(partial, h.rows, h.ncb)


# --------------------------------------------------------------- pipeline
def pipeline(rows, cols, row, col, val, C, R, W, seed=0, sample_size=4096, quantile=0.9,
             ordering="hash"):
    """The reference's documented flow (pkg/README.md:34-39; __init__.py:1-12)."""
    row_ptr, col_idx, values = coo_to_csr(rows, cols, row, col, val)
    grid = make_grid(row_ptr, col_idx, rows, cols, C, R, W)
    params = sample_hash_params(grid, sample_size, seed, quantile)
    if ordering == "hash":
        perms, probes = hash_permutations(grid, params)
    elif ordering == "identity":
        perms, probes = identity_permutations(grid), 0
    else:
        perms, probes = sort_permutations(grid), 0
    h = build_hbp(row_ptr, col_idx, values, grid, perms)
    return dict(row_ptr=row_ptr, col_idx=col_idx, values=values, grid=grid,
                params=params, perms=perms, probes=probes, hbp=h)


def block2d_spmv_baseline(row_ptr, col_idx, values, grid: DenseGrid, x):
    """engine.py:204-225 -> _kernels.py:50-59 (C restatement) + combine."""
    partial = np.empty(grid.ncb * grid.rows)
    lib().orc_block2d(_p(np.ascontiguousarray(col_idx, np.int64)),
                      _p(np.ascontiguousarray(values, np.float64)),
                      _p(np.ascontiguousarray(grid.row_counts, np.int32)),
                      _p(np.ascontiguousarray(grid.row_starts, np.int64)),
                      _p(np.ascontiguousarray(grid.block_nnz, np.int64)), I64(grid.rows),
                      I64(grid.R), I64(grid.nrb), I64(grid.ncb),
                      _p(np.ascontiguousarray(x, np.float64)), _p(partial))
    return combine(partial, grid.rows, grid.ncb)
