"""Synthetic benchmark inputs -- bench/test harness, not product.

The reference package ships only uniform/powerlaw generators (synth.py); the
benchmark configs also need R-MAT, banded and Laplacian matrices, generated
here directly as CSR.  GPU versions use torch ops (input generation is not
timed and not part of the HBP path); CPU (numpy) versions feed the reference
arm's bounded samples.
"""
from __future__ import annotations

import numpy as np

GRAPH500 = (0.57, 0.19, 0.19)  # a, b, c (d = 0.05)


def rmat_csr_torch(scale: int, edge_factor: int, seed: int, device, value_dtype,
                   permute: bool = True):
    """Graph500-style R-MAT: 2^scale vertices, edge_factor * 2^scale generated
    edges, quadrant probabilities (0.57, 0.19, 0.19, 0.05), random vertex
    relabeling, duplicates removed; values uniform(-1, 1).  Returns
    (rows, cols, row_ptr int64, col int32, val) on `device`."""
    import torch
    n = 1 << scale
    m = edge_factor * n
    a, b, c = GRAPH500
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    row = torch.zeros(m, dtype=torch.int64, device=device)
    col = torch.zeros(m, dtype=torch.int64, device=device)
    chunk = 1 << 26
    for lvl in range(scale):
        for s in range(0, m, chunk):
            e = min(m, s + chunk)
            r = torch.rand(e - s, generator=g, device=device)
            rb = r >= (a + b)
            cb = ((r >= a) & (r < a + b)) | (r >= a + b + c)
            row[s:e] = row[s:e] * 2 + rb
            col[s:e] = col[s:e] * 2 + cb
        del r, rb, cb
    if permute:
        perm = torch.randperm(n, generator=g, device=device)
        row = perm[row]
        col = perm[col]
        del perm
    key = row * n + col
    del row, col
    key = torch.unique(key, sorted=True)
    row = key // n
    col = (key % n).to(torch.int32)
    del key
    counts = torch.bincount(row, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    del row, counts
    val = (torch.rand(col.numel(), generator=g, device=device, dtype=torch.float64) * 2 - 1)
    return n, n, row_ptr, col, val.to(value_dtype)


def rmat_csr_numpy(scale: int, edge_factor: int, seed: int, permute: bool = True):
    """CPU twin of rmat_csr_torch (same distribution, numpy RNG)."""
    n = 1 << scale
    m = edge_factor * n
    a, b, c = GRAPH500
    rng = np.random.default_rng(seed)
    row = np.zeros(m, np.int64)
    col = np.zeros(m, np.int64)
    for _ in range(scale):
        r = rng.random(m)
        rb = r >= (a + b)
        cb = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        row = row * 2 + rb
        col = col * 2 + cb
    if permute:
        perm = rng.permutation(n)
        row, col = perm[row], perm[col]
    key = np.unique(row * n + col)
    row, col = key // n, key % n
    row_ptr = np.concatenate(([0], np.cumsum(np.bincount(row, minlength=n)))).astype(np.int64)
    val = rng.uniform(-1.0, 1.0, key.size)
    return n, n, row_ptr, col, val


def laplacian_csr(grid_n: int):
    """5-point Laplacian on a grid_n x grid_n grid (4 on the diagonal, -1 off), numpy CSR."""
    n = grid_n * grid_n
    i, j = np.divmod(np.arange(n), grid_n)
    cols = [np.where(i > 0, np.arange(n) - grid_n, -1), np.where(j > 0, np.arange(n) - 1, -1),
            np.arange(n), np.where(j < grid_n - 1, np.arange(n) + 1, -1),
            np.where(i < grid_n - 1, np.arange(n) + grid_n, -1)]
    vals = [-1.0, -1.0, 4.0, -1.0, -1.0]
    C = np.stack(cols, 1)
    V = np.broadcast_to(np.array(vals), C.shape)
    ok = C >= 0
    counts = ok.sum(1)
    row_ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    return n, n, row_ptr, C[ok].astype(np.int64), V[ok].astype(np.float64)


def banded_csr(n: int, half_band: int = 32, step: int = 2, seed: int = 0):
    """Banded FEM-like matrix: diagonals at offsets -half_band..half_band in
    steps of `step` (33 diagonals for 32/2), values uniform(-1, 1)."""
    offs = np.arange(-half_band, half_band + 1, step)
    rng = np.random.default_rng(seed)
    r = np.arange(n)[:, None]
    C = r + offs[None, :]
    ok = (C >= 0) & (C < n)
    counts = ok.sum(1)
    row_ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    col = C[ok].astype(np.int64)
    return n, n, row_ptr, col, rng.uniform(-1.0, 1.0, col.size)


def banded_csr_torch(n: int, device, value_dtype, half_band: int = 32, step: int = 2,
                     seed: int = 0):
    """GPU twin of banded_csr (same structure; values from torch's generator):
    nnz = 33 n - 544 for the default band."""
    import torch
    offs = torch.arange(-half_band, half_band + 1, step, device=device)
    r = torch.arange(n, device=device)
    first = torch.clamp(((-r - offs.min()) + step - 1) // step, min=0)   # first valid diagonal
    last = torch.clamp((n - 1 - r - offs.min()) // step, max=offs.numel() - 1)
    counts = (last - first + 1).clamp(min=0)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    nnz = int(row_ptr[-1].item())
    row = torch.repeat_interleave(r, counts)
    k = torch.arange(nnz, device=device) - row_ptr[row]
    col = (row + offs.min() + (first[row] + k) * step).to(torch.int32)
    del row, k
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    val = torch.rand(nnz, generator=g, device=device, dtype=torch.float64) * 2 - 1
    return n, n, row_ptr, col, val.to(value_dtype)


def uniform_csr_torch(rows: int, cols: int, mean: float, seed: int, device, value_dtype):
    """Poisson(mean) entries per row, uniform distinct columns (duplicates
    drawn with replacement are removed), values uniform(-1, 1)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    counts = torch.poisson(torch.full((rows,), float(mean), device=device), generator=g).long()
    row = torch.repeat_interleave(torch.arange(rows, device=device), counts)
    col = torch.randint(0, cols, (row.numel(),), generator=g, device=device)
    key = torch.unique(row * cols + col, sorted=True)
    row, col = key // cols, (key % cols).to(torch.int32)
    row_ptr = torch.zeros(rows + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(torch.bincount(row, minlength=rows), 0)
    val = torch.rand(col.numel(), generator=g, device=device, dtype=torch.float64) * 2 - 1
    return rows, cols, row_ptr, col, val.to(value_dtype)


def synth_csr_torch(rows: int, cols: int, pattern: str, mean: float, seed: int, device,
                    value_dtype):
    """The reference's own generator (synth.py generate(SyntheticSpec(...)),
    reproduced bit for bit by paper_2504_08860_b200.synth; its stable sorts
    run on `device`) as device CSR.  cfg4 = SyntheticSpec(8388608, 8388608,
    "uniform", 16.0, seed=0): 134,197,939 nnz."""
    import torch
    from paper_2504_08860_b200.synth import SyntheticSpec, generate_arrays
    r, c, v = generate_arrays(SyntheticSpec(rows, cols, pattern, mean, seed=seed), device=device)
    row_ptr = torch.zeros(rows + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(torch.bincount(torch.as_tensor(r, device=device), minlength=rows), 0)
    col = torch.as_tensor(c.astype(np.int32), device=device)
    val = torch.as_tensor(v, device=device).to(value_dtype)
    return rows, cols, row_ptr, col, val
