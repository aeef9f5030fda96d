"""HostPipeline (end-to-end path with host buffers): every y_i equals the
device-resident SpMV of x_i, for any pipeline depth and sequence length."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch
    import paper_2504_08860_b200 as H


@pytest.mark.parametrize("depth,chunks", [(1, 1), (2, 1), (3, 1), (2, 3), (3, 8)])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_pipeline_matches_device_spmv(depth, chunks, dtype):
    rng = np.random.default_rng(depth)
    rows, cols = 5000, 7000
    lens = rng.poisson(9, rows)
    lens[rng.choice(rows, 5, replace=False)] = 3000
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size)
    if dtype == "f32":
        v = v.astype(np.float32)
    cfg = H.PartitionConfig(col_width=cols if dtype == "f32" else 1024)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    tdt = torch.float32 if dtype == "f32" else torch.float64
    xs = [torch.as_tensor(rng.uniform(-1, 1, cols)).to(tdt).pin_memory() for _ in range(7)]
    ys = [torch.empty(rows, dtype=tdt).pin_memory() for _ in range(7)]
    pipe = H.HostPipeline(hbp, depth=depth, chunks=chunks)
    pipe.run(xs, ys)
    torch.cuda.synchronize()
    op = H.SpmvOperator(hbp)
    for xh, yh in zip(xs, ys):
        want = op(xh.cuda()).cpu()
        assert torch.equal(yh, want)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("C,hot", [(None, True), (None, False), (700, True), (700, False)])
def test_operator_cuda_graph(dtype, C, hot):
    """SpmvOperator.capture: a CUDA graph of one SpMV (hot gather + stream
    kernel, or + combine) replays to the same y as a direct call."""
    import torch
    rng = np.random.default_rng(11)
    rows, cols = 3000, 2000
    lens = np.minimum(rng.zipf(1.8, rows) + 2, cols // 2)
    r = np.repeat(np.arange(rows), lens)
    w = 1.0 / np.arange(1, cols + 1)
    c = rng.choice(cols, r.size, p=w / w.sum())
    key = np.unique(r.astype(np.int64) * cols + c)
    r, c = key // cols, key % cols
    v = rng.uniform(-1, 1, r.size).astype(dtype)
    cfg = H.PartitionConfig(col_width=C or cols, row_height=512, warp_size=32)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    op = H.SpmvOperator(hbp, hot=hot)
    assert (op.hot is not None) == hot
    x = torch.as_tensor(rng.uniform(-1, 1, cols).astype(dtype), device="cuda")
    y = torch.empty(rows, dtype=x.dtype, device="cuda")
    want = op(x).clone()
    g = op.capture(x, y)
    y.zero_()
    x2 = torch.as_tensor(rng.uniform(-1, 1, cols).astype(dtype), device="cuda")
    want2 = op(x2).clone()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)
    x.copy_(x2)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want2)
