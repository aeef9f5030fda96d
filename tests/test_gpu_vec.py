"""hbp_sumsq / hbp_scale (the power-iteration step of config 5) vs torch f64."""
from __future__ import annotations

import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch
    import paper_2504_08860_b200 as H


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("n", [0, 1, 31, 1000, 1 << 20, 3_000_001])
def test_sumsq_scale(dtype, n):
    dt = getattr(torch, dtype)
    g = torch.Generator(device="cuda").manual_seed(n)
    y = torch.rand(n, device="cuda", generator=g, dtype=torch.float64).mul_(2).sub_(1).to(dt)
    sq = torch.zeros(1, dtype=torch.float64, device="cuda")
    H.sumsq(y, sq)
    ref = (y.to(torch.float64) ** 2).sum()
    assert torch.allclose(sq[0], ref, rtol=1e-12, atol=0.0)
    sq2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    H.sumsq(y, sq2)
    assert torch.equal(sq, sq2)  # deterministic
    if n:
        out = torch.empty_like(y)
        H.scale(y, sq, out)
        want = y * (1.0 / torch.sqrt(sq)).to(dt)
        assert torch.equal(out, want)
        H.scale(y, sq, y)  # in place
        assert torch.equal(y, want)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_spmv_x_sumsq_scaling(dtype):
    """SpmvOperator(x, y, x_sumsq): y = A x / sqrt(x_sumsq[0]) (the power
    iteration's normalisation folded into the SpMV's y stores)."""
    import numpy as np
    dt = getattr(torch, dtype)
    rng = np.random.default_rng(3)
    rows = cols = 4000
    lens = rng.poisson(8, rows)
    r = np.repeat(np.arange(rows), lens)
    c = rng.integers(0, cols, r.size)
    key = np.unique(r * cols + c)
    r, c = key // cols, key % cols
    v = rng.uniform(-1, 1, r.size).astype(np.float32 if dtype == "float32" else np.float64)
    cfg = H.PartitionConfig(col_width=cols)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    op = H.SpmvOperator(hbp)
    x = torch.as_tensor(rng.uniform(-1, 1, cols), device="cuda").to(dt)
    plain = op(x).clone()
    one = torch.ones(1, dtype=torch.float64, device="cuda")
    assert torch.equal(op(x, x_sumsq=one), plain)  # scale 1 is exact
    s = torch.tensor([6.25], dtype=torch.float64, device="cuda")
    got = op(x, x_sumsq=s).to(torch.float64)
    want = plain.to(torch.float64) / 2.5
    tol = 1e-6 if dtype == "float32" else 1e-14
    assert torch.allclose(got, want, rtol=tol, atol=tol)
    assert torch.equal(op(x), plain)  # the scale does not stick
