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
