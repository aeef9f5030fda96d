"""The thresholded hub-row path of the stream kernel in exact (f64) mode
(SpmvOperator(hub_min=...), hbp_balanced_t.hub_min).

Groups longer than hub_min elements are cut across warps and summed in
fast-mode order: deterministic and within 1e-12 componentwise (north_star's
fp64 bound), not bitwise.  Every row of every other group stays bitwise the
reference (_kernels.py:41-46 order).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch
    import paper_2504_08860_b200 as H
    from oracle import oracle as O

FP64_TOL = 1e-12  # north_star: 1e-12 relative for fp64 (componentwise, |A||x| scale)


def _skewed(seed=3, rows=4096, cols=50000):
    rng = np.random.default_rng(seed)
    lens = rng.poisson(6, rows)
    hot = rng.choice(rows, 12, replace=False)
    lens[hot] = rng.integers(min(20000, cols // 2), min(40000, cols), hot.size)
    lens[rows // 2: rows // 2 + 40] = 900
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, k, replace=False) for k in lens])
    v = rng.uniform(-1, 1, r.size)
    return rows, cols, r, c, v


def _hbp(rows, cols, r, c, v, C):
    cfg = H.PartitionConfig(col_width=C, row_height=512, warp_size=32)
    csr = H.coo_to_csr(H.TripletMatrix(rows, cols, r, c, v))
    grid = H.make_grid(csr, cfg)
    return H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))


def _hub_rows(hbp, hub_min):
    """Rows whose group holds more than hub_min elements."""
    gs = hbp.group_start_c.cpu().numpy()
    glen = np.diff(gs)
    R = hbp.config.row_height
    gpb = R // 32
    br = hbp.blk_br.cpu().numpy()
    perm = hbp.perm.cpu().numpy().reshape(-1, R)
    rows = set()
    for g in np.nonzero(glen > hub_min)[0]:
        blk, gi = divmod(int(g), gpb)
        for lane in range(32):
            s = gi * 32 + lane
            row = br[blk] * R + perm[blk, s]
            if s < min(R, hbp.rows - br[blk] * R):
                rows.add(int(row))
    return np.array(sorted(rows), dtype=np.int64)


@pytest.mark.parametrize("hub_min", [1024, 5000, "auto"])
@pytest.mark.parametrize("workers", [37, None])
def test_hub_rows_within_tolerance_rest_bitwise(hub_min, workers):
    rows, cols, r, c, v = _skewed()
    hbp = _hbp(rows, cols, r, c, v, C=cols)
    x = np.random.default_rng(1).uniform(-1, 1, cols)
    xd = torch.as_tensor(x, device="cuda")
    exact = H.SpmvOperator(hbp, schedule="stream", workers=workers)
    hub = H.SpmvOperator(hbp, schedule="stream", workers=workers, hub_min=hub_min)
    assert hub.hub_min > 0 and exact.hub_min == 0
    y0 = exact(xd).cpu().numpy()
    y1 = hub(xd).cpu().numpy()
    y2 = hub(xd).cpu().numpy()
    np.testing.assert_array_equal(y1, y2)  # deterministic
    p = O.pipeline(rows, cols, r, c, v, cols, 512, 32)
    ref = O.hbp_spmv(p["hbp"], x, workers=2)
    np.testing.assert_array_equal(y0, ref)  # exact mode: bitwise
    hubs = _hub_rows(hbp, hub.hub_min)
    assert hubs.size > 0
    rest = np.setdiff1d(np.arange(rows), hubs)
    np.testing.assert_array_equal(y1[rest], ref[rest])
    err = O.componentwise_error(rows, r, c, v, x, y1)
    assert err <= FP64_TOL, err


def test_hub_with_partials_several_column_blocks():
    """ncb > 1: hub pieces land in the partial; the combine is unchanged."""
    rows, cols, r, c, v = _skewed(seed=4, rows=3000, cols=40000)
    hbp = _hbp(rows, cols, r, c, v, C=15000)
    x = np.random.default_rng(2).uniform(-1, 1, cols)
    y = H.SpmvOperator(hbp, schedule="stream", hub_min=800)(
        torch.as_tensor(x, device="cuda")).cpu().numpy()
    err = O.componentwise_error(rows, r, c, v, x, y)
    assert err <= FP64_TOL, err


def test_hub_min_validation():
    rows, cols, r, c, v = _skewed(seed=5, rows=600, cols=3000)
    hbp = _hbp(rows, cols, r, c, v, C=cols)
    with pytest.raises(ValueError, match="hub_min"):
        H.SpmvOperator(hbp, schedule="stream", hub_min=-1)
