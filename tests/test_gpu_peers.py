"""Peer copies of y (hbp_balanced_t.y_peer, the fused power iteration's
store path) and the CUDA IPC helpers, in one process: the peers are other
buffers on the same device, so the copies must equal y bit for bit.  The
two-process IPC case is in test_gpu_stripes.py."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

import paper_2504_08860_b200 as H
from paper_2504_08860_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _op(n, dtype, density=8, seed=0, empty_tail=0):
    rng = np.random.default_rng(seed)
    lens = rng.poisson(density, n)
    if empty_tail:
        lens[n - empty_tail:] = 0  # whole empty row blocks at the end
    r = np.repeat(np.arange(n), lens)
    c = rng.integers(0, n, r.size)
    trip = H.TripletMatrix(n, n, r, c, rng.uniform(-1, 1, r.size).astype(dtype))
    csr = H.coo_to_csr(trip.canonicalized())
    cfg = H.PartitionConfig(col_width=n)
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    return H.SpmvOperator(hbp, schedule="stream")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("npeers", [1, 3, 7])
def test_peer_copies_equal_y(dtype, npeers):
    n = 40000
    op = _op(n, dtype, empty_tail=1536)
    assert op.has_empty_row_blocks
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, n).astype(dtype), device="cuda")
    sq = torch.tensor([7.0], dtype=torch.float64, device="cuda")
    ref = op(x, x_sumsq=sq).clone()
    # peers hold garbage first: every row (empty row blocks too) must be written
    peers = [torch.full((n + 64,), float("nan"), dtype=x.dtype, device="cuda")
             for _ in range(npeers)]
    y = torch.empty_like(ref)
    op(x, y, x_sumsq=sq, y_peers=[p.data_ptr() + 64 * p.element_size() for p in peers])
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    for p in peers:
        assert torch.equal(p[64:], ref)
        assert torch.isnan(p[:64]).all()  # nothing outside the stripe
    # the next call without peers leaves them alone
    for p in peers:
        p.fill_(0)
    op(x, y)
    torch.cuda.synchronize()
    assert all(int(torch.count_nonzero(p)) == 0 for p in peers)


def test_peer_copies_need_one_column_block_stream():
    n = 20000
    rng = np.random.default_rng(0)
    r = np.repeat(np.arange(n), 4)
    c = rng.integers(0, n, r.size)
    trip = H.TripletMatrix(n, n, r, c, rng.uniform(-1, 1, r.size))
    csr = H.coo_to_csr(trip.canonicalized())
    cfg = H.PartitionConfig(col_width=4096)
    grid = H.make_grid(csr, cfg)
    hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)))
    op = H.SpmvOperator(hbp, schedule="stream")
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    peer = torch.empty(n, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="y_peers"):
        op(x, y_peers=[peer.data_ptr()])
    op1 = _op(5000, np.float64)
    with pytest.raises(ValueError, match="at most"):
        op1(torch.zeros(5000, dtype=torch.float64, device="cuda"),
            y_peers=[peer.data_ptr()] * (L.MAX_PEERS + 1))


def test_ipc_export_offsets():
    """hbp_ipc_export reports the tensor's byte offset inside its CUDA
    allocation (caching-allocator tensors start inside a segment)."""
    t = torch.empty(1 << 20, dtype=torch.float32, device="cuda")

    def export(v):
        h = (ctypes.c_char * L.IPC_HANDLE_BYTES)()
        off = L.c_i64(0)
        L.call("hbp_ipc_export", L.P(v), h, ctypes.byref(off))
        return bytes(h), off.value

    h0, o0 = export(t)
    h1, o1 = export(t[1000:])
    assert h0 == h1 and o1 - o0 == 4000
