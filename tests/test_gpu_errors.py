"""Error paths of the drop-in boundary, ported from the reference's tests.

- structural corruption: /root/reference/pkg/tests/test_hbp.py:134-178
  (validate_structure messages "output_hash", "add_sign", "zero_row";
  the chain walker's rejections);
- the .hbp codec: test_hbp.py:181-248 (round trip, "magic", "version",
  "truncated", structure validated on load) -- the header checks run before
  anything touches the GPU, so those cases are CPU tests;
- argument checks: "duplicate" (formats.py:252-255, test_formats.py:183),
  "worker count" / "workers" (engine.py:139-140, test_engine.py:86,152),
  "length" (engine.py:182-183, test_engine.py:145), "config"
  (hbp.py:158-159, test_hbp.py:93-99), "permutation" (hbp.py:180-181),
  TripletMatrix's "equal length" / "row index" / "column index"
  (test_formats.py:130-136);
- block_spmv with a caller-made PartialVector(values, rows, ncb)
  (engine.py:59-68, 123-134) and the reference's combine of it.
"""
from __future__ import annotations

import io

import numpy as np
import pytest

from conftest import has_gpu, triplets_from_dense

import paper_2504_08860_b200 as H
from paper_2504_08860_b200.hbp import HbpFormatError, deserialize_hbp

gpu = pytest.mark.gpu

if has_gpu():
    import torch
    from oracle import oracle as O


# ---------------------------------------------------------------- CPU cases
def test_bad_magic():
    with pytest.raises(HbpFormatError, match="magic"):
        deserialize_hbp(io.BytesIO(b"XXXX" + b"\x00" * 100))


def test_bad_version():
    buf = io.BytesIO(b"HBP1" + (99).to_bytes(4, "little") + b"\x00" * 64)
    with pytest.raises(HbpFormatError, match="version"):
        deserialize_hbp(buf)


def test_truncated_header_and_arrays():
    # a well-formed header for an 8x8 identity (C=4, R=4, W=2) followed by
    # array records cut short at every boundary kind
    import struct
    head = b"HBP1" + struct.pack("<I", 1) + struct.pack("<8Q", 8, 8, 8, 4, 4, 2, 2, 2)
    body = struct.pack("<Q", 9) + b"\x00" * 72 + struct.pack("<Q", 8) + b"\x00" * 16
    whole = head + body
    for cut in (0, 3, 40, len(head) + 4, len(whole) - 1):
        with pytest.raises(HbpFormatError, match="truncated"):
            deserialize_hbp(io.BytesIO(whole[:cut]))


def test_bad_config_in_header():
    import struct
    head = b"HBP1" + struct.pack("<I", 1) + struct.pack("<8Q", 8, 8, 0, 4, 6, 4, 2, 2)
    arrays = b"".join(struct.pack("<Q", 0) for _ in range(6))
    with pytest.raises(HbpFormatError, match="config"):
        deserialize_hbp(io.BytesIO(head + arrays))


# ---------------------------------------------------------------- GPU cases
def _build_hashed(trip, cfg, seed=0):
    """test_hbp.py:37-41."""
    csr = H.coo_to_csr(trip)
    grid = H.make_grid(csr, cfg)
    params = H.sample_hash_params(grid, cfg, seed=seed)
    return H.build_hbp(csr, grid, H.hash_permutations(grid, params))


def _build_identity(dense, cfg):
    csr = H.coo_to_csr(H.TripletMatrix(*triplets_from_dense(dense)))
    grid = H.make_grid(csr, cfg)
    return H.build_hbp(csr, grid, H.identity_permutations(grid))


def _validation_matrix():
    """test_hbp.py:135-138."""
    cfg = H.PartitionConfig(col_width=32, row_height=16, warp_size=4)
    trip = H.generate(H.SyntheticSpec(64, 64, "uniform", 5.0, seed=3))
    return _build_hashed(trip, cfg)


@gpu
def test_clean_build_validates():
    _validation_matrix().validate_structure()


@gpu
def test_detects_output_hash_duplicate():
    hbp = _validation_matrix()
    hbp.output_hash[1] = hbp.output_hash[0]
    with pytest.raises(HbpFormatError, match="output_hash"):
        hbp.validate_structure()


@gpu
def test_detects_group_start_regression():
    hbp = _validation_matrix()
    hbp.group_start[1] = hbp.group_start[-1] + 1
    with pytest.raises(HbpFormatError):
        hbp.validate_structure()


@gpu
def test_detects_bad_stride_domain():
    hbp = _validation_matrix()
    hbp.add_sign[0] = -2
    with pytest.raises(HbpFormatError, match="add_sign"):
        hbp.validate_structure()


@gpu
def test_detects_zero_row_mismatch():
    hbp = _validation_matrix()
    z0 = int(hbp.zero_row[0])
    hbp.zero_row[0] = 7 if z0 != 7 else 5
    with pytest.raises(HbpFormatError, match="zero_row"):
        hbp.validate_structure()


@gpu
def test_detects_zero_row_of_empty_block():
    """A slot of an EMPTY block (no compact storage) corrupted in the dense
    view is still caught (it used to be re-synthesised)."""
    cfg = H.PartitionConfig(col_width=4, row_height=4, warp_size=2)
    hbp = _build_identity(np.eye(8), cfg)
    buf = io.BytesIO()
    H.serialize_hbp(hbp, buf)
    raw = bytearray(buf.getvalue())
    # zero_row is the 5th array: find it by walking the records
    import struct
    off = 4 + 4 + 64
    for k in range(4):
        (cnt,) = struct.unpack_from("<Q", raw, off)
        off += 8 + cnt * (8 if k in (0, 2) else 4)
    (cnt,) = struct.unpack_from("<Q", raw, off)
    zr = np.frombuffer(bytes(raw[off + 8:off + 8 + 4 * cnt]), np.int32).copy()
    # block (1, 0) (rows 4..7, column block 0) is empty: all its slots are -1
    assert (zr[4:8] == -1).all()
    zr[5] = 0
    raw[off + 8:off + 8 + 4 * cnt] = zr.tobytes()
    with pytest.raises(HbpFormatError, match="zero_row"):
        deserialize_hbp(io.BytesIO(bytes(raw)))


@gpu
def test_walker_rejects_zero_stride():
    hbp = _validation_matrix()
    pos = int(torch.argmax((hbp.add_sign > 0).to(torch.int32)))
    hbp.add_sign[pos] = 0
    with pytest.raises(HbpFormatError):
        H.hbp_to_triplets(hbp)


@gpu
def test_walker_rejects_out_of_block_column():
    hbp = _validation_matrix()
    hbp.col[0] = hbp.cols + 5
    with pytest.raises(HbpFormatError):
        H.hbp_to_triplets(hbp)


@gpu
def test_codec_round_trip_and_truncation():
    """test_hbp.py:207-237: the real stream of a built matrix, cut anywhere."""
    cfg = H.PartitionConfig(col_width=4, row_height=4, warp_size=2)
    hbp = _build_identity(np.eye(8), cfg)
    buf = io.BytesIO()
    H.serialize_hbp(hbp, buf)
    whole = buf.getvalue()
    assert len(whole) == 448  # test_hbp.py:200-208
    back = deserialize_hbp(io.BytesIO(whole))
    ref = hbp.to_reference()
    got = back.to_reference()
    for k in ("col", "data", "add_sign", "zero_row", "group_start", "output_hash"):
        np.testing.assert_array_equal(got[k], ref[k])
    np.testing.assert_array_equal(H.hbp_spmv(back, np.arange(8.0)).cpu().numpy(), np.arange(8.0))
    for cut in (0, 3, 40, len(whole) - 1):
        with pytest.raises(HbpFormatError, match="truncated"):
            deserialize_hbp(io.BytesIO(whole[:cut]))


@gpu
def test_deserialized_structure_is_validated():
    """test_hbp.py:239-248."""
    cfg = H.PartitionConfig(col_width=4, row_height=4, warp_size=2)
    hbp = _build_identity(np.eye(8), cfg)
    buf = io.BytesIO()
    H.serialize_hbp(hbp, buf)
    raw = bytearray(buf.getvalue())
    raw[-64:-60] = raw[-60:-56]
    with pytest.raises(HbpFormatError, match="output_hash"):
        deserialize_hbp(io.BytesIO(bytes(raw)))


@gpu
def test_deserialize_bad_group_start_length():
    """Wrong-length group_start is an HbpFormatError, not an IndexError."""
    import struct
    cfg = H.PartitionConfig(col_width=4, row_height=4, warp_size=2)
    hbp = _build_identity(np.eye(8), cfg)
    buf = io.BytesIO()
    H.serialize_hbp(hbp, buf)
    raw = bytes(buf.getvalue())
    off = 4 + 4 + 64
    (cnt,) = struct.unpack_from("<Q", raw, off)
    bad = raw[:off] + struct.pack("<Q", 0) + raw[off + 8 + 8 * cnt:]
    with pytest.raises(HbpFormatError, match="group_start"):
        deserialize_hbp(io.BytesIO(bad))


@gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_codec_round_trip_hashed(seed):
    """A hashed power-law matrix: load_hbp(save_hbp(m)) rebuilds the compact
    runtime arrays on the device (chain lengths) and gives the same y."""
    cfg = H.PartitionConfig(col_width=64, row_height=32, warp_size=8)
    trip = H.generate(H.SyntheticSpec(300, 200, "powerlaw", 6.0, seed=seed))
    hbp = _build_hashed(trip, cfg)
    buf = io.BytesIO()
    H.serialize_hbp(hbp, buf)
    back = deserialize_hbp(io.BytesIO(buf.getvalue()))
    assert back.nzb == hbp.nzb
    np.testing.assert_array_equal(back.slot_len.cpu().numpy(), hbp.slot_len.cpu().numpy())
    np.testing.assert_array_equal(back.perm.cpu().numpy(), hbp.perm.cpu().numpy())
    np.testing.assert_array_equal(back.group_start_c.cpu().numpy(),
                                  hbp.group_start_c.cpu().numpy())
    x = np.random.default_rng(seed).uniform(-1, 1, 200)
    np.testing.assert_array_equal(H.hbp_spmv(back, x).cpu().numpy(),
                                  H.hbp_spmv(hbp, x).cpu().numpy())
    out = io.BytesIO()
    H.serialize_hbp(back, out)
    assert out.getvalue() == buf.getvalue()


@gpu
def test_duplicates_rejected():
    """formats.py:252-255 / test_formats.py:179-184."""
    m = H.TripletMatrix(2, 2, np.array([0, 0]), np.array([1, 1]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError, match="duplicate"):
        H.coo_to_csr(m)


@gpu
def test_triplet_validation():
    with pytest.raises(ValueError, match="equal length"):
        H.TripletMatrix(2, 2, np.array([0]), np.array([0, 1]), np.array([1.0]))
    with pytest.raises(ValueError, match="row index"):
        H.TripletMatrix(2, 2, np.array([2]), np.array([0]), np.array([1.0]))
    with pytest.raises(ValueError, match="column index"):
        H.TripletMatrix(2, 2, np.array([0]), np.array([-1]), np.array([1.0]))


@gpu
def test_config_mismatch_rejected():
    """test_hbp.py:93-99."""
    csr = H.coo_to_csr(H.TripletMatrix(*triplets_from_dense(np.eye(4))))
    cfg = H.PartitionConfig(col_width=4, row_height=4, warp_size=4)
    grid = H.make_grid(csr, cfg)
    other = H.PartitionConfig(col_width=8, row_height=4, warp_size=4)
    with pytest.raises(ValueError, match="config"):
        H.build_hbp(csr, grid, H.identity_permutations(grid), other)


@gpu
def test_non_bijective_permutation_rejected():
    """hbp.py:180-181: a dense table whose block is not a bijection."""
    csr = H.coo_to_csr(H.TripletMatrix(*triplets_from_dense(np.eye(8))))
    cfg = H.PartitionConfig(col_width=4, row_height=4, warp_size=2)
    grid = H.make_grid(csr, cfg)
    table = np.tile(np.arange(4, dtype=np.uint32), 2 * 2)
    H.build_hbp(csr, grid, table)  # the identity table is fine
    table[5] = table[4]  # block (1, 0): two slots -> local row 0
    with pytest.raises(ValueError, match=r"permutation of block \(1, 0\)"):
        H.build_hbp(csr, grid, table)
    with pytest.raises(ValueError, match="length"):
        H.build_hbp(csr, grid, table[:-1])


@gpu
def test_worker_checks():
    """test_engine.py:84-87, 143-153."""
    dense = np.eye(32)
    cfg = H.PartitionConfig(col_width=8, row_height=8, warp_size=4, fixed_fraction=0.7)
    hbp = _build_identity(dense, cfg)
    csr = H.coo_to_csr(H.TripletMatrix(*triplets_from_dense(dense)))
    grid = H.make_grid(csr, cfg)
    with pytest.raises(ValueError, match="workers"):
        H.plan_execution(grid, cfg, workers=0)
    with pytest.raises(ValueError, match="length"):
        H.hbp_spmv(hbp, np.zeros(31))
    plan = H.plan_execution(hbp, cfg, workers=2)
    with pytest.raises(ValueError, match="worker count"):
        H.run_spmv(hbp, np.zeros(32), plan, workers=3)
    with pytest.raises(ValueError, match="workers"):
        H.hbp_spmv(hbp, np.zeros(32), workers=0)


@gpu
def test_operator_argument_checks():
    """SpmvOperator takes raw pointers: device, dtype, length and
    contiguity are checked before any launch."""
    cfg = H.PartitionConfig(col_width=16, row_height=32, warp_size=32)
    trip = H.generate(H.SyntheticSpec(64, 48, "uniform", 4.0, seed=1))
    hbp = _build_hashed(trip, cfg)
    op = H.SpmvOperator(hbp)
    x = torch.rand(48, dtype=torch.float64, device="cuda")
    y = op(x)
    assert y.shape == (64,)
    with pytest.raises(ValueError, match="CUDA"):
        op(x.cpu())
    with pytest.raises(ValueError, match="dtype"):
        op(x.float())
    with pytest.raises(ValueError, match="length"):
        op(x[:47])
    with pytest.raises(ValueError, match="length"):
        op(torch.rand(96, dtype=torch.float64, device="cuda")[::2])
    with pytest.raises(ValueError, match="length"):
        op(x, torch.empty(63, dtype=torch.float64, device="cuda"))


@gpu
@pytest.mark.parametrize("as_numpy", [True, False])
def test_block_spmv_reference_partial(as_numpy):
    """engine.py:123-134 with a caller-made PartialVector(values, rows, ncb):
    every nonzero block into the dense partial, then combine -- bitwise the
    oracle's dense partial and y."""
    rng = np.random.default_rng(5)
    rows, cols = 70, 50
    d = rng.uniform(-1, 1, (rows, cols)) * (rng.random((rows, cols)) < 0.2)
    C, R, W = 16, 16, 4
    cfg = H.PartitionConfig(col_width=C, row_height=R, warp_size=W)
    hbp = _build_hashed(H.TripletMatrix(*triplets_from_dense(d)), cfg)
    x = rng.uniform(-1, 1, cols)
    ncb = hbp.num_col_blocks
    if as_numpy:
        values = np.zeros(ncb * rows)
    else:
        values = torch.zeros(ncb * rows, dtype=torch.float64, device="cuda")
    partial = H.PartialVector(values, rows, ncb)
    for br, bc in H.plan_execution(hbp, cfg, workers=1).block_order:
        H.block_spmv(hbp, (br, bc), x, partial)
    r, c = np.nonzero(d)
    p = O.pipeline(rows, cols, r, c, d[r, c], C, R, W)
    plan = O.plan_execution(p["hbp"].block_nnz_matrix(), 0.7, 1)
    want_partial, _ = O.run_spmv(p["hbp"], x, plan, 1)
    got = values if as_numpy else values.cpu().numpy()
    np.testing.assert_array_equal(got, want_partial)
    y = H.combine(partial).cpu().numpy()
    np.testing.assert_array_equal(y, O.hbp_spmv(p["hbp"], x, workers=1))
    np.testing.assert_array_equal(y, H.hbp_spmv(hbp, x).cpu().numpy())
