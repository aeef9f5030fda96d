"""bench.py's host-side helpers (CPU): the gather roofline arithmetic, the
format-bytes estimate, the config table and the reference-arm scope."""
from __future__ import annotations

import json
import os
import types

import pytest
import torch

import bench


def test_gather_roofline_arithmetic():
    with open(os.path.join(bench.ROOT, "profiles", "gather_peaks.json")) as fh:
        g = json.load(fh)
    nnz, ms, mhz, sms = 100_000_000, 0.5, 1965.0, 148
    r = bench.gather_roofline(nnz, 0.25, 0.0, True, ms, mhz, sms)
    hz = mhz * 1e6 * sms
    t = nnz * max(0.25 / g["lds_mix"]["per_sm_cycle_pure_lds"],
                  0.75 / g["ldg_l2_resident"]["per_sm_cycle"]) / hz  # the paths overlap
    assert r["min_ms"] == pytest.approx(t * 1e3, rel=1e-4)
    assert r["frac"] == pytest.approx(t * 1e3 / ms, rel=1e-3)
    assert r["tiers"]["cold"] == pytest.approx(0.75)
    far = bench.gather_roofline(nnz, 0.0, 0.0, False, ms, mhz, sms)
    assert far["min_ms"] > r["min_ms"]  # beyond L2 is slower per gather
    assert bench.gather_roofline(nnz, 0.0, 0.0, True, ms, None, sms) is None
    # all-shared: bound by the shared-memory rate alone
    lds = bench.gather_roofline(nnz, 1.0, 0.0, True, ms, mhz, sms)
    assert lds["min_ms"] == pytest.approx(nnz / g["lds_mix"]["per_sm_cycle_pure_lds"] / hz * 1e3, rel=1e-4)


def _fake(schedule, nzb=10, R=512, nnz=100_000, rows=5000, cols=7000, esz=4, hot=None,
          partial=None, nph=1234):
    hbp = types.SimpleNamespace(
        config=types.SimpleNamespace(row_height=R), nzb=nzb, nnz=nnz, rows=rows, cols=cols,
        phases=torch.zeros(1), phase_ptr=torch.tensor([0, nph]))
    op = types.SimpleNamespace(schedule=schedule, hot=hot, partial=partial)
    return op, hbp


def test_format_bytes_stream_and_partial():
    op, hbp = _fake("stream")
    fb = bench.format_bytes(op, hbp, 4)
    ngroups, slots = 10 * 16, 10 * 512
    assert fb["elements"] == 100_000 * 8
    assert fb["metadata"] == ngroups * 16 + slots * 4 + 1234 * 8
    assert fb["x_staging"] == 0 and fb["partial_round_trip"] == 0
    assert fb["total"] == fb["elements"] + fb["metadata"] + (5000 + 7000) * 4
    hot = types.SimpleNamespace(n_hot=64, n_warm=1000)
    op, hbp = _fake("seg", hot=hot, partial=torch.zeros(slots, dtype=torch.float64))
    fb = bench.format_bytes(op, hbp, 8)
    assert fb["metadata"] == ngroups * 8 + slots * 8
    assert fb["x_staging"] == 1064 * (4 + 16)
    assert fb["partial_round_trip"] == slots * 8 * 2


def test_config_table_and_reference_scope():
    assert {"cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "H"} <= set(bench.CONFIGS)
    assert bench.REF_FULL <= set(bench.CONFIGS)
    assert "cfg3" not in bench.REF_FULL and "cfg5" not in bench.REF_FULL  # host-infeasible
    for name, (desc, gen, dt, C) in bench.CONFIGS.items():
        assert dt in ("f32", "f64") and isinstance(desc, str) and "kind" in gen


def test_pipeline_pieces_cover_the_vector():
    """HostPipeline copies each vector as `chunks` consecutive pieces."""
    from paper_2504_08860_b200.engine import HostPipeline
    p = HostPipeline.__new__(HostPipeline)
    for n in (1, 7, 1000, 1 << 20):
        for k in (1, 2, 3, 8, 16):
            p.chunks = k
            pcs = p._pieces(n)
            assert pcs[0][0] == 0 and pcs[-1][1] == n
            assert all(a < b for a, b in pcs) and len(pcs) <= k
            assert all(pcs[i][1] == pcs[i + 1][0] for i in range(len(pcs) - 1))
