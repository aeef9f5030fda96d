"""Shared fixtures: the gpu marker, golden-case loading, and matrix builders."""
from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden", "cases")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load_golden(name):
    with np.load(os.path.join(GOLDEN_DIR, name + ".npz")) as z:
        d = {k: z[k] for k in z.files}
    for k in ("rows", "cols", "C", "R", "W", "seed", "fixed_count", "workers", "probes"):
        d[k] = int(d[k])
    d["fixed_fraction"] = float(d["fixed_fraction"])
    d["fp32"] = bool(d["fp32"])
    d["name"] = str(d["name"])
    d["ordering"] = str(d["ordering"])
    d["col_idx"] = d["trip_col"]
    d["values"] = d["trip_val"]
    return d


def triplets_from_dense(dense):
    dense = np.asarray(dense, dtype=np.float64)
    r, c = np.nonzero(dense)
    return dense.shape[0], dense.shape[1], r, c, dense[r, c]


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(autouse=True)
def _no_pending_cuda_error(request):
    """GPU tests: no libhbp.so call may leave a CUDA error pending (it would
    surface in an unrelated later launch check)."""
    yield
    if request.node.get_closest_marker("gpu") is None or not has_gpu():
        return
    from paper_2504_08860_b200 import _lib as L
    if L._lib is None:
        return
    st = L.lib().hbp_last_error()
    assert st == 0, f"pending CUDA error {st} after {request.node.nodeid}"
