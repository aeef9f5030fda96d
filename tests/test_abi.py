"""CPU checks: the C-ABI library loads and exports every symbol include/hbp.h
declares; host-side logic that needs no device."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hbp.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hbp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2504_08860_b200 import build
    return build.build()


def test_header_declares_core_entry_points():
    names = _declared()
    for must in ("hbp_hash_perm", "hbp_emit", "hbp_spmv_blocks", "hbp_combine",
                 "hbp_grid_count_runs", "hbp_sample_counts", "hbp_expand_reference"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hbp_[a-z0-9_]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(libpath):
    from paper_2504_08860_b200 import _lib as L
    lib = L.load_library(libpath)
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) <= set(L.EXPORTED)
    assert lib.hbp_abi_version() == 3
    assert lib.hbp_status_string(1002).decode().startswith("permutation")


def test_kernels_compiled_for_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_partition_config_validation():
    from paper_2504_08860_b200 import PartitionConfig
    c = PartitionConfig()
    assert (c.col_width, c.row_height, c.warp_size, c.fixed_fraction) == (4096, 512, 32, 0.7)
    for kw in ({"col_width": 0}, {"row_height": 0}, {"warp_size": 0},
               {"row_height": 10, "warp_size": 4}, {"fixed_fraction": -0.1},
               {"fixed_fraction": 1.5}):
        with pytest.raises(ValueError):
            PartitionConfig(**kw)
    with pytest.raises(AttributeError):
        c.col_width = 1


def test_hash_params_and_slot():
    from paper_2504_08860_b200 import BUCKET_MAX, HashParams, hash_slot
    with pytest.raises(ValueError, match="shift"):
        HashParams(a=-1, b=4, c=1, d=4)
    with pytest.raises(ValueError, match="stride"):
        HashParams(a=0, b=0, c=1, d=0)
    with pytest.raises(ValueError, match="d must equal b"):
        HashParams(a=0, b=4, c=1, d=5)
    with pytest.raises(ValueError, match="co-prime"):
        HashParams(a=0, b=4, c=2, d=4)
    assert hash_slot(100, 5, HashParams(a=0, b=4, c=1, d=4)) == BUCKET_MAX * 4 + 1 == 33
    assert hash_slot(13, 4, HashParams(a=1, b=7, c=3, d=7)) == 47


def test_geometry_helpers():
    from paper_2504_08860_b200.partition import (groups_in_row_block, groups_per_col_block,
                                                 rows_in_row_block)
    assert rows_in_row_block(100, 32, 3) == 4
    assert groups_in_row_block(100, 32, 8, 3) == 1
    assert groups_per_col_block(100, 32, 8) == 13


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2504_08860_b200 import TripletMatrix
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        TripletMatrix(2, 2, np.array([0]), np.array([1]), np.array([1.0]))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2504_08860_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


def test_struct_mirrors_match_the_header(libpath):
    """The ctypes mirrors have the C structs' sizes (a field added on one
    side only would shift every later field)."""
    import ctypes
    from paper_2504_08860_b200 import _lib as L
    lib = L.load_library(libpath)
    out = (ctypes.c_int64 * 4)()
    assert lib.hbp_struct_sizes(out) == 0
    assert list(out) == [ctypes.sizeof(t) for t in (L.FormatT, L.ScheduleT, L.BalancedT, L.SegT)]
