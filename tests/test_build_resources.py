"""Resource guards on the built libhbp.so (no GPU needed: cuobjdump reads the
cubin).  The measured occupancy of the SpMV kernels depends on ptxas
register allocations that small source edits can break:

* k_spmv_stream at 896 threads (28 warps/SM, one CTA per SM) needs <= 72
  registers, at 768 threads (warm tier, 24 warps) <= 80;
* the fp64 row-block kernel (8 CTAs x 256 threads per SM) must fit 32
  registers WITHOUT spilling (a 48-56 B spill cost 15 % on cfg1).
"""
from __future__ import annotations

import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2504_08860_b200", "libhbp.so")


def _resources():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(exe):
        pytest.skip("libhbp.so or cuobjdump missing")
    out = subprocess.run([exe, "-res-usage", LIB], capture_output=True, text=True,
                         check=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and name:
            res[name] = (int(m.group(1)), int(m.group(2)))
            name = None
    return res


def test_stream_kernel_register_budget():
    res = _resources()
    stream = {k: v for k, v in res.items() if "k_spmv_stream" in k}
    assert stream, "no k_spmv_stream instantiations found"
    for k, (reg, _) in stream.items():
        if "Li896E" in k:
            assert reg <= 72, (k, reg)
        elif "Li768E" in k:
            assert reg <= 80, (k, reg)


def test_rowblock_f64_spill_free():
    res = _resources()
    hits = [(k, v) for k, v in res.items() if "k_spmv_rowblockIdLb1ELi256ELi8ELi2E" in k]
    assert hits, "default fp64 row-block instantiation not found"
    for k, (reg, stack) in hits:
        assert reg <= 32 and stack == 0, (k, reg, stack)
