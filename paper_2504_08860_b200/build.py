"""Build libhbp.so in-tree with nvcc for sm_100a (B200).

`python -m paper_2504_08860_b200.build` or `__graft_entry__.build()`.
The .so lands next to this file so it travels with the repo snapshot to the
GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libhbp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]  # + -c / -shared per step


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + [
        os.path.join(ROOT, "include", "hbp.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def _compile(src: str, obj: str) -> subprocess.CompletedProcess:
    cmd = [NVCC, *ARCH, *FLAGS, "-c", "-I", os.path.join(ROOT, "include"), "-o", obj, src]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc per translation unit (in parallel), then one shared link."""
    if not force and up_to_date():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    odir = os.path.join(PKG, "build")
    os.makedirs(odir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(odir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs, objs))
    for r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libhbp.so")
        if verbose:
            sys.stderr.write(r.stderr)
    link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB + ".tmp", *objs]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libhbp.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
