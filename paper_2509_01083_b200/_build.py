"""Builds libdsde.so (the C-ABI + sm_100a kernels) in-tree with nvcc.

Only nvcc/g++ are used (no torch JIT cache): the .so lands next to this file
so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libdsde.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _nccl_include() -> str:
    cands = []
    try:
        import nvidia.nccl  # the NCCL torch bundles: same version as the one loaded at run time
        cands += [os.path.join(p, "include") for p in nvidia.nccl.__path__]
    except Exception:
        pass
    cands += ["/usr/include", "/usr/local/cuda/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    deps.append(os.path.join(CSRC, "exports.map"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [_nvcc(), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3",
           f"-I{INCLUDE}", f"-I{CSRC}", f"-I{_nccl_include()}",
           "-Xlinker", f"--version-script={os.path.join(CSRC, 'exports.map')}",
           *os.environ.get("DSDE_NVCC_FLAGS", "").split(),
           "-o", LIB + ".tmp", *sources(), "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
