"""Build libsma.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The library is plain CUDA C++ behind the C ABI in include/sma.h; it does not
link NCCL (it dlopen()s the process's libnccl.so.2) and links the CUDA runtime
statically, so it loads in any process that has a CUDA driver.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsma.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    for p in sys.path:
        cand = os.path.join(p, "nvidia", "nccl", "include")
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include"
    raise RuntimeError("nccl.h not found (needed for NCCL types only)")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps() -> list[str]:
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + \
        sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        [os.path.join(ROOT, "include", "sma.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(p) <= t for p in deps()):
            return LIB
    cmd = [nvcc, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
           "-shared", "-cudart", "static", f"-I{_nccl_include()}", f"-I{os.path.join(ROOT, 'include')}",
           *sources(), "-o", LIB + ".tmp", "-ldl"]
    extra = os.environ.get("SMA_NVCC_EXTRA")   # experiments only, e.g. -DSMA_SPLIT_MINB=1
    if extra:
        cmd[1:1] = extra.split()
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
