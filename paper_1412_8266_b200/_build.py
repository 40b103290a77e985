"""Build libshv.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libshv.so")
SOURCES = [os.path.join(CSRC, f) for f in ("kernels_mrg.cu", "kernels_philox.cu", "kernels_threefry.cu",
                                            "kernels_tinymt32.cu", "kernels_leapfrog.cu", "kernels_audit.cu", "kernels_mtgp32.cu",
                                            "shv_api.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "shv_internal.h"), os.path.join(CSRC, "kernels_common.cuh"), os.path.join(ROOT, "include", "shv_device.cuh"), os.path.join(ROOT, "include", "shv.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def build(force: bool = False, verbose: bool = False) -> str:
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in DEPS)):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2",
           "-shared", "-cudart", "static", "-I", os.path.join(ROOT, "include"),
           "-o", tmp, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
