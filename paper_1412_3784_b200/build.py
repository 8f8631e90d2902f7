"""Build the sm_100a shared library libnemdcell.so in-tree with nvcc."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC_DIR = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(SRC_DIR, "nemdcell.cu")]
DEPS = SOURCES + [os.path.join(SRC_DIR, f) for f in ("kernels.cuh", "k3_seg.cuh", "k3_sparse.cuh", "k3_rows.cuh", "k3_sparse64.cuh", "geom.hpp", "nccl_slab.cuh", "slab_dc.cuh", "ipc_slab.cuh")] + [
    os.path.join(os.path.dirname(HERE), "include", "nemdcell.h")]
LIB = os.path.join(HERE, "libnemdcell.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared",
    # one CUDA runtime per process: share libcudart.so.12 with torch instead of a
    # private static copy (two runtimes tearing down the same context at exit crashed)
    "-cudart", "shared", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
    "-ldl",  # NCCL is dlopen'ed at run time (csrc/nccl_slab.cuh)
]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *NVCC_FLAGS, *SOURCES, "-o", tmp]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
