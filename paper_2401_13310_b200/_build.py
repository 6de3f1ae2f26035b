"""Build libbhist.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.environ.get("BHIST_LIBRARY") or os.path.join(HERE, "libbhist.so")   # override: A/B experiments
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("bhist.cu", "bhist_kernels.cuh")]
HEADER = os.path.join(ROOT, "include", "bhist.h")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-diag-suppress", "177"]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in SOURCES + [HEADER])


def build(force: bool = False, verbose: bool = False, defines=()) -> str:
    if force or stale():
        cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", SO + ".tmp",
               os.path.join(HERE, "csrc", "bhist.cu")]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force=True, verbose=True))
