"""Build libbhist.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

The fill-kernel templates are split over one translation unit per (DIM, weighted)
pair (csrc/bhist_fill_d*.cu) so the objects compile in parallel; bhist.cu holds the
C ABI, the host logic and the one-off kernels.
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.environ.get("BHIST_LIBRARY") or os.path.join(HERE, "libbhist.so")   # override: A/B experiments
HEADER = os.path.join(ROOT, "include", "bhist.h")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "177"]


def units() -> list[str]:
    return [os.path.join(CSRC, "bhist.cu")] + sorted(glob.glob(os.path.join(CSRC, "bhist_fill_d*.cu")))


def sources() -> list[str]:
    return units() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [HEADER]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in sources())


def build(force: bool = False, verbose: bool = False, defines=()) -> str:
    if not (force or stale()):
        return SO
    objdir = os.path.join(os.path.dirname(SO), "build", os.path.basename(SO) + ".obj")
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src: str) -> str:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *NVCC_FLAGS, *dflags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        return obj

    srcs = units()
    with concurrent.futures.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", SO + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force=True, verbose=True))
