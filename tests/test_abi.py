"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol the
header declares, and fails loudly (status codes, no crash, no fallback) without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2401_13310_b200 as pkg
from paper_2401_13310_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "bhist.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bh_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_loads():
    _build.build()
    assert os.path.exists(_build.SO)
    assert pkg.bh_version() >= 10000


def test_every_declared_symbol_exported():
    declared = _declared()
    assert declared == sorted(pkg.EXPORTED)
    L = ctypes.CDLL(_build.SO)
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _build.SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(bh_\w+)", out))
    assert set(declared) <= exported


def test_kernels_are_sm100a_sass():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _build.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_hot_kernels_use_no_local_memory():
    """The bench headline kernel (C2: k_fill<1, weighted, PRIV, vector, compact>) and the
    GLOBAL / unit-CACHE kernels keep the kernel parameters out of local memory: a reference or
    pointer into FillP made nvcc copy it to local memory (STL at entry, generic returning
    atomics, +9% instructions on C2)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _build.SO], capture_output=True, text=True).stdout
    funcs = {}
    name = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name:
            funcs[name].append(line)
    for k in ("_ZN2bh6k_fillILi1ELb1ELi0ELb1ELi3EEEvNS_5FillPE",      # C2
              "_ZN2bh6k_fillILi2ELb1ELi1ELb1ELi0EEEvNS_5FillPE",      # C3w GLOBAL
              "_ZN2bh6k_fillILi2ELb0ELi2ELb1ELi0EEEvNS_5FillPE"):     # C5 H6 unit CACHE / WINDOW
        body = "\n".join(funcs[k])
        assert not re.search(r"\b(STL|LDL)\b", body), k
        assert "ATOM.E.ADD" not in body, k                           # no generic returning atomics


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pkg.BHistError) as ei:
        pkg.bh_create([(10, 0.0, 1.0)], 0)
    assert ei.value.status in (-4, -3)   # BH_EDEVICE / BH_ECUDA, never a silent success


def test_null_handle_rejected():
    L = pkg.lib()
    assert L.bh_reset(None, None) == -1
    assert L.bh_fill(None, 1, None, None, None) == -1
    assert "NULL" in pkg.bh_last_error()


def test_product_does_not_import_oracle():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2401_13310_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower(), f


def test_header_constants_match_binding():
    # every #define BH_* integer of the header has the same value in the Python binding
    src = open(os.path.join(ROOT, "include", "bhist.h")).read()
    consts = {k: int(v) for k, v in re.findall(r"#define\s+(BH_[A-Z0-9_]+)\s+\(?(-?\d+)\)?", src)}
    assert {"BH_STRATEGY_AUTO", "BH_STRATEGY_SORT", "BH_DEBUG_SKIP_COPY_WAIT"} <= set(consts)
    from paper_2401_13310_b200 import bhist
    for k, v in consts.items():
        if hasattr(bhist, k):
            assert getattr(bhist, k) == v, k
    for k in ("BH_STRATEGY_AUTO", "BH_STRATEGY_PRIV", "BH_STRATEGY_GLOBAL", "BH_STRATEGY_CACHE",
              "BH_STRATEGY_EXACT", "BH_STRATEGY_SORT"):
        assert getattr(pkg, k) == consts[k], k


def test_build_units_cover_every_dim_and_weight():
    names = sorted(os.path.basename(u) for u in _build.units())
    assert names[0] == "bhist.cu"
    assert names[1:-1] == [f"bhist_fill_d{d}{w}.cu" for d in (1, 2, 3) for w in ("u", "w")]
    assert names[-1] == "bhist_jit.cu"


def test_jit_fused_kernel_compiles_for_sm100a():
    """The one-pass fused kernel of bh_fill_multi, instantiated for C5's two-role plan,
    compiles with NVRTC for sm_100a (no GPU needed)."""
    expr = ("bh::k_fused<bh::Role<19u, bh::Grp<bh::HS<2,1,true,3,1,0,0,3,0,0>, bh::HS<0,1,false,1,0,0,0,0,0,0>>, "
            "bh::Grp<bh::HS<1,1,true,3,1,0,0,0,0,0>, bh::HS<4,1,false,1,4,0,0,0,0,0>, bh::HS<3,1,false,0,2,0,0,2,0,0>>>, "
            "bh::Role<19u, bh::Grp<bh::HS<5,2,true,3,0,3,0,0,0,0>>, "
            "bh::Grp<bh::HS<7,2,true,3,4,5,0,0,0,0>, bh::HS<6,2,false,2,1,5,0,0,0,0>>>>")
    msg = pkg.bh_jit_compile_check(expr, 768, 1)
    assert msg.startswith("ok:") and "sm_100a" in msg
    with pytest.raises(pkg.BHistError):
        pkg.bh_jit_compile_check("bh::k_fused<bh::Role<0u, bh::Grp<bh::HS<0,4,true,0,0,0,0,0,0,0>>, bh::Grp<>>>")  # DIM 4
