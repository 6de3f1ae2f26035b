"""CPU oracle for bulk histogram filling — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2401_13310_b200) never imports it and shares no code with it; the only
module both use is bhgen (seeded input bytes, no method arithmetic).

The arithmetic lives in bhist_oracle.c (plain C, IEEE binary64, Neumaier sums);
see its header for the PAPER.md passages each step follows.  This wrapper only
marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bhist_oracle.c")
_SO = os.path.join(_HERE, "libbhist_oracle.so")
_lib = None
_P = ctypes.c_void_p


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.or_find_bin_fixed.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.or_find_bin_fixed.restype = ctypes.c_int
        L.or_find_bin_variable.argtypes = [ctypes.c_int32, _P, ctypes.c_double]
        L.or_find_bin_variable.restype = ctypes.c_int
        L.or_create.argtypes = [ctypes.c_int, _P, _P, _P, _P]
        L.or_create.restype = _P
        L.or_destroy.argtypes = [_P]
        L.or_find_bins.argtypes = [_P, ctypes.c_int64, _P, _P]
        L.or_fill.argtypes = [_P, ctypes.c_int64, _P, _P]
        L.or_merge.argtypes = [_P, _P]
        L.or_merge.restype = ctypes.c_int
        L.or_read.argtypes = [_P, _P, _P, _P, _P, _P, _P]
        L.or_nbins_total.argtypes = [_P]
        L.or_nbins_total.restype = ctypes.c_int64
        L.or_nstats.argtypes = [_P]
        L.or_nstats.restype = ctypes.c_int
        L.or_global_bin.argtypes = [_P, _P]
        L.or_global_bin.restype = ctypes.c_int64
        _lib = L
    return _lib


def find_bin_fixed(nbins: int, xmin: float, xmax: float, x: float) -> int:
    return lib().or_find_bin_fixed(nbins, xmin, xmax, x)


def find_bin_variable(edges, x: float) -> int:
    e = np.ascontiguousarray(edges, dtype=np.float64)
    return lib().or_find_bin_variable(len(e) - 1, e.ctypes.data, x)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleHist:
    """axes: list of (nbins, xmin, xmax) for fixed or np.ndarray edges for variable axes."""

    def __init__(self, axes):
        self.dim = len(axes)
        nb = (ctypes.c_int32 * 3)()
        lo = (ctypes.c_double * 3)()
        hi = (ctypes.c_double * 3)()
        ep = (ctypes.c_void_p * 3)()
        self._keep = []
        for a, ax in enumerate(axes):
            if isinstance(ax, np.ndarray) or (isinstance(ax, (list, tuple)) and len(ax) != 3):
                e = _f64(ax)
                self._keep.append(e)
                nb[a] = len(e) - 1
                ep[a] = e.ctypes.data
            else:
                nb[a], lo[a], hi[a] = int(ax[0]), float(ax[1]), float(ax[2])
                ep[a] = None
        h = lib().or_create(self.dim, ctypes.addressof(nb), ctypes.addressof(lo), ctypes.addressof(hi),
                            ctypes.addressof(ep))
        if not h:
            raise ValueError("oracle: invalid axes")
        self._h = h
        self.G = lib().or_nbins_total(h)
        self.K = lib().or_nstats(h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_destroy(self._h)
            self._h = None

    def _coords(self, coords):
        cs = [_f64(c) for c in coords]
        assert len(cs) == self.dim
        n = len(cs[0])
        assert all(len(c) == n for c in cs)
        arr = (ctypes.c_void_p * 3)(*([c.ctypes.data for c in cs] + [None] * (3 - self.dim)))
        return cs, n, arr

    def fill(self, coords, w=None):
        cs, n, arr = self._coords(coords)
        wa = None if w is None else _f64(w)
        if wa is not None:
            assert len(wa) == n
        lib().or_fill(self._h, n, ctypes.addressof(arr), None if wa is None else wa.ctypes.data)
        return self

    def find_bins(self, coords) -> np.ndarray:
        cs, n, arr = self._coords(coords)
        out = np.empty(n, dtype=np.int32)
        lib().or_find_bins(self._h, n, ctypes.addressof(arr), out.ctypes.data)
        return out

    def global_bin(self, b) -> int:
        arr = (ctypes.c_int * 3)(*(list(b) + [0] * (3 - len(b))))
        return lib().or_global_bin(self._h, ctypes.addressof(arr))

    def merge(self, other: "OracleHist") -> "OracleHist":
        if lib().or_merge(self._h, other._h) != 0:
            raise ValueError("oracle: incompatible histograms")
        return self

    def read(self) -> dict:
        c = np.empty(self.G)
        s2 = np.empty(self.G)
        ac = np.empty(self.G)
        st = np.empty(self.K)
        sa = np.empty(self.K)
        ent = ctypes.c_int64()
        lib().or_read(self._h, c.ctypes.data, s2.ctypes.data, ac.ctypes.data, st.ctypes.data,
                      sa.ctypes.data, ctypes.addressof(ent))
        return {"content": c, "sumw2": s2, "abs_content": ac, "stats": st, "stats_abs": sa,
                "entries": int(ent.value)}


def oracle_axes(hist) -> list:
    """bhgen.Hist -> OracleHist axes spec."""
    return hist.axes_spec()


def finalize_stats(stats, dim: int):
    """Per-axis (mean, stddev) from the GetStats sums:
    mean_a = sumwx_a/sumw, std_a = sqrt(max(0, sumwx2_a/sumw - mean_a^2))."""
    sumw = stats[0]
    if not sumw > 0:
        raise ValueError("empty histogram")
    idx = [(2, 3), (4, 5), (7, 8)][:dim]
    out = []
    for i, j in idx:
        m = stats[i] / sumw
        out.append((m, float(np.sqrt(max(0.0, stats[j] / sumw - m * m)))))
    return out
