"""bhgen — seeded synthetic workloads shared by the oracle and the CUDA path.

This module is the ONLY code both sides use.  It produces input bytes
(coordinates, weights, variable-axis edges) and holds none of the method's
arithmetic.  The workload recipes follow SURVEY.md §8(d) ("Data generator" and
the C1–C5 table), which shape the paper's benchmark (PAPER.md:240–251,
§4.2 lst:histond_benchmark: 1D histogram of uniform doubles on [0,1]) and the
BASELINE.json configs.

Generator (bhgen.c): u(s, i) = (splitmix64(s ^ splitmix64(i)) >> 11) * 2^-53.
Seeds: 0xB2000000 + 16*config + column (column 15 = variable-axis edges).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libbhgen.so")
_lib = None

UNIFORM, GAUSS, CAUCHY, EXP = 0, 1, 2, 3


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "bhgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fno-fast-math",
                               "-o", _SO, src, "-lm", "-lpthread"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.bg_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                              ctypes.c_double, ctypes.c_double, ctypes.c_void_p, ctypes.c_int]
        L.bg_fill.restype = ctypes.c_int
        L.bg_edges_random_widths.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p]
        L.bg_edges_random_widths.restype = ctypes.c_int
        L.bg_edges_log.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_void_p]
        L.bg_edges_log.restype = ctypes.c_int
        L.bg_splitmix64.argtypes = [ctypes.c_uint64]
        L.bg_splitmix64.restype = ctypes.c_uint64
        L.bg_u01.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.bg_u01.restype = ctypes.c_double
        _lib = L
    return _lib


def default_threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


def fill_ptr(kind: int, seed: int, start: int, n: int, p0: float, p1: float, ptr: int,
             nthreads: int | None = None) -> None:
    """Write events [start, start+n) of a stream into host memory at `ptr` (float64)."""
    rc = lib().bg_fill(kind, seed, start, n, p0, p1, ptr, nthreads or default_threads())
    if rc != 0:
        raise ValueError("bg_fill: bad arguments")


def sample(kind: int, seed: int, start: int, n: int, p0: float, p1: float,
           out: np.ndarray | None = None, nthreads: int | None = None) -> np.ndarray:
    if out is None:
        out = np.empty(n, dtype=np.float64)
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size >= n
    fill_ptr(kind, seed, start, n, p0, p1, out.ctypes.data, nthreads)
    return out[:n]


def edges_random_widths(seed: int, n: int) -> np.ndarray:
    e = np.empty(n + 1, dtype=np.float64)
    if lib().bg_edges_random_widths(seed, n, e.ctypes.data) != 0:
        raise ValueError("bad edges request")
    return e


def edges_log(lo: float, hi: float, n: int) -> np.ndarray:
    e = np.empty(n + 1, dtype=np.float64)
    if lib().bg_edges_log(lo, hi, n, e.ctypes.data) != 0:
        raise ValueError("bad edges request")
    return e


def seed_of(config: int, column: int) -> int:
    return 0xB2000000 + 16 * config + column


# --------------------------------------------------------------------------- recipes
@dataclass
class Column:
    kind: int
    p0: float
    p1: float
    seed: int


@dataclass
class Axis:
    """nbins + (xmin, xmax) for a fixed axis, or nbins + edges for a variable axis."""
    nbins: int
    xmin: float = 0.0
    xmax: float = 1.0
    edges: np.ndarray | None = None


@dataclass
class Hist:
    axes: list          # list[Axis]
    cols: list          # column index per axis
    weighted: bool

    def axes_spec(self) -> list:
        """[(nbins, xmin, xmax) | edges ndarray] per axis, the form both bindings accept."""
        return [ax.edges if ax.edges is not None else (ax.nbins, ax.xmin, ax.xmax) for ax in self.axes]


@dataclass
class Workload:
    name: str
    n_events: int
    columns: list       # list[Column]; the weight column, if any, is `wcol`
    hists: list         # list[Hist]
    wcol: int | None = None
    note: str = ""
    extra: dict = field(default_factory=dict)

    def column(self, c: int, start: int, n: int, out: np.ndarray | None = None,
               nthreads: int | None = None) -> np.ndarray:
        col = self.columns[c]
        return sample(col.kind, col.seed, start, n, col.p0, col.p1, out, nthreads)

    def column_ptr(self, c: int, start: int, n: int, ptr: int, nthreads: int | None = None) -> None:
        col = self.columns[c]
        fill_ptr(col.kind, col.seed, start, n, col.p0, col.p1, ptr, nthreads)

    @property
    def bytes_per_event(self) -> int:
        used = {c for h in self.hists for c in h.cols}
        if any(h.weighted for h in self.hists) and self.wcol is not None:
            used.add(self.wcol)
        return 8 * len(used)


def c2_edges() -> np.ndarray:
    return edges_random_widths(seed_of(2, 15), 10000)


def workload(name: str, n_events: int | None = None) -> Workload:
    """The five BASELINE.json configs, plus weighted variants C3w/C4w."""
    name = name.upper()
    if name == "C1":   # TH1D 100 fixed bins, 1e6 uniform doubles, unit weights
        return Workload("C1", n_events or 1_000_000, [Column(UNIFORM, 0.0, 1.0, seed_of(1, 0))],
                        [Hist([Axis(100, 0.0, 1.0)], [0], False)],
                        note="TH1D(100,0,1); x~U[0,1); unit weights")
    if name == "C2":   # TH1D 10,000 variable bins, 5e8 Gaussian events, random weights
        return Workload("C2", n_events or 500_000_000,
                        [Column(GAUSS, 0.5, 0.15, seed_of(2, 0)), Column(UNIFORM, 0.5, 1.5, seed_of(2, 1))],
                        [Hist([Axis(10000, edges=c2_edges())], [0], True)], wcol=1,
                        note="TH1D 10000 variable bins (random widths, ratio<=3) on [0,1]; "
                             "x~N(0.5,0.15); w~U[0.5,1.5)")
    if name in ("C3", "C3W"):   # TH2D 1000x1000 fixed, 2e8 events
        w = name == "C3W"
        cols = [Column(UNIFORM, 0.0, 1.0, seed_of(3, 0)), Column(UNIFORM, 0.0, 1.0, seed_of(3, 1))]
        if w:
            cols.append(Column(UNIFORM, 0.5, 1.5, seed_of(3, 2)))
        return Workload(name, n_events or 200_000_000, cols,
                        [Hist([Axis(1000, 0.0, 1.0), Axis(1000, 0.0, 1.0)], [0, 1], w)],
                        wcol=2 if w else None, note="TH2D(1000,0,1,1000,0,1); x,y~U[0,1)")
    if name in ("C4", "C4W"):   # TH3D 100^3 with flow, 2e8 sharply peaked events
        w = name == "C4W"
        cols = [Column(CAUCHY, 0.505, 0.002, seed_of(4, a)) for a in range(3)]
        if w:
            cols.append(Column(UNIFORM, 0.5, 1.5, seed_of(4, 3)))
        return Workload(name, n_events or 200_000_000, cols,
                        [Hist([Axis(100, 0.0, 1.0)] * 3, [0, 1, 2], w)],
                        wcol=3 if w else None,
                        note="TH3D(100,0,1)^3; x,y,z~Cauchy(0.505,0.002): ~43% of events in one bin")
    if name == "C5":   # analysis batch: 8 histograms from 7 columns, 1e9 events
        cols = [Column(UNIFORM, 0.0, 1.0, seed_of(5, 0)),
                Column(GAUSS, 0.5, 0.15, seed_of(5, 1)),
                Column(EXP, 5.0, 0.0, seed_of(5, 2)),
                Column(UNIFORM, -0.2, 1.2, seed_of(5, 3)),
                Column(CAUCHY, 0.505, 0.002, seed_of(5, 4)),
                Column(GAUSS, 0.5, 0.05, seed_of(5, 5)),
                Column(UNIFORM, 0.5, 1.5, seed_of(5, 6))]
        e2 = c2_edges()
        e3 = edges_log(1e-3, 2.0, 1000)
        hists = [Hist([Axis(100, 0.0, 1.0)], [0], False),
                 Hist([Axis(1000, 0.0, 1.0)], [1], True),
                 Hist([Axis(10000, edges=e2)], [1], True),
                 Hist([Axis(1000, edges=e3)], [2], False),
                 Hist([Axis(100, 0.0, 1.0)], [4], False),
                 Hist([Axis(100, 0.0, 1.0), Axis(100, 0.0, 1.0)], [0, 3], True),
                 Hist([Axis(1000, 0.0, 1.0), Axis(1000, 0.0, 1.0)], [1, 5], False),
                 Hist([Axis(50, 0.0, 1.0), Axis(50, 0.0, 1.0)], [4, 5], True)]
        return Workload("C5", n_events or 1_000_000_000, cols, hists, wcol=6,
                        note="8 histograms (1D/2D mix) over 7 float64 columns")
    raise KeyError(name)


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous event range [start, stop) of `rank`."""
    return (n * rank) // world, (n * (rank + 1)) // world
