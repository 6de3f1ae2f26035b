"""ctypes binding of include/bhist.h — argument marshalling only.

Every function named bh_* mirrors the C entry point of the same name (see the
header for semantics, layouts, ownership and errors).  Pointers are passed as
Python ints (e.g. torch ``tensor.data_ptr()``); streams as ints
(``torch.cuda.Stream.cuda_stream``) or None for the legacy default stream.
``Histogram`` is a convenience wrapper over torch tensors (PyTorch is used for
device memory and streams only; every step of the fill runs in libbhist).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

BH_OK, BH_EINVAL, BH_ENOMEM, BH_ECUDA, BH_EDEVICE, BH_EMISMATCH = 0, -1, -2, -3, -4, -5
BH_STRATEGY_AUTO, BH_STRATEGY_PRIV, BH_STRATEGY_GLOBAL, BH_STRATEGY_CACHE, BH_STRATEGY_EXACT, BH_STRATEGY_SORT = 0, 1, 2, 3, 4, 5
BH_DEBUG_SKIP_COPY_WAIT = 1
BH_DEBUG_FIND_BINS_GLOBAL = 2
BH_DEBUG_REQUIRE_JIT = 4
BH_MULTI_PASSES, BH_MULTI_ONE_PASS = 0, 1
BH_CONTENT_F64, BH_CONTENT_F32, BH_CONTENT_I32 = 0, 1, 2

# every symbol include/bhist.h declares (checked by tests/test_abi.py)
EXPORTED = ["bh_version", "bh_last_error", "bh_create", "bh_destroy", "bh_reset", "bh_fill", "bh_fill_host",
            "bh_fill_multi", "bh_fill_expr", "bh_fill_f32", "bh_fill_i32", "bh_find_bins", "bh_info", "bh_packed_size", "bh_pack", "bh_unpack", "bh_read", "bh_read_as", "bh_set_strategy",
            "bh_fill_host_f32", "bh_fill_host_i32", "bh_packed_size_multi", "bh_pack_multi", "bh_unpack_multi",
            "bh_jit_compile_check",
            "bh_get_strategy", "bh_set_chunk", "bh_set_debug", "bh_set_multi_mode", "bh_launch_count",
            "bh_bulk_begin", "bh_bulk_submit", "bh_bulk_wait", "bh_bulk_fill", "bh_bulk_end"]


class BHistError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"bhist error {status}: {msg}")
        self.status = status


class _Op(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("dst", ctypes.c_int32), ("a", ctypes.c_int32), ("b", ctypes.c_int32),
                ("c", ctypes.c_int32), ("pad", ctypes.c_int32), ("imm", ctypes.c_double)]


# opcodes of bh_fill_expr (include/bhist.h BH_OP_*)
OPS = {name: i for i, name in enumerate(
    ["const", "copy", "add", "sub", "mul", "div", "sqrt", "abs", "neg", "min", "max", "lt", "le", "gt", "ge",
     "eq", "ne", "and", "or", "not", "select"])}


class _Axis(ctypes.Structure):
    _fields_ = [("nbins", ctypes.c_int32), ("xmin", ctypes.c_double), ("xmax", ctypes.c_double),
                ("edges", ctypes.c_void_p)]


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32


def library_path() -> str:
    return _build.SO


def lib(build_if_stale: bool = False):
    """Load libbhist.so.  Raises if it is missing: there is no fallback path."""
    global _lib
    if _lib is None:
        if build_if_stale:
            _build.build()
        if not os.path.exists(_build.SO):
            raise ImportError(f"libbhist.so not built ({_build.SO}); run __graft_entry__.build()")
        L = ctypes.CDLL(_build.SO)
        sig = {
            "bh_version": ([], _I32),
            "bh_last_error": ([], ctypes.c_char_p),
            "bh_create": ([_I32, _P, _I32, _P], _I32),
            "bh_destroy": ([_P], _I32),
            "bh_reset": ([_P, _P], _I32),
            "bh_fill": ([_P, _I64, _P, _P, _P], _I32),
            "bh_fill_host": ([_P, _I64, _P, _P, _P], _I32),
            "bh_fill_host_f32": ([_P, _I64, _P, _P, _P], _I32),
            "bh_fill_host_i32": ([_P, _I64, _P, _P, _P], _I32),
            "bh_packed_size_multi": ([_P, _I32, _P, _P], _I32),
            "bh_pack_multi": ([_P, _I32, _P, _P, _P], _I32),
            "bh_unpack_multi": ([_P, _I32, _P, _P, _P], _I32),
            "bh_jit_compile_check": ([ctypes.c_char_p, _I32, _I32, ctypes.c_char_p, _I64], _I32),
            "bh_find_bins": ([_P, _I64, _P, _P, _P], _I32),
            "bh_fill_multi": ([_P, _I32, _P, _P, _I64, _P, _I32, _P, _P], _I32),
            "bh_fill_expr": ([_P, _I64, _P, _I32, _P, _I32, _P, _I32, _I32, _P], _I32),
            "bh_fill_f32": ([_P, _I64, _P, _P, _P], _I32),
            "bh_fill_i32": ([_P, _I64, _P, _P, _P], _I32),
            "bh_info": ([_P, _P, _P, _P], _I32),
            "bh_packed_size": ([_P, _P], _I32),
            "bh_pack": ([_P, _P, _P], _I32),
            "bh_unpack": ([_P, _P, _P], _I32),
            "bh_read": ([_P, _P, _P, _P, _P, _P], _I32),
            "bh_read_as": ([_P, _I32, _P, _P, _P, _P, _P], _I32),
            "bh_set_strategy": ([_P, _I32], _I32),
            "bh_get_strategy": ([_P, _I32, _P], _I32),
            "bh_set_chunk": ([_P, _I64], _I32),
            "bh_set_debug": ([_P, _I32], _I32),
            "bh_set_multi_mode": ([_P, _I32], _I32),
            "bh_bulk_begin": ([_P, _I32, _I32, _P], _I32),
            "bh_bulk_submit": ([_P, _I64, _P, _P, _P], _I32),
            "bh_bulk_wait": ([_P, _I64], _I32),
            "bh_bulk_fill": ([_P, _I64, _P, _P], _I32),
            "bh_bulk_end": ([_P], _I32),
            "bh_launch_count": ([_P, _P], _I32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st: int):
    if st != BH_OK:
        raise BHistError(st, bh_last_error())


def _ptrs(ptrs):
    arr = (ctypes.c_void_p * 3)(*(list(ptrs) + [None] * (3 - len(ptrs))))
    return arr


# ---------------------------------------------------------------- C-ABI mirrors
def bh_version() -> int:
    return lib().bh_version()


def bh_last_error() -> str:
    return lib().bh_last_error().decode()


def bh_create(axes, device: int = 0):
    """axes: list of (nbins, xmin, xmax) for fixed axes or 1-D float64 arrays of edges."""
    dim = len(axes)
    arr = (_Axis * 3)()
    keep = []
    for a, ax in enumerate(axes):
        if isinstance(ax, np.ndarray) or (isinstance(ax, (list, tuple)) and len(ax) != 3):
            e = np.ascontiguousarray(ax, dtype=np.float64)
            keep.append(e)
            arr[a] = _Axis(len(e) - 1, 0.0, 0.0, e.ctypes.data)
        else:
            arr[a] = _Axis(int(ax[0]), float(ax[1]), float(ax[2]), None)
    out = ctypes.c_void_p()
    _check(lib().bh_create(dim, ctypes.addressof(arr), device, ctypes.byref(out)))
    return out.value


def bh_destroy(h) -> None:
    _check(lib().bh_destroy(h))


def bh_reset(h, stream=None) -> None:
    _check(lib().bh_reset(h, stream))


def bh_fill(h, n: int, coord_ptrs, w_ptr=None, stream=None) -> None:
    arr = _ptrs(coord_ptrs)      # must outlive the call
    _check(lib().bh_fill(h, n, ctypes.addressof(arr), w_ptr, stream))


def bh_fill_f32(h, n: int, coord_ptrs, w_ptr=None, stream=None) -> None:
    arr = _ptrs(coord_ptrs)
    _check(lib().bh_fill_f32(h, n, ctypes.addressof(arr), w_ptr, stream))


def bh_fill_i32(h, n: int, coord_ptrs, w_ptr=None, stream=None) -> None:
    arr = _ptrs(coord_ptrs)
    _check(lib().bh_fill_i32(h, n, ctypes.addressof(arr), w_ptr, stream))


def bh_fill_host(h, n: int, coord_ptrs, w_ptr=None, stream=None) -> None:
    arr = _ptrs(coord_ptrs)
    _check(lib().bh_fill_host(h, n, ctypes.addressof(arr), w_ptr, stream))


def bh_fill_host_f32(h, n: int, coord_ptrs, w_ptr=None, stream=None) -> None:
    arr = _ptrs(coord_ptrs)
    _check(lib().bh_fill_host_f32(h, n, ctypes.addressof(arr), w_ptr, stream))


def bh_fill_host_i32(h, n: int, coord_ptrs, w_ptr=None, stream=None) -> None:
    arr = _ptrs(coord_ptrs)
    _check(lib().bh_fill_host_i32(h, n, ctypes.addressof(arr), w_ptr, stream))


def _multi_args(handles, unit):
    nh = len(handles)
    hs = (ctypes.c_void_p * nh)(*handles)
    u = None if unit is None else (ctypes.c_uint8 * nh)(*[1 if x else 0 for x in unit])
    return nh, hs, u


def bh_packed_size_multi(handles, unit=None) -> int:
    nh, hs, u = _multi_args(handles, unit)
    n = _I64()
    _check(lib().bh_packed_size_multi(ctypes.addressof(hs), nh, None if u is None else ctypes.addressof(u),
                                      ctypes.byref(n)))
    return n.value


def bh_pack_multi(handles, unit, dev_out_ptr, stream=None) -> None:
    nh, hs, u = _multi_args(handles, unit)
    _check(lib().bh_pack_multi(ctypes.addressof(hs), nh, None if u is None else ctypes.addressof(u), dev_out_ptr,
                               stream))


def bh_unpack_multi(handles, unit, dev_in_ptr, stream=None) -> None:
    nh, hs, u = _multi_args(handles, unit)
    _check(lib().bh_unpack_multi(ctypes.addressof(hs), nh, None if u is None else ctypes.addressof(u), dev_in_ptr,
                                 stream))


def bh_jit_compile_check(kernel_expr: str, threads: int = 512, ept: int = 2) -> str:
    """NVRTC-compile a fused-kernel instantiation for sm_100a (no GPU needed); returns the message."""
    buf = ctypes.create_string_buffer(4096)
    _check(lib().bh_jit_compile_check(kernel_expr.encode(), threads, ept, buf, len(buf)))
    return buf.value.decode()


def bh_fill_multi(handles, col_of_axis, weighted, n: int, col_ptrs, w_ptr=None, stream=None) -> None:
    """handles: list of bh_hist handles; col_of_axis: per histogram a list of column indices."""
    nh = len(handles)
    hs = (ctypes.c_void_p * nh)(*handles)
    coa = (ctypes.c_int32 * (3 * nh))()
    for i, cs in enumerate(col_of_axis):
        for a, c in enumerate(cs):
            coa[3 * i + a] = c
    wt = (ctypes.c_uint8 * nh)(*[1 if x else 0 for x in weighted])
    cp = (ctypes.c_void_p * len(col_ptrs))(*col_ptrs)
    _check(lib().bh_fill_multi(ctypes.addressof(hs), nh, ctypes.addressof(coa), ctypes.addressof(wt), n,
                               ctypes.addressof(cp), len(col_ptrs), w_ptr, stream))


def bh_fill_expr(h, n: int, col_ptrs, prog, axis_regs, weight_reg: int = -1, filter_reg: int = -1,
                 stream=None) -> None:
    """prog: list of (opname, dst, a, b, c, imm) tuples (see Program)."""
    cp = (ctypes.c_void_p * max(1, len(col_ptrs)))(*col_ptrs)
    ops = (_Op * max(1, len(prog)))()
    for k, (name, dst, a, b, c, imm) in enumerate(prog):
        ops[k] = _Op(OPS[name], dst, a, b, c, 0, float(imm))
    ar = (ctypes.c_int32 * 3)(*(list(axis_regs) + [0] * (3 - len(axis_regs))))
    _check(lib().bh_fill_expr(h, n, ctypes.addressof(cp), len(col_ptrs), ctypes.addressof(ops), len(prog),
                              ctypes.addressof(ar), weight_reg, filter_reg, stream))


class Program:
    """Builder for bh_fill_expr register programs: registers 0..ncols-1 are the input
    columns; every method appends one op and returns the register it wrote."""

    def __init__(self, ncols: int):
        self.ncols = ncols
        self.ops = []
        self._next = ncols

    def _emit(self, name, a=0, b=0, c=0, imm=0.0):
        if self._next >= 16:
            raise ValueError("out of registers (16)")
        r = self._next
        self._next += 1
        self.ops.append((name, r, a, b, c, imm))
        return r

    def const(self, v):
        return self._emit("const", imm=v)

    def land(self, a, b):
        return self._emit("and", a, b)

    def lor(self, a, b):
        return self._emit("or", a, b)

    def lnot(self, a):
        return self._emit("not", a)

    def __getattr__(self, name):
        if name in OPS and name != "const":
            return lambda a=0, b=0, c=0: self._emit(name, a, b, c)
        raise AttributeError(name)


def fill_expr(hist, cols, prog: "Program", axis_regs, weight_reg: int = -1, filter_reg: int = -1, stream=None):
    """Filter + Define + fill in one kernel: cols are contiguous float64 CUDA tensors."""
    import torch
    n = cols[0].numel() if cols else 0
    _check_cols(cols, (torch.float64,), n, hist.device, "cols")
    bh_fill_expr(hist.h, n, [c.data_ptr() for c in cols], prog.ops, axis_regs, weight_reg, filter_reg,
                 _stream_handle(stream, hist.device))


def fill_multi(hists, col_of_axis, weighted, cols, w=None, stream=None, mode=None) -> None:
    """Histogram-level wrapper: cols are contiguous float64 CUDA tensors of equal length;
    mode (BH_MULTI_*, None = leave as set) is the plan, set on hists[0]."""
    import torch
    if mode is not None:
        bh_set_multi_mode(hists[0].h, mode)
    n = cols[0].numel()
    _check_cols(cols + ([w] if w is not None else []), (torch.float64,), n, hists[0].device, "cols / w")
    bh_fill_multi([h.h for h in hists], col_of_axis, weighted, n, [c.data_ptr() for c in cols],
                  None if w is None else w.data_ptr(), _stream_handle(stream, hists[0].device))


def bh_find_bins(h, n: int, coord_ptrs, out_ptr, stream=None) -> None:
    arr = _ptrs(coord_ptrs)
    _check(lib().bh_find_bins(h, n, ctypes.addressof(arr), out_ptr, stream))


def bh_info(h):
    d, g, k = _I32(), _I64(), _I32()
    _check(lib().bh_info(h, ctypes.byref(d), ctypes.byref(g), ctypes.byref(k)))
    return d.value, g.value, k.value


def bh_packed_size(h) -> int:
    n = _I64()
    _check(lib().bh_packed_size(h, ctypes.byref(n)))
    return n.value


def bh_pack(h, dev_out_ptr, stream=None) -> None:
    _check(lib().bh_pack(h, dev_out_ptr, stream))


def bh_unpack(h, dev_in_ptr, stream=None) -> None:
    _check(lib().bh_unpack(h, dev_in_ptr, stream))


def bh_read(h, stream=None) -> dict:
    _, G, K = bh_info(h)
    c = np.empty(G)
    s2 = np.empty(G)
    st = np.empty(K)
    ent = _I64()
    _check(lib().bh_read(h, c.ctypes.data, s2.ctypes.data, st.ctypes.data, ctypes.byref(ent), stream))
    return {"content": c, "sumw2": s2, "stats": st, "entries": ent.value}


def bh_read_as(h, content_type: int, stream=None) -> dict:
    """bh_read with TH1F / TH1I-style contents (BH_CONTENT_F32: float32, BH_CONTENT_I32: int32)."""
    if content_type == BH_CONTENT_F64:
        return bh_read(h, stream)
    _, G, K = bh_info(h)
    dt = {BH_CONTENT_F32: np.float32, BH_CONTENT_I32: np.int32}.get(content_type)
    if dt is None:
        raise BHistError(f"unknown content type {content_type}")
    c = np.empty(G, dtype=dt)
    s2 = np.empty(G, dtype=dt)
    st = np.empty(K)
    ent = _I64()
    _check(lib().bh_read_as(h, content_type, c.ctypes.data, s2.ctypes.data, st.ctypes.data, ctypes.byref(ent), stream))
    return {"content": c, "sumw2": s2, "stats": st, "entries": ent.value}


def bh_set_strategy(h, strategy: int) -> None:
    _check(lib().bh_set_strategy(h, strategy))


def bh_get_strategy(h, weighted: bool) -> int:
    s = _I32()
    _check(lib().bh_get_strategy(h, int(bool(weighted)), ctypes.byref(s)))
    return s.value


def bh_set_chunk(h, events: int) -> None:
    _check(lib().bh_set_chunk(h, events))


def bh_set_debug(h, flags: int) -> None:
    _check(lib().bh_set_debug(h, flags))


def bh_bulk_begin(h, weighted: bool, timeout_ms: int = 0, stream=None) -> None:
    _check(lib().bh_bulk_begin(h, int(bool(weighted)), timeout_ms, stream))


def bh_bulk_submit(h, n: int, host_col_ptrs, host_w_ptr=None) -> int:
    arr = _ptrs(host_col_ptrs)
    t = _I64()
    _check(lib().bh_bulk_submit(h, n, ctypes.addressof(arr), host_w_ptr, ctypes.byref(t)))
    return t.value


def bh_bulk_wait(h, ticket: int) -> None:
    _check(lib().bh_bulk_wait(h, ticket))


def bh_bulk_fill(h, n: int, host_col_ptrs, host_w_ptr=None) -> None:
    arr = _ptrs(host_col_ptrs)
    _check(lib().bh_bulk_fill(h, n, ctypes.addressof(arr), host_w_ptr))


def bh_bulk_end(h) -> None:
    _check(lib().bh_bulk_end(h))


def bh_set_multi_mode(h, mode: int) -> None:
    _check(lib().bh_set_multi_mode(h, mode))


def bh_launch_count(h) -> int:
    n = _I64()
    _check(lib().bh_launch_count(h, ctypes.byref(n)))
    return n.value


# ---------------------------------------------------------------- torch convenience
def _stream_handle(stream, device=None):
    """None -> the current torch stream of `device` (the histogram's device, not the
    caller's current device); torch.cuda.Stream or a raw cudaStream_t int otherwise."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check_cols(cols, dtypes, n, device, what):
    """Every column: a contiguous CUDA tensor of an allowed dtype, `n` elements, on `device`."""
    for c in cols:
        if not (c.is_cuda and c.dtype in dtypes and c.is_contiguous() and c.numel() == n):
            raise ValueError(f"{what} must be contiguous CUDA tensors of dtype {dtypes} and length {n}")
        if c.device.index != device:
            raise ValueError(f"{what} live on cuda:{c.device.index}, the histogram on cuda:{device}")


def _host_col(a, n, what, dtype=np.float64):
    """A host column for the bh_fill_host* calls: contiguous, `n` elements of `dtype`, not on a GPU."""
    import torch
    tdt = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32}[dtype]
    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != tdt or not a.is_contiguous() or a.numel() != n:
            raise ValueError(f"{what} must be a contiguous {tdt} host tensor of length {n}")
        return a.data_ptr()
    if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous and a.size == n):
        raise ValueError(f"{what} must be a contiguous {np.dtype(dtype).name} numpy array of length {n}")
    return a.ctypes.data


class Histogram:
    """A device-resident TH1D/TH2D/TH3D-style histogram (owns a bh_hist)."""

    def __init__(self, axes, device: int = 0, strategy: int = BH_STRATEGY_AUTO):
        self.device = device
        self.h = bh_create(axes, device)
        self.dim, self.nbins_total, self.nstats = bh_info(self.h)
        if strategy != BH_STRATEGY_AUTO:
            bh_set_strategy(self.h, strategy)

    def close(self):
        if getattr(self, "h", None):
            bh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _s(self, stream):
        return _stream_handle(stream, self.device)

    def _coords(self, coords):
        if len(coords) != self.dim:
            raise ValueError(f"need {self.dim} coordinate columns, got {len(coords)}")
        return coords[0].numel()

    def reset(self, stream=None):
        bh_reset(self.h, self._s(stream))
        return self

    def fill(self, coords, w=None, stream=None):
        """coords: list of `dim` contiguous float64 CUDA tensors; w: float64 CUDA tensor or None."""
        import torch
        n = self._coords(coords)
        _check_cols(coords + ([w] if w is not None else []), (torch.float64,), n, self.device, "coords / w")
        bh_fill(self.h, n, [c.data_ptr() for c in coords], None if w is None else w.data_ptr(), self._s(stream))
        return self

    def fill_f32(self, coords, w=None, stream=None):
        """float32 CUDA tensors (widened exactly to float64 inside the kernel)."""
        import torch
        n = self._coords(coords)
        _check_cols(coords + ([w] if w is not None else []), (torch.float32,), n, self.device, "coords / w")
        bh_fill_f32(self.h, n, [c.data_ptr() for c in coords], None if w is None else w.data_ptr(), self._s(stream))
        return self

    def fill_i32(self, coords, w=None, stream=None):
        """int32 coordinate CUDA tensors, optional float32 weights (coordinates widened exactly)."""
        import torch
        n = self._coords(coords)
        _check_cols(coords, (torch.int32,), n, self.device, "coords")
        if w is not None:
            _check_cols([w], (torch.float32,), n, self.device, "w")
        bh_fill_i32(self.h, n, [c.data_ptr() for c in coords], None if w is None else w.data_ptr(), self._s(stream))
        return self

    def fill_host(self, coords, w=None, stream=None):
        """coords / w: host (preferably pinned) contiguous float64 torch tensors or numpy arrays."""
        if len(coords) != self.dim:
            raise ValueError(f"need {self.dim} coordinate columns, got {len(coords)}")
        n = len(coords[0])
        ptrs = [_host_col(c, n, "coords") for c in coords]
        bh_fill_host(self.h, n, ptrs, None if w is None else _host_col(w, n, "w"), self._s(stream))
        return self

    # persistent bulk consumer (bh_bulk_*): one resident kernel for a sequence of host bulks
    def bulk_begin(self, weighted: bool, timeout_ms: int = 0, stream=None):
        bh_bulk_begin(self.h, weighted, timeout_ms, self._s(stream))
        return self

    def _bulk_ptrs(self, coords, w):
        if len(coords) != self.dim:
            raise ValueError(f"need {self.dim} coordinate columns, got {len(coords)}")
        n = len(coords[0])
        return n, [_host_col(c, n, "coords") for c in coords], None if w is None else _host_col(w, n, "w")

    def bulk_submit(self, coords, w=None) -> int:
        """Post host columns (pinned: read in place, keep them unmodified until bulk_wait)."""
        n, ptrs, wp = self._bulk_ptrs(coords, w)
        return bh_bulk_submit(self.h, n, ptrs, wp)

    def bulk_wait(self, ticket: int):
        bh_bulk_wait(self.h, ticket)
        return self

    def bulk_fill(self, coords, w=None):
        n, ptrs, wp = self._bulk_ptrs(coords, w)
        bh_bulk_fill(self.h, n, ptrs, wp)
        return self

    def bulk_end(self):
        bh_bulk_end(self.h)
        return self

    def fill_host_f32(self, coords, w=None, stream=None):
        """Host float32 columns (pinned preferably): half the PCIe bytes of fill_host."""
        self._fill_host_4(coords, w, np.float32, bh_fill_host_f32, stream)
        return self

    def fill_host_i32(self, coords, w=None, stream=None):
        """Host int32 coordinate columns, optional host float32 weights."""
        self._fill_host_4(coords, w, np.int32, bh_fill_host_i32, stream)
        return self

    def _fill_host_4(self, coords, w, cdt, fn, stream):
        if len(coords) != self.dim:
            raise ValueError(f"need {self.dim} coordinate columns, got {len(coords)}")
        n = len(coords[0])
        ptrs = [_host_col(c, n, "coords", cdt) for c in coords]
        fn(self.h, n, ptrs, None if w is None else _host_col(w, n, "w", np.float32), self._s(stream))

    def find_bins(self, coords, stream=None):
        import torch
        n = self._coords(coords)
        _check_cols(coords, (torch.float64,), n, self.device, "coords")
        out = torch.empty(n, dtype=torch.int32, device=coords[0].device)
        bh_find_bins(self.h, n, [c.data_ptr() for c in coords], out.data_ptr(), self._s(stream))
        return out

    def pack(self, out=None, stream=None):
        import torch
        n = bh_packed_size(self.h)
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=f"cuda:{self.device}")
        _check_cols([out], (torch.float64,), n, self.device, "out")
        bh_pack(self.h, out.data_ptr(), self._s(stream))
        return out

    def unpack(self, buf, stream=None):
        import torch
        _check_cols([buf], (torch.float64,), bh_packed_size(self.h), self.device, "buf")
        bh_unpack(self.h, buf.data_ptr(), self._s(stream))
        return self

    def read(self, stream=None, content_type: int = BH_CONTENT_F64) -> dict:
        return bh_read_as(self.h, content_type, self._s(stream))

    def strategy(self, weighted: bool) -> int:
        return bh_get_strategy(self.h, weighted)
