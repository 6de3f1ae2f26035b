"""Oracle of the fused Filter + Define path (bh_fill_expr) — TEST INFRASTRUCTURE ONLY.

Plain numpy evaluation of the register program, op by op over whole columns (IEEE
binary64: + - * / sqrt are correctly rounded in numpy as in CUDA), then the selection
(RDataFrame Filter: only passing events reach the histogram) and the
plain oracle fill of the derived coordinates."""
import numpy as np

from . import OracleHist


def run_program(cols, prog, n):
    r = [np.asarray(c, dtype=np.float64) for c in cols] + [np.zeros(n) for _ in range(16 - len(cols))]
    with np.errstate(all="ignore"):
        for name, dst, a, b, c, imm in prog:
            A, B = r[a], r[b]
            if name == "const":
                v = np.full(n, imm)
            elif name == "copy":
                v = A.copy()
            elif name == "add":
                v = A + B
            elif name == "sub":
                v = A - B
            elif name == "mul":
                v = A * B
            elif name == "div":
                v = A / B
            elif name == "sqrt":
                v = np.sqrt(A)
            elif name == "abs":
                v = np.abs(A)
            elif name == "neg":
                v = -A
            elif name == "min":
                v = np.fmin(A, B)
            elif name == "max":
                v = np.fmax(A, B)
            elif name in ("lt", "le", "gt", "ge", "eq", "ne"):
                v = {"lt": A < B, "le": A <= B, "gt": A > B, "ge": A >= B, "eq": A == B, "ne": A != B}[name]
                v = v.astype(np.float64)
            elif name == "and":
                v = ((A != 0) & (B != 0)).astype(np.float64)
            elif name == "or":
                v = ((A != 0) | (B != 0)).astype(np.float64)
            elif name == "not":
                v = (~(A != 0)).astype(np.float64)
            elif name == "select":
                v = np.where(A != 0, B, r[c])
            else:
                raise ValueError(name)
            r[dst] = v
    return r


def fill_expr(axes, cols, prog, axis_regs, weight_reg=-1, filter_reg=-1):
    n = len(cols[0]) if cols else 0
    r = run_program(cols, prog, n)
    sel = np.ones(n, bool) if filter_reg < 0 else (r[filter_reg] != 0)
    coords = [r[k][sel] for k in axis_regs]
    w = None if weight_reg < 0 else r[weight_reg][sel]
    return OracleHist(axes).fill(coords, w)
