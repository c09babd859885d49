"""Measured parity bars (reading Q19): where the Krylov process itself
amplifies rounding, the H / x bars are 10x the gap between the oracle's run
and a second oracle run that differs from it ONLY in rounding -- here every
mat-vec formed in extended precision and rounded once to fp64 / complex128
(``LDOperator``), a legitimate alternative rounding of the same product.
Test infrastructure: wraps oracle/ objects, holds no method arithmetic."""
from __future__ import annotations

import numpy as np


class LDOperator:
    """The oracle's Operator interface; y = A x accumulated in long double and
    rounded once."""

    def __init__(self, A_csr):
        S = A_csr.tocsr()
        self.n = S.shape[0]
        self.dtype = S.dtype
        self.mvms = 0
        self._S = S.astype(np.clongdouble if np.iscomplexobj(S.data) else np.longdouble)

    def matvec(self, x):
        self.mvms += 1
        out = np.result_type(self.dtype, x.dtype)
        if np.iscomplexobj(x) and not np.iscomplexobj(self._S.data):
            y = (self._S @ x.real.astype(np.longdouble)).astype(np.float64) + \
                1j * (self._S @ x.imag.astype(np.longdouble)).astype(np.float64)
            return y.astype(out)
        xl = x.astype(np.clongdouble if np.iscomplexobj(x) else np.longdouble)
        return np.asarray(self._S @ xl).astype(out)

    __matmul__ = matvec


def gaps(res_o, res_2):
    """(H gap normwise, x gap relative) between two oracle results."""
    h = float(np.abs(res_2.H - res_o.H).max() / np.abs(res_o.H).max())
    x = float(np.linalg.norm(res_2.x - res_o.x) / np.linalg.norm(res_o.x))
    return h, x


def measured_bars(res_o, rerun, A_csr, h_floor=1e-11, x_floor=1e-10):
    """rerun(op) repeats the oracle run of res_o with operator ``op``; returns
    (h_bar, x_bar, h_gap, x_gap)."""
    r2 = rerun(LDOperator(A_csr))
    hg, xg = gaps(res_o, r2)
    return max(h_floor, 10 * hg), max(x_floor, 10 * xg), hg, xg
