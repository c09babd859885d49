"""O9: y = A x with SciPy's CSR kernel, split into row chunks over a thread pool.

SciPy's ``csr_matvec`` releases the GIL and each output row is computed by the
same sequential loop regardless of chunking, so the result is bit-identical to a
single-threaded product.  The mat-vec is the paper's cost unit
("mvm").
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class Operator:
    """Wraps a scipy CSR matrix; counts mat-vecs."""

    def __init__(self, A_csr, threads: int | None = None):
        self.A = A_csr.tocsr()
        self.n = self.A.shape[0]
        self.dtype = self.A.dtype
        self.threads = threads or _threads()
        self.mvms = 0
        rows = self.n
        nchunk = self.threads if rows >= 65536 else 1
        bounds = np.linspace(0, rows, nchunk + 1).astype(np.int64)
        self.chunks = [(int(bounds[i]), int(bounds[i + 1])) for i in range(nchunk)]
        self.blocks = [self.A[lo:hi] for lo, hi in self.chunks]
        self.pool = ThreadPoolExecutor(self.threads) if nchunk > 1 else None

    def matvec(self, x: np.ndarray) -> np.ndarray:
        self.mvms += 1
        out_dtype = np.result_type(self.dtype, x.dtype)
        if self.pool is None:
            return np.asarray(self.A @ x, dtype=out_dtype)
        y = np.empty(self.n, dtype=out_dtype)

        def work(i):
            lo, hi = self.chunks[i]
            y[lo:hi] = self.blocks[i] @ x

        list(self.pool.map(work, range(len(self.chunks))))
        return y

    __matmul__ = matvec


class SquaredOperator:
    """A = Q^2 applied as two consecutive mat-vecs with Q ("we
    rather compute A^2 x for a given vector x as two consecutive mvms"); each
    application counts 2 mvms, the unit of Table 2."""

    def __init__(self, op: Operator):
        self.op = op
        self.n = op.n
        self.dtype = op.dtype

    @property
    def mvms(self) -> int:
        return self.op.mvms

    def matvec(self, x: np.ndarray) -> np.ndarray:
        return self.op.matvec(self.op.matvec(x))

    __matmul__ = matvec
