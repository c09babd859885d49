"""Seeded right-hand sides (reading Q13: b ~ N(0,1) i.i.d., complex CN(0,1) with
Re, Im ~ N(0, 1/2); not normalised -- results are linear in b)."""
from __future__ import annotations

import numpy as np


def gaussian_vector(n: int, seed: int, complex_: bool = False) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if not complex_:
        return rng.standard_normal(n)
    z = rng.standard_normal((n, 2))
    return (z[:, 0] + 1j * z[:, 1]) / np.sqrt(2.0)


def sample_indices(n: int, k: int, seed: int) -> np.ndarray:
    """Sorted distinct indices for sampled full-size comparisons: k seeded
    random rows plus the first and last 1024 rows (the ragged tail of the last
    SELL slice / CGS2 chunk).  Selection only -- no arithmetic of the method."""
    rng = np.random.default_rng(seed)
    pick = rng.choice(n, size=min(k, n), replace=False)
    edge = np.concatenate([np.arange(min(1024, n)), np.arange(max(0, n - 1024), n)])
    return np.unique(np.concatenate([pick, edge])).astype(np.int64)


def probe_projections(x: np.ndarray, k: int, seed: int, chunk: int = 1 << 20) -> np.ndarray:
    """G x for a k x n matrix G of i.i.d. N(0,1) entries generated chunk by
    chunk (column block c from default_rng([seed, c])), without storing G.
    ||G d|| / sqrt(k) estimates ||d|| for any vector d (relative spread about
    1/sqrt(2k)), so comparing G x_a with G x_b bounds ||x_a - x_b|| from k
    numbers per side.  A probe, not part of the method."""
    n = x.shape[0]
    out = np.zeros(k, dtype=np.result_type(x.dtype, np.float64))
    for c, lo in enumerate(range(0, n, chunk)):
        hi = min(n, lo + chunk)
        G = np.random.default_rng([seed, c]).standard_normal((k, hi - lo))
        out += G @ x[lo:hi]
    return out
