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
