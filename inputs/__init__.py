"""Seeded synthetic inputs shared by the CUDA path's tests/bench and by the oracle.

This package holds ONLY problem definitions: sparse operators (CSR arrays), their
closed-form spectral intervals (the paper's P:419 formula and its 2D / convection-
diffusion analogues), and seeded right-hand sides.  It contains none of the
method's arithmetic (no polynomial, no Krylov step, no f(H_m)), so that both the
CUDA library and ``oracle/`` can consume the same inputs without sharing code.
"""
from .operators import (  # noqa: F401
    CSR,
    laplacian,
    convdiff,
    wilson_dirac,
    haar_su3,
    laplacian_interval,
    convdiff_interval,
)
from .vectors import gaussian_vector  # noqa: F401
from .configs import CONFIGS, Config, build  # noqa: F401
