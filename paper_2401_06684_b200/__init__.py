"""B200-native polynomially preconditioned f(A)b (arXiv 2401.06684).

The hot path -- left polynomially preconditioned Arnoldi/Lanczos for A^{-1/2}b
and A^{1/2}b = A^{-1/2}(Ab) (Algorithm 1) -- lives in
the C-ABI library ``libppf.so`` (include/ppf.h; CUDA kernels for sm_100a plus
host C++).  ``api`` is a thin ctypes binding with the same names.
"""
from . import _lib  # noqa: F401
from .api import (  # noqa: F401
    Context,
    Matrix,
    Plan,
    Poly,
    RunReport,
    Workspace,
    dense_invsqrt_e1,
    hessenberg,
    history,
    nccl_unique_id,
    run,
    run_host,
)
