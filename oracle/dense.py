"""O6: y_m = β0 · H_m^{-1/2} e_1 for the small projected matrix.

Principal branch.  Hermitian H: eigh, y = β0 S (Θ^{-1/2} ∘ S[0,:]^*).
Non-Hermitian: eig, y = β0 X (Λ^{-1/2} ∘ X^{-1} e_1); if cond(X) > 1e8 fall back
to scipy.linalg.sqrtm followed by a linear solve ("computing
H_m^{1/2} ... and then solving a linear system").  Raises BranchError if an
eigenvalue lies on (-inf, 0].
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .newton import BranchError


def _check_branch(lam):
    for t in np.atleast_1d(lam):
        t = complex(t)
        if abs(t.imag) <= 1e-14 * max(abs(t), 1e-300) and t.real <= 0.0:
            raise BranchError(f"eigenvalue {t} of H_m on (-inf, 0]")


def invsqrt_e1(H: np.ndarray, beta0: float, hermitian: bool) -> np.ndarray:
    m = H.shape[0]
    if hermitian:
        Hs = (H + H.conj().T) / 2.0
        theta, S = np.linalg.eigh(Hs)
        _check_branch(theta)
        return beta0 * (S @ (theta ** -0.5 * S[0, :].conj()))
    lam, X = np.linalg.eig(H)
    _check_branch(lam)
    e1 = np.zeros(m, dtype=np.complex128)
    e1[0] = 1.0
    if np.linalg.cond(X) <= 1e8:
        y = beta0 * (X @ (lam.astype(np.complex128) ** -0.5 * np.linalg.solve(X, e1)))
    else:
        R = sla.sqrtm(H.astype(np.complex128))
        y = beta0 * np.linalg.solve(R, e1)
    if np.isrealobj(H):
        return y.real.copy()
    return y


def invsqrt_dense(A: np.ndarray) -> np.ndarray:
    """Principal A^{-1/2} of a small dense matrix by eigendecomposition (test helper)."""
    lam, X = np.linalg.eig(A)
    _check_branch(lam)
    return X @ np.diag(lam.astype(np.complex128) ** -0.5) @ np.linalg.inv(X)


def sign_dense(Q: np.ndarray) -> np.ndarray:
    """sign(Q) = X diag(sign(Re λ)) X^{-1} from the eigendecomposition
    (Higham, Functions of Matrices, §5; the definition behind),
    requiring no eigenvalue on the imaginary axis; Hermitian Q uses eigh."""
    if np.allclose(Q, Q.conj().T, rtol=0, atol=1e-14 * np.abs(Q).max()):
        lam, X = np.linalg.eigh(Q)
        if np.any(lam == 0):
            raise ValueError("eigenvalue on the imaginary axis")
        return (X * np.sign(lam)) @ X.conj().T
    lam, X = np.linalg.eig(Q)
    if np.any(np.abs(lam.real) <= 1e-14 * np.abs(lam).max()):
        raise ValueError("eigenvalue on the imaginary axis")
    return (X * np.sign(lam.real)) @ np.linalg.inv(X)
