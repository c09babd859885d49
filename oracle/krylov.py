"""O4, O5, O7, O8: m steps of left polynomially preconditioned Arnoldi / Lanczos
for A^{-1/2}b (Algorithm 1) and A^{1/2}b = A^{-1/2}(Ab)
(PAPER.md:237-241).

Step by step, in the paper's notation:
  line 1  q given (chebyshev.ChebPoly or newton.NewtonPoly)
  line 2  c = q(A)s, v_1 = c/‖c‖, with s = b (inverse sqrt) or s = A b (sqrt)
  line 4  u = A v_j, y = q(A)u, w = q(A)y            (three stages)
  line 5-7 orthogonalise; reading Q8: Lanczos three-term recurrence for
          Hermitian A, classical Gram-Schmidt with one reorthogonalisation (CGS2)
          otherwise; h_{ij} = <w, v_i> = v_i^H w (reading Q7)
  line 8-9 h_{j+1,j} = ‖w‖, v_{j+1} = w / h_{j+1,j}
  line 11 f_m = V_m (H_m^{-1/2} e_1 ‖c‖)
Stopping (reading Q11/Q12): every ``check_every`` steps compute y_m; the paper's
estimate δ_m = ‖[y_{m-k}; 0] - y_m‖ / ‖y_m‖ (= ‖f_m - f_{m-k}‖/‖f_m‖ because V is
orthonormal) and, when a reference is given, the true error.
Breakdown (reading Q9): h_{j+1,j} ≤ 1e-14 β0 ends the iteration.
Counters (reading): mvms in the paper's unit; inner
products (norms included, the initial ‖c‖ not, matching Table 1's 2 per
Lanczos iteration): Lanczos 2 per step (α, ‖w‖), CGS2 2j+1 at
step j (h, g, ‖w‖).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import chebyshev, newton
from .dense import invsqrt_e1


@dataclass
class Result:
    x: np.ndarray
    m: int
    H: np.ndarray          # (m+1) x m
    beta0: float
    y: np.ndarray
    term: str              # "converged" | "max_iter" | "breakdown"
    mvms: int
    inner_products: int
    history: list = field(default_factory=list)  # dicts: m, est, err, mvms


def apply_q(q, op, v):
    if isinstance(q, chebyshev.ChebPoly):
        return chebyshev.apply(q, op, v)
    return newton.apply(q, op, v)


def run(op, b: np.ndarray, q, *, func: str = "invsqrt", krylov: str = "cgs2",
        m_max: int = 60, stop: str = "fixed", tol: float = 1e-8, check_every: int = 1,
        x_ref: np.ndarray | None = None, breakdown_rtol: float = 1e-14,
        keep_basis: bool = False) -> Result:
    """Algorithm 1.  ``stop`` in {"fixed", "est", "true"}; ``fixed`` runs m_max steps."""
    mv0 = op.mvms
    dt = np.result_type(b.dtype, op.dtype, np.float64)
    if isinstance(q, newton.NewtonPoly):
        dt = np.complex128
    s = op.matvec(b) if func == "sqrt" else b
    c = apply_q(q, op, s.astype(dt))                               # line 2
    beta0 = float(np.linalg.norm(c))
    ips = 0
    n = b.shape[0]
    V = np.zeros((n, m_max + 1), dtype=dt)
    H = np.zeros((m_max + 1, m_max), dtype=dt)
    V[:, 0] = c / beta0
    hermitian = krylov == "lanczos"
    hist = []
    y_prev = None
    term = "max_iter"
    m_done = 0
    y = None
    ref_norm = np.linalg.norm(x_ref) if x_ref is not None else None
    for j in range(m_max):
        w = op.matvec(V[:, j])                                       # line 4: u = A v_j
        w = apply_q(q, op, w)                                        #          y = q(A) u
        w = apply_q(q, op, w)                                        #          w = q(A) y
        if hermitian:
            if j > 0:
                w = w - H[j, j - 1] * V[:, j - 1]
            alpha = np.vdot(V[:, j], w)
            w = w - alpha * V[:, j]
            H[j, j] = alpha.real if np.iscomplexobj(alpha) else alpha
            if j > 0:
                H[j - 1, j] = H[j, j - 1]
            ips += 2
        else:
            Vj = V[:, : j + 1]
            h = Vj.conj().T @ w
            w = w - Vj @ h
            g = Vj.conj().T @ w
            w = w - Vj @ g
            H[: j + 1, j] = h + g
            ips += 2 * (j + 1) + 1
        hn = float(np.linalg.norm(w))
        H[j + 1, j] = hn
        m_done = j + 1
        broke = hn <= breakdown_rtol * beta0
        if not broke:
            V[:, j + 1] = w / hn
        m = m_done
        if broke or m % check_every == 0 or m == m_max:
            y = invsqrt_e1(H[:m, :m], beta0, hermitian)
            rec = {"m": m, "mvms": op.mvms - mv0}
            est = None
            if y_prev is not None:
                yp = np.zeros_like(y)
                yp[: len(y_prev)] = y_prev
                est = float(np.linalg.norm(yp - y) / np.linalg.norm(y))
            rec["est"] = est
            err = None
            if x_ref is not None:
                xm = V[:, :m] @ y
                err = float(np.linalg.norm(xm - x_ref) / ref_norm)
            rec["err"] = err
            hist.append(rec)
            y_prev = y
            if broke:
                term = "breakdown"
                break
            if stop == "est" and est is not None and est <= tol:
                term = "converged"
                break
            if stop == "true" and err is not None and err <= tol:
                term = "converged"
                break
    m = m_done
    if y is None or len(y) != m:
        y = invsqrt_e1(H[:m, :m], beta0, hermitian)
    x = V[:, :m] @ y                                                # line 11
    res = Result(x=x, m=m, H=H[: m + 1, :m].copy(), beta0=beta0, y=y, term=term,
                 mvms=op.mvms - mv0, inner_products=ips, history=hist)
    if keep_basis:
        res.V = V[:, : m + 1].copy()
    return res


def find_m_star(op, b, q, *, func, krylov, m_max, tol, x_ref) -> Result:
    """O8: m* = first m (checked every step) with true relative error ≤ tol."""
    return run(op, b, q, func=func, krylov=krylov, m_max=m_max, stop="true", tol=tol,
               check_every=1, x_ref=x_ref)
