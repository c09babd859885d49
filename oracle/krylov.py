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

Also:
  * right preconditioning, Algorithm 2: v_1 = s/‖s‖;
    y_j = q(A)v_j, u = q(A)y_j, w = A u; f_m = Y_m (H_m^{-1/2} e_1 ‖s‖) with
    the y_j stored.  Y_m is not orthonormal, so the estimate
    ‖f_m - f_{m-k}‖/‖f_m‖ is formed from the iterates themselves;
  * the plain (unpreconditioned, d = 1) method: q = None, w = A v_j;
  * two-pass Lanczos ("the first part does not store the basis
    vectors but just assembles the tridiagonal matrix H_m ... a second pass is
    done which then combines the anew computed basis vectors"): ``run_two_pass``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import chebyshev, contour_ls, newton
from .dense import invsqrt_e1
from .spmv import SquaredOperator


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
    if q is None:                       # plain method (d = 1): no preconditioner
        return v
    if isinstance(q, chebyshev.ChebPoly):
        return chebyshev.apply(q, op, v)
    if isinstance(q, contour_ls.LSPoly):
        return contour_ls.apply(q, op, v)
    return newton.apply(q, op, v)


def run(op, b: np.ndarray, q, *, func: str = "invsqrt", krylov: str = "cgs2",
        m_max: int = 60, stop: str = "fixed", tol: float = 1e-8, check_every: int = 1,
        x_ref: np.ndarray | None = None, breakdown_rtol: float = 1e-14,
        keep_basis: bool = False, precond: str = "left") -> Result:
    """Algorithm 1 (precond="left") or Algorithm 2 (precond="right"); q = None is
    the plain method.  ``stop`` in {"fixed", "est", "true"}; ``fixed`` runs m_max
    steps."""
    if precond not in ("left", "right"):
        raise ValueError(precond)
    right = precond == "right" and q is not None
    mv0 = op.mvms
    dt = np.result_type(b.dtype, op.dtype, np.float64)
    if isinstance(q, (newton.NewtonPoly, contour_ls.LSPoly)):
        dt = np.complex128
    s = op.matvec(b) if func == "sqrt" else b
    if right:
        c = s.astype(dt)                                             # Alg 2 line 2
    else:
        c = apply_q(q, op, s.astype(dt))                             # Alg 1 line 2
    beta0 = float(np.linalg.norm(c))
    ips = 0
    n = b.shape[0]
    V = np.zeros((n, m_max + 1), dtype=dt, order="F")   # columns contiguous
    Y = np.zeros((n, m_max), dtype=dt, order="F") if right else None
    H = np.zeros((m_max + 1, m_max), dtype=dt)
    V[:, 0] = c / beta0
    hermitian = krylov == "lanczos"
    hist = []
    y_prev = None
    x_prev = None
    term = "max_iter"
    m_done = 0
    y = None
    ref_norm = np.linalg.norm(x_ref) if x_ref is not None else None
    for j in range(m_max):
        if right:
            Y[:, j] = apply_q(q, op, V[:, j])                        # Alg 2 line 4: y_j = q(A) v_j
            w = apply_q(q, op, Y[:, j])                              #               u = q(A) y_j
            w = op.matvec(w)                                         #               w = A u
        else:
            w = op.matvec(V[:, j])                                   # Alg 1 line 4: u = A v_j
            w = apply_q(q, op, w)                                    #               y = q(A) u
            w = apply_q(q, op, w)                                    #               w = q(A) y
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
            xm = None
            if right:
                # Y_m is not orthonormal: the estimate needs the iterates
                xm = Y[:, :m] @ y
                if x_prev is not None:
                    est = float(np.linalg.norm(xm - x_prev) / np.linalg.norm(xm))
                x_prev = xm
            elif y_prev is not None:
                yp = np.zeros_like(y)
                yp[: len(y_prev)] = y_prev
                est = float(np.linalg.norm(yp - y) / np.linalg.norm(y))
            rec["est"] = est
            err = None
            if x_ref is not None:
                if xm is None:
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
    x = (Y[:, :m] if right else V[:, :m]) @ y                       # line 11
    res = Result(x=x, m=m, H=H[: m + 1, :m].copy(), beta0=beta0, y=y, term=term,
                 mvms=op.mvms - mv0, inner_products=ips, history=hist)
    if keep_basis:
        res.V = V[:, : m + 1].copy()
    return res


def run_two_pass(op, b: np.ndarray, q, *, func: str = "invsqrt", precond: str = "left",
                 m_max: int = 60, stop: str = "fixed", tol: float = 1e-8, check_every: int = 1,
                 breakdown_rtol: float = 1e-14) -> Result:
    """Two-pass Lanczos for Hermitian A, left or right
    preconditioning or plain (q = None).

    Pass 1: the Lanczos recurrence keeping only v_{j-1}, v_j; it assembles the
    tridiagonal H_m (α_j, β_j) and stops on ``stop`` ("fixed": m_max steps;
    "est": δ_m = ‖[y_{m-k}; 0] - y_m‖/‖y_m‖ ≤ tol -- for left preconditioning
    the paper's estimate; for right preconditioning, whose iterates cannot be
    formed without the basis, the same coefficient difference is used as a
    proxy, reading in DESIGN.md).  Then y_m = ‖c‖ H_m^{-1/2} e_1.
    Pass 2: the recurrence again from v_1 with the stored α, β (no inner
    products) regenerating v_1..v_m and accumulating x = Σ_j (y_m)_j v_j; with
    right preconditioning f_m = Y_m y_m = q(A)(V_m y_m), one
    extra application of q(A).
    """
    right = precond == "right" and q is not None
    mv0 = op.mvms
    dt = np.result_type(b.dtype, op.dtype, np.float64)
    s = op.matvec(b) if func == "sqrt" else b
    c = s.astype(dt) if right else apply_q(q, op, s.astype(dt))
    beta0 = float(np.linalg.norm(c))
    v1 = c / beta0

    def op_apply(v):
        if right:
            return op.matvec(apply_q(q, op, apply_q(q, op, v)))
        return apply_q(q, op, apply_q(q, op, op.matvec(v)))

    # ---- pass 1: assemble H_m ----
    alphas, betas = [], []
    v_prev, v = None, v1
    y_prev, y = None, None
    term, ips, m = "max_iter", 0, 0
    hist = []
    for j in range(m_max):
        w = op_apply(v)
        if j > 0:
            w = w - betas[j - 1] * v_prev
        alpha = float(np.vdot(v, w).real)
        w = w - alpha * v
        beta = float(np.linalg.norm(w))
        ips += 2
        alphas.append(alpha)
        betas.append(beta)
        m = j + 1
        broke = beta <= breakdown_rtol * beta0
        if broke or m % check_every == 0 or m == m_max:
            T = np.diag(alphas) + np.diag(betas[: m - 1], 1) + np.diag(betas[: m - 1], -1)
            y = invsqrt_e1(T, beta0, True)
            est = None
            if y_prev is not None:
                yp = np.zeros_like(y)
                yp[: len(y_prev)] = y_prev
                est = float(np.linalg.norm(yp - y) / np.linalg.norm(y))
            hist.append({"m": m, "mvms": op.mvms - mv0, "est": est, "err": None})
            y_prev = y
            if broke:
                term = "breakdown"
                break
            if stop == "est" and est is not None and est <= tol:
                term = "converged"
                break
        v_prev, v = v, w / beta
    T = np.diag(alphas[:m]) + np.diag(betas[: m - 1], 1) + np.diag(betas[: m - 1], -1)
    y = invsqrt_e1(T, beta0, True)
    H = np.zeros((m + 1, m))
    H[:m, :m] = T
    H[m, m - 1] = betas[m - 1]
    # ---- pass 2: regenerate the basis, x = V_m y_m ----
    x = y[0] * v1
    v_prev, v = None, v1
    for j in range(m - 1):
        w = op_apply(v)
        if j > 0:
            w = w - betas[j - 1] * v_prev
        w = w - alphas[j] * v
        v_prev, v = v, w / betas[j]
        x = x + y[j + 1] * v
    if right:
        x = apply_q(q, op, x)                                       # f_m = q(A) V_m y_m
    return Result(x=x, m=m, H=H, beta0=beta0, y=y, term=term, mvms=op.mvms - mv0,
                  inner_products=ips, history=hist)


def run_sign(op, b: np.ndarray, q, *, krylov: str = "cgs2", **kw) -> Result:
    """sign(Q) b = Q (Q^2)^{-1/2} b: Algorithm 1 (or 2) for
    the inverse square root of A = Q^2, applied as two mat-vecs with Q per
    application (2 mvms each, Table 2's unit), then one more mat-vec with Q.
    q approximates z^{-1/2} on spec(Q^2) (e.g. Ritz values of Q^2)."""
    res = run(SquaredOperator(op), b, q, func="invsqrt", krylov=krylov, **kw)
    res.x_invsqrt_sq = res.x
    res.x = op.matvec(res.x)
    res.mvms += 1
    return res


def find_m_star(op, b, q, *, func, krylov, m_max, tol, x_ref) -> Result:
    """O8: m* = first m (checked every step) with true relative error ≤ tol."""
    return run(op, b, q, func=func, krylov=krylov, m_max=m_max, stop="true", tol=tol,
               check_every=1, x_ref=x_ref)
