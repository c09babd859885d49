"""O1 / O3: the Chebyshev preconditioning polynomial q ≈ z^{-1/2} on [a, b].

PAPER.md:323-332 (§5.1, eq. cheb_expansion): q(z) = Σ_{i=0}^{k} c_i T_i^{[a,b]}(z)
with c_0 = (1/π)∫ w f T_0, c_i = (2/π)∫ w f T_i, w(z) = ((z-a)(b-z))^{-1/2}.

Reading Q2: the coefficient integrals are evaluated with the
d = deg+1 point Gauss-Chebyshev rule, i.e. q is the Chebyshev interpolant at the
d first-kind points.  This reproduces the paper's §3.2 numbers (κ_pre = 1.5153,
PAPER.md:222), which the exactly integrated series does not.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ChebPoly:
    a: float
    b: float
    c: np.ndarray  # c_0 .. c_deg

    @property
    def deg(self) -> int:
        return len(self.c) - 1


def coefficients(a: float, b: float, deg: int) -> ChebPoly:
    """PAPER.md:329 coefficients by d-point Gauss-Chebyshev quadrature (reading Q2).

    Substituting z = (a+b)/2 + (b-a)/2 cos θ turns (1/π)∫ w f T_i dz into
    (1/π)∫_0^π f(z(θ)) cos(iθ) dθ, evaluated at θ_l = π(l+1/2)/d, l = 0..d-1.
    """
    if not (0.0 < a < b):
        raise ValueError("need 0 < a < b")
    d = deg + 1
    theta = np.pi * (np.arange(d) + 0.5) / d
    z = (a + b) / 2.0 + (b - a) / 2.0 * np.cos(theta)
    fz = z ** -0.5
    c = np.empty(d)
    for i in range(d):
        c[i] = (2.0 / d) * np.sum(fz * np.cos(i * theta))
    c[0] /= 2.0
    return ChebPoly(float(a), float(b), c)


def evaluate(q: ChebPoly, z) -> np.ndarray:
    """Scalar q(z) = Σ c_i T_i(t), t = (2z - a - b)/(b - a), by the forward
    three-term recurrence T_{i+1} = 2t T_i - T_{i-1}."""
    z = np.asarray(z, dtype=np.float64)
    t = (2.0 * z - q.a - q.b) / (q.b - q.a)
    T0 = np.ones_like(t)
    acc = q.c[0] * T0
    if q.deg == 0:
        return acc
    T1 = t
    acc = acc + q.c[1] * T1
    for i in range(1, q.deg):
        T0, T1 = T1, 2.0 * t * T1 - T0
        acc = acc + q.c[i + 1] * T1
    return acc


def certificate_points(a: float, b: float) -> np.ndarray:
    """Check grid for the positivity certificate:
    z_k = a + (b-a) k/1000, k = 0..1000 (1001 points including both endpoints)."""
    return a + (b - a) * np.arange(1001) / 1000.0


def certify(q: ChebPoly) -> float:
    """min q on the check grid; q > 0 on [a, b] ⇒ ((q(A))^2)^{1/2} = q(A)."""
    return float(np.min(evaluate(q, certificate_points(q.a, q.b))))


def apply(q: ChebPoly, op, v: np.ndarray) -> np.ndarray:
    """O3: q(A)v via the forward recurrence t_0 = v, t_1 = Â v,
    t_{i+1} = 2 Â t_i - t_{i-1}, q(A)v = Σ c_i t_i with Â = αA + βI,
    α = 2/(b-a), β = -(a+b)/(b-a).  Exactly deg mat-vecs (the device uses the
    Clenshaw form instead, so rounding differs)."""
    alpha = 2.0 / (q.b - q.a)
    beta = -(q.a + q.b) / (q.b - q.a)

    def Ahat(x):
        return alpha * op.matvec(x) + beta * x

    acc = q.c[0] * v
    if q.deg == 0:
        return acc
    t_prev = v
    t_cur = Ahat(v)
    acc = acc + q.c[1] * t_cur
    for i in range(1, q.deg):
        t_prev, t_cur = t_cur, 2.0 * Ahat(t_cur) - t_prev
        acc = acc + q.c[i + 1] * t_cur
    return acc
