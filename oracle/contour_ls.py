"""Least-squares preconditioning polynomial on a contour (§5.3).

ORACLE -- test infrastructure only (see oracle/__init__.py).

Step by step in the paper's notation:
  * Γ is a contour around the spectrum that excludes (-inf, 0],
    discretised into ω = {z_1, ..., z_N}.
  * ⟨p1, p2⟩_ω = Σ_i p1(z_i) conj(p2(z_i)) (eq. polynomial_inner_product).
  * q = argmin_{q ∈ P_{d-1}} ‖z^{-1/2} - q(z)‖_ω.
  * The Arnoldi process on diag(z_1..z_N) from [1..1]^T / N^{1/2} builds the
    orthonormal basis polynomials p_0..p_{d-1}: the k-th Arnoldi vector is
    vec(p_{k-1}), with the Hessenberg recurrence
    z p_{k-1}(z) = Σ_{i<=k} h_{i,k-1} p_i(z).
  * α = P_d^* vec(z^{-1/2}), so q = Σ_j α_j p_j.
  * q(A)v by the same recurrence with A in place of z ("an Arnoldi-like process
    that does not require knowledge of P_d ... d-1 matrix-vector products with
    A and O(d^2) vector operations, but no inner products").
  * Certificate: Re q(z_i) > 0 at every contour point.
The arithmetic here is the paper's (full recurrence, no short-cut); the device
path uses an equivalent Newton form of the same polynomial.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class LSPoly:
    points: np.ndarray   # z_1..z_N on Γ (complex)
    H: np.ndarray        # (d x d-1) Hessenberg of the Arnoldi process on diag(z)
    alpha: np.ndarray    # coefficients in the orthonormal basis p_0..p_{d-1}
    p0: complex          # p_0(z) = 1/sqrt(N)

    @property
    def deg(self) -> int:
        return len(self.alpha) - 1


def circle(center: complex, radius: float, N: int) -> np.ndarray:
    """N equispaced points on |z - center| = radius."""
    t = 2.0 * np.pi * np.arange(N) / N
    return center + radius * np.exp(1j * t)


def construct(points, deg: int) -> LSPoly:
    """Arnoldi on diag(points) (CGS with one reorthogonalisation),
    then α = P^* vec(z^{-1/2}) (principal branch)."""
    z = np.asarray(points, dtype=np.complex128)
    N = len(z)
    d = deg + 1
    if d >= N:
        raise ValueError("need deg + 1 < N")
    if np.any((np.abs(z.imag) <= 1e-14 * np.abs(z)) & (z.real <= 0)):
        raise ValueError("contour touches the branch cut (-inf, 0]")
    P = np.zeros((N, d), dtype=np.complex128)
    H = np.zeros((d, d - 1), dtype=np.complex128)
    P[:, 0] = 1.0 / np.sqrt(N)
    for k in range(1, d):
        w = z * P[:, k - 1]
        h = P[:, :k].conj().T @ w
        w = w - P[:, :k] @ h
        g = P[:, :k].conj().T @ w
        w = w - P[:, :k] @ g
        H[:k, k - 1] = h + g
        H[k, k - 1] = np.linalg.norm(w)
        P[:, k] = w / H[k, k - 1]
    f = z ** -0.5
    alpha = P.conj().T @ f
    return LSPoly(points=z, H=H, alpha=alpha, p0=1.0 / np.sqrt(N))


def _recurrence(q: LSPoly, mul, v):
    """Σ_j α_j p_j(X) v with p_0 = 1/sqrt(N) and
    p_k = (X p_{k-1} - Σ_{i<k} h_{i,k-1} p_i) / h_{k,k-1}."""
    basis = [q.p0 * v]
    acc = q.alpha[0] * basis[0]
    for k in range(1, q.deg + 1):
        w = mul(basis[k - 1])
        for i in range(k):
            w = w - q.H[i, k - 1] * basis[i]
        basis.append(w / q.H[k, k - 1])
        acc = acc + q.alpha[k] * basis[k]
    return acc


def evaluate(q: LSPoly, z) -> np.ndarray:
    """Scalar q(z) by the same recurrence (X = z)."""
    z = np.asarray(z, dtype=np.complex128)
    return _recurrence(q, lambda x: z * x, np.ones_like(z))


def apply(q: LSPoly, op, v: np.ndarray) -> np.ndarray:
    """q(A)v: deg mat-vecs, O(deg^2) vector operations, no inner products."""
    return _recurrence(q, op.matvec, v.astype(np.complex128))


def certify(q: LSPoly) -> float:
    """min Re q(z_i) over the contour points; must be > 0."""
    return float(np.min(evaluate(q, q.points).real))


def ritz_polygon(theta, r_min: float, step: float) -> np.ndarray:
    """Contour from Ritz values ("constructed as a polygon from the
    Ritz values"): the boundary of the Ritz values --
    reading (Q29): their convex hull, counter-clockwise (MATLAB's
    `boundary`, a shrink-factor hull, is not reproducible); a hull of collinear
    values degenerates to the segment between the extremes, traversed both
    ways -- then every part closer to 0 than r_min replaced by the circular
    arc of radius r_min, discretised in steps of (approximately) uniform
    length `step`.  Points on (-inf, 0] are never produced for r_min > 0 unless
    the hull surrounds 0 (rejected)."""
    th = np.asarray(theta, dtype=np.complex128)
    pts = np.unique(np.round(np.stack([th.real, th.imag], 1), 15), axis=0)
    if len(pts) == 1:
        raise ValueError("need at least two distinct Ritz values")
    # Andrew's monotone chain convex hull
    P = sorted(map(tuple, pts))

    def cross(o, a, b):
        return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])
    lower, upper = [], []
    for p in P:
        while len(lower) >= 2 and cross(lower[-2], lower[-1], p) <= 0:
            lower.pop()
        lower.append(p)
    for p in reversed(P):
        while len(upper) >= 2 and cross(upper[-2], upper[-1], p) <= 0:
            upper.pop()
        upper.append(p)
    hull = lower[:-1] + upper[:-1]
    verts = np.array([complex(x, y) for x, y in hull])
    if len(verts) == 2:                       # collinear: there and back
        verts = np.array([verts[0], verts[1]])
    # densify the closed polygon
    out = []
    nv = len(verts)
    for i in range(nv):
        a, c = verts[i], verts[(i + 1) % nv]
        L = abs(c - a)
        k = max(1, int(np.ceil(L / step)))
        out.extend(a + (c - a) * np.arange(k) / k)
    z = np.array(out)
    # the hull must not surround 0 (then every contour would meet the branch cut)
    wind = np.sum(np.angle(np.roll(z, -1) / z))
    if abs(wind) > np.pi:
        raise ValueError("the Ritz polygon surrounds 0")
    # minimum distance: project points closer than r_min radially onto the
    # circle, then resample that arc uniformly
    close = np.abs(z) < r_min
    if np.any(close):
        z = np.where(close, r_min * np.exp(1j * np.angle(z)), z)
        # uniform resampling along the (modified) closed curve
        seg = np.abs(np.diff(np.concatenate([z, z[:1]])))
        total = seg.sum()
        s = np.concatenate([[0.0], np.cumsum(seg)])
        zc = np.concatenate([z, z[:1]])
        tgt = np.arange(0.0, total, step)
        idx = np.clip(np.searchsorted(s, tgt, side="right") - 1, 0, len(z) - 1)
        frac = (tgt - s[idx]) / np.where(seg[idx] > 0, seg[idx], 1.0)
        z = zc[idx] + frac * (zc[idx + 1] - zc[idx])
        # chords of the arc dip below r_min by O(step^2 / r_min): back onto the circle
        z = np.where(np.abs(z) < r_min, r_min * np.exp(1j * np.angle(z)), z)
    return z
