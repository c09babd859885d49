"""O2 / O3: the Ritz-value interpolation polynomial in Newton form on Lejà-ordered
nodes (§5.2).

q is "the polynomial of degree d-1 that interpolates 1/sqrt(z) at the d Ritz
values" of H_d from d Arnoldi steps with A started from b,
represented "in its Newton form based on a Lejà ordering of the Ritz values"
(PAPER.md:354).  Conventions (readings): Lejà order starts at the
node of maximum modulus and then greedily maximises Σ log|θ - θ_chosen|; ties go
to the smaller index after sorting nodes by (Re, Im) (SPEC design decision).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class BranchError(ValueError):
    """A node or eigenvalue lies on the branch cut (-inf, 0]."""


@dataclass
class NewtonPoly:
    nodes: np.ndarray  # θ_0 .. θ_deg (Lejà order), complex
    dd: np.ndarray     # divided differences f[θ_0..θ_j], complex

    @property
    def deg(self) -> int:
        return len(self.nodes) - 1


def arnoldi_plain(op, b: np.ndarray, steps: int):
    """``steps`` Arnoldi steps with A itself (no polynomial), CGS2 orthogonalisation.

    Returns (H[steps+1, steps], inner_products).  This is the "d additional
    Arnoldi steps" of PAPER.md:340 that cost d mat-vecs.
    """
    n = b.shape[0]
    dt = np.result_type(b.dtype, op.dtype, np.float64)
    V = np.zeros((n, steps + 1), dtype=dt)
    H = np.zeros((steps + 1, steps), dtype=dt)
    V[:, 0] = b / np.linalg.norm(b)
    ips = 1
    for j in range(steps):
        w = op.matvec(V[:, j])
        Vj = V[:, : j + 1]
        h = Vj.conj().T @ w
        w = w - Vj @ h
        g = Vj.conj().T @ w
        w = w - Vj @ g
        H[: j + 1, j] = h + g
        H[j + 1, j] = np.linalg.norm(w)
        ips += 2 * (j + 1) + 1
        V[:, j + 1] = w / H[j + 1, j]
    return H, ips


def ritz_values(H_square: np.ndarray) -> np.ndarray:
    """θ = eig(H_d); rejects any θ on (-inf, 0].

    Pinned by closed forms of finite Arnoldi runs (tests/test_oracle_poly.py::
    test_ritz_values_closed_form_partial_krylov: the 1D Laplacian from e_1 has
    H_d = T_d and Ritz values 2 - 2cos(k pi/(d+1)); a start vector in a
    d-dimensional invariant subspace gives those d eigenvalues).  For generic
    inputs the values carry ~1e-11 of rounding, so GPU-vs-oracle
    node comparisons are multiset comparisons at 1e-8 and H/x parity imports
    the oracle's q."""
    theta = np.linalg.eigvals(H_square).astype(np.complex128)
    for t in theta:
        if abs(t.imag) <= 1e-13 * max(abs(t), 1e-300) and t.real <= 0.0:
            raise BranchError(f"Ritz value {t} on the branch cut")
    return theta


def harmonic_ritz_values(H: np.ndarray) -> np.ndarray:
    """Harmonic Ritz values: the eigenvalues of
    H~_d = H_d + h_{d+1,d}^2 H_d^{-*} e_d e_d^*, from the (d+1) x d Arnoldi
    Hessenberg H.  Rejects any value on (-inf, 0]."""
    d = H.shape[1]
    Hd = H[:d, :d].astype(np.complex128)
    h = H[d, d - 1]
    ed = np.zeros(d, dtype=np.complex128)
    ed[-1] = 1.0
    f = np.linalg.solve(Hd.conj().T, ed)          # H_d^{-*} e_d
    Ht = Hd + (abs(h) ** 2) * np.outer(f, ed.conj())
    return ritz_values(Ht)


def leja_order(theta: np.ndarray) -> np.ndarray:
    """Lejà ordering: max modulus first, then argmax Σ log|θ - θ_i|."""
    theta = np.asarray(theta, dtype=np.complex128)
    order0 = np.lexsort((theta.imag, theta.real))  # sort by (Re, Im)
    pts = theta[order0]
    n = len(pts)
    chosen = [int(np.argmax(np.abs(pts)))]
    remaining = [i for i in range(n) if i != chosen[0]]
    while remaining:
        best, best_val = None, -np.inf
        for i in remaining:
            s = 0.0
            for j in chosen:
                s += np.log(abs(pts[i] - pts[j]))
            if s > best_val:
                best, best_val = i, s
        chosen.append(best)
        remaining.remove(best)
    return pts[chosen]


def divided_differences(nodes: np.ndarray) -> np.ndarray:
    """Newton divided differences of f(z) = z^{-1/2} (principal branch):
    dd = f(θ); for k = 1..d-1: dd[k:] = (dd[k:] - dd[k-1:-1]) / (θ[k:] - θ[:-k])."""
    nodes = np.asarray(nodes, dtype=np.complex128)
    dd = 1.0 / np.sqrt(nodes)
    d = len(nodes)
    for k in range(1, d):
        dd[k:] = (dd[k:] - dd[k - 1:-1]) / (nodes[k:] - nodes[:-k])
    return dd


def from_nodes(nodes) -> NewtonPoly:
    ordered = leja_order(np.asarray(nodes, dtype=np.complex128))
    return NewtonPoly(ordered, divided_differences(ordered))


def ritz_newton(op, b: np.ndarray, deg: int, harmonic: bool = False):
    """Full O2 construction: deg+1 Arnoldi steps from b, Ritz values (or
    harmonic Ritz values), Lejà, dd.
    Returns (NewtonPoly, mvms, inner_products)."""
    d = deg + 1
    m0 = op.mvms
    H, ips = arnoldi_plain(op, b, d)
    theta = harmonic_ritz_values(H) if harmonic else ritz_values(H[:d, :d])
    return from_nodes(theta), op.mvms - m0, ips


def evaluate(q: NewtonPoly, z) -> np.ndarray:
    """Scalar q(z) = Σ_j dd_j Π_{i<j} (z - θ_i)."""
    z = np.asarray(z, dtype=np.complex128)
    acc = np.zeros_like(z)
    prod = np.ones_like(z)
    for j in range(q.deg + 1):
        acc = acc + q.dd[j] * prod
        prod = prod * (z - q.nodes[j])
    return acc


def apply(q: NewtonPoly, op, v: np.ndarray) -> np.ndarray:
    """O3: q(A)v via the forward Newton basis p_0 = v, p_{j+1} = (A - θ_j) p_j,
    q(A)v = Σ dd_j p_j (the device uses the Horner form).
    Exactly deg mat-vecs."""
    v = v.astype(np.complex128)
    p = v
    acc = q.dd[0] * p
    for j in range(q.deg):
        p = op.matvec(p) - q.nodes[j] * p
        acc = acc + q.dd[j + 1] * p
    return acc
