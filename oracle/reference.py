"""R1-R4: reference solutions x* = f(A)b, f the principal z^{∓1/2}.

R1 Dirichlet Laplacian (C1, C3): the orthonormal DST-I diagonalises the 1D factor
   tridiag(-1, 2, -1) with eigenvalues μ_k = 2 - 2cos(kπ/(N+1)), so
   x* = S^{⊗dim} diag(f(Σ μ)) S^{⊗dim} b  (S symmetric, S^2 = I).
R2 Centred convection-diffusion (C2, C4): the 1D factor is D_ρ T_s D_ρ^{-1} with
   ρ = sqrt((1+P)/(1-P)), P = βh/2, T_s symmetric with eigenvalues
   σ_k = (2 - 2 sqrt(1-P^2) cos(kπ/(N+1)))/h^2, so
   x* = D S diag(f(Σσ)) S D^{-1} b with D = D_ρ^{⊗dim}; evaluated in long double
   because cond(D) = ρ^{dim(N-1)} (4.2e8 for C2).
R3 Free Wilson operator and pure gauge: D(p) = a(p) I + i S(p),
   a = m0 + Σ(1 - cos p_μ), S = Σ γ_μ sin p_μ, S^2 = |s|^2 I, so
   f(D(p)) = f(a+i|s|) (I + S/|s|)/2 + f(a-i|s|) (I - S/|s|)/2; links
   U_μ(x) = G(x) G(x+μ)^† give f(D_G) b = 𝒢 f(D_free) 𝒢^† b.
R4 Haar links: no closed form; the unpreconditioned (deg 0) Arnoldi run to an
   estimate ≤ 1e-14, as the paper does for its own QCD reference.
"""
from __future__ import annotations

import numpy as np
import scipy.fft as sfft

from inputs.operators import _gammas


def _fpow(func: str):
    return -0.5 if func == "invsqrt" else 0.5


def laplacian_fAb(N: int, dim: int, b: np.ndarray, func: str = "invsqrt") -> np.ndarray:
    """R1."""
    k = np.arange(1, N + 1)
    mu = 2.0 - 2.0 * np.cos(k * np.pi / (N + 1))
    lam = np.zeros((N,) * dim)
    for d in range(dim):
        shape = [1] * dim
        shape[d] = N
        lam = lam + mu.reshape(shape)
    B = b.reshape((N,) * dim)
    Bh = sfft.dstn(B, type=1, norm="ortho")
    Bh = Bh * lam ** _fpow(func)
    return sfft.idstn(Bh, type=1, norm="ortho").reshape(-1)


def convdiff_fAb(N: int, dim: int, beta, b: np.ndarray, func: str = "sqrt",
                 h: float | None = None) -> np.ndarray:
    """R2 in long double (π = arccos(-1) in long double)."""
    ld = np.longdouble
    if h is None:
        h = ld(1) / ld(N + 1)
    else:
        h = ld(h)
    pi = np.arccos(ld(-1))
    k = np.arange(1, N + 1, dtype=ld)
    j = np.arange(1, N + 1, dtype=ld)
    lam = np.zeros((N,) * dim, dtype=ld)
    Dfac = np.ones((N,) * dim, dtype=ld)
    # array axis a corresponds to grid axis (dim-1-a) because index = ix + N iy (+ N^2 iz)
    for a in range(dim):
        axis = dim - 1 - a
        P = ld(beta[axis]) * h / ld(2)
        rho = np.sqrt((ld(1) + P) / (ld(1) - P))
        sig = (ld(2) - ld(2) * np.sqrt(ld(1) - P * P) * np.cos(k * pi / ld(N + 1))) / (h * h)
        shape = [1] * dim
        shape[a] = N
        lam = lam + sig.reshape(shape)
        Dfac = Dfac * (rho ** j).reshape(shape)
    B = np.asarray(b, dtype=ld).reshape((N,) * dim)
    B = B / Dfac
    for a in range(dim):
        B = sfft.dst(B, type=1, norm="ortho", axis=a)
    B = B * lam ** ld(_fpow(func))
    for a in range(dim):
        B = sfft.idst(B, type=1, norm="ortho", axis=a)
    B = B * Dfac
    return np.asarray(B, dtype=np.float64).reshape(-1)


def wilson_free_fAb(L: int, m0: float, b: np.ndarray, func: str = "invsqrt",
                    G: np.ndarray | None = None) -> np.ndarray:
    """R3.  ``G`` (L^4, 3, 3) unitary gauge transformation for the pure-gauge
    links U_μ(x) = G(x) G(x+μ)^†; None means the free operator U ≡ 1."""
    pw = _fpow(func)
    psi = np.asarray(b, dtype=np.complex128).reshape(L ** 4, 4, 3)
    if G is not None:
        psi = np.einsum("sba,sib->sia", G.conj(), psi)  # 𝒢^† b: G(x)^† acting on colour
    arr = psi.reshape(L, L, L, L, 4, 3)  # axes [t, z, y, x, spin, colour]
    ph = np.fft.fftn(arr, axes=(0, 1, 2, 3))
    pvals = 2.0 * np.pi * np.arange(L) / L  # p = 2π n / L in FFT index order
    g = _gammas()
    # momentum grids: array axis 3 is x (μ=0), axis 2 is y (μ=1), axis 1 z (μ=2), axis 0 t (μ=3)
    P = np.meshgrid(pvals, pvals, pvals, pvals, indexing="ij")  # P[a] varies along array axis a
    p_mu = [P[3], P[2], P[1], P[0]]
    a = m0 + sum(1.0 - np.cos(p) for p in p_mu)
    svec = [np.sin(p) for p in p_mu]
    snorm = np.sqrt(sum(s * s for s in svec))
    S = sum(svec[mu][..., None, None] * g[mu] for mu in range(4))  # [...,4,4]
    I4 = np.eye(4)
    fp = (a + 1j * snorm).astype(np.complex128) ** pw
    fm = (a - 1j * snorm).astype(np.complex128) ** pw
    safe = np.where(snorm > 0, snorm, 1.0)
    Shat = S / safe[..., None, None]
    F = (fp[..., None, None] * (I4 + Shat) + fm[..., None, None] * (I4 - Shat)) / 2.0
    zero = snorm == 0
    if np.any(zero):
        F[zero] = (a[zero].astype(np.complex128) ** pw)[:, None, None] * I4
    out = np.einsum("...st,...tc->...sc", F, ph)
    x = np.fft.ifftn(out, axes=(0, 1, 2, 3)).reshape(L ** 4, 4, 3)
    if G is not None:
        x = np.einsum("sab,sib->sia", G, x)
    return x.reshape(-1)


def pure_gauge_links(G: np.ndarray, L: int) -> np.ndarray:
    """U_μ(x) = G(x) G(x+μ)^† on the periodic L^4 lattice; returns (4, L^4, 3, 3)."""
    V = L ** 4
    site = np.arange(V)
    links = np.empty((4, V, 3, 3), dtype=np.complex128)
    for mu in range(4):
        c = (site // L ** mu) % L
        fwd = site + (((c + 1) % L) - c) * L ** mu
        links[mu] = G @ np.swapaxes(G[fwd].conj(), 1, 2)
    return links


def arnoldi_reference(op, b, func: str = "invsqrt", tol: float = 1e-13, m_max: int = 400):
    """R4: plain (deg 0, q ≡ 1) CGS2 Arnoldi until the estimate ≤ tol.

    (1e-13 rather than SURVEY's 1e-14: on small lattices the estimate floors near
    1e-13 from rounding; agreement with a dense sqrtm solve is ~6e-14.)"""
    from . import chebyshev, krylov
    # deg-0 constant polynomial q = 1 is the unpreconditioned method (Table 1, d = 1)
    q = chebyshev.ChebPoly(0.5, 2.0, np.array([1.0]))
    return krylov.run(op, b, q, func=func, krylov="cgs2", m_max=m_max, stop="est",
                      tol=tol, check_every=2)
