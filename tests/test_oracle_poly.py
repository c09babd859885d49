"""Pins for oracle/chebyshev.py and oracle/newton.py against the paper's printed
numbers (§3.2 worked example), closed forms and textbook special cases."""
import json
import os

import numpy as np
import pytest

from inputs import configs
from inputs import operators as ops
from oracle import chebyshev, krylov, newton, reference
from oracle.spmv import Operator

from .conftest import GOLDEN


def test_sec32_worked_example():
    """κ(A) ≈ 1054, ε = 0.1263, κ_pre ≤ 1.7345, κ_pre = 1.5153."""
    g = json.load(open(os.path.join(GOLDEN, "sec3_2_example.json")))
    N = g["grid_N"]
    a, b = ops.laplacian_interval(N, 2)
    assert abs(b / a - g["kappa_A"]) < 1.0                           # "≈ 1054" (1053.48)
    q = chebyshev.coefficients(a, b, g["d"] - 1)
    z = np.linspace(a, b, 400001)
    eps = np.max(np.abs(1.0 - np.sqrt(z) * chebyshev.evaluate(q, z)))
    assert abs(eps - g["epsilon"]) < g["tol_epsilon"]
    bound = (1 + 2 * eps + eps**2) / (1 - 2 * eps - eps**2)          # Prop 3.2
    assert abs(bound - g["kappa_pre_bound"]) < g["tol_kappa_pre_bound"]
    k = np.arange(1, N + 1)
    mu = 2 - 2 * np.cos(k * np.pi / (N + 1))
    lam = (mu[:, None] + mu[None, :]).ravel()                        # closed-form spec(A)
    pre = lam * chebyshev.evaluate(q, lam) ** 2                      # spec(A q(A)^2)
    assert abs(pre.max() / pre.min() - g["kappa_pre"]) < g["tol_kappa_pre"]
    # Prop 3.2's interval contains the preconditioned spectrum
    assert pre.min() >= 1 - 2 * eps - eps**2 - 1e-12 and pre.max() <= 1 + 2 * eps + eps**2 + 1e-12


def test_chebyshev_closed_form_evaluation():
    """q(z) = Σ c_i cos(i arccos t): the closed form of T_i on [-1, 1]."""
    q = chebyshev.coefficients(0.3, 17.0, 25)
    z = np.linspace(0.3, 17.0, 1001)
    t = np.clip((2 * z - 0.3 - 17.0) / (17.0 - 0.3), -1, 1)
    ref = sum(q.c[i] * np.cos(i * np.arccos(t)) for i in range(26))
    assert np.abs(chebyshev.evaluate(q, z) - ref).max() < 1e-13


def test_chebyshev_interpolates_at_nodes():
    """The d-point rule makes q interpolate z^{-1/2} at the first-kind nodes (F1)."""
    a, b, deg = 0.05, 9.0, 12
    q = chebyshev.coefficients(a, b, deg)
    d = deg + 1
    th = np.pi * (np.arange(d) + 0.5) / d
    zl = (a + b) / 2 + (b - a) / 2 * np.cos(th)
    assert np.abs(chebyshev.evaluate(q, zl) - zl**-0.5).max() < 1e-12 * np.max(zl**-0.5)
    # and matches numpy's independent interpolant construction
    from numpy.polynomial import chebyshev as npc
    c_np = npc.chebinterpolate(lambda t: ((a + b) / 2 + (b - a) / 2 * t) ** -0.5, deg)
    assert np.abs(c_np - q.c).max() < 1e-13


def test_chebyshev_degree0_and_certificate():
    q = chebyshev.coefficients(1.0, 1.0 + 1e-12, 0)
    assert q.c[0] == pytest.approx(1.0, rel=1e-11)
    a, b = ops.laplacian_interval(50, 2)
    assert chebyshev.certify(chebyshev.coefficients(a, b, 31)) > 0
    pts = chebyshev.certificate_points(2.0, 5.0)
    assert len(pts) == 1001 and pts[0] == 2.0 and pts[-1] == 5.0


def test_chebyshev_apply_vs_dst_closed_form():
    """O3 chain: q(A)b = S q(Λ) S b for the Dirichlet Laplacian (R1 eigenbasis)."""
    import scipy.fft as sfft
    N = 20
    A = ops.laplacian(N, 2)
    a, b = ops.laplacian_interval(N, 2)
    q = chebyshev.coefficients(a, b, 9)
    v = np.random.default_rng(4).standard_normal(N * N)
    op = Operator(A.to_scipy())
    got = chebyshev.apply(q, op, v)
    assert op.mvms == 9                                               # deg mvms
    k = np.arange(1, N + 1)
    mu = 2 - 2 * np.cos(k * np.pi / (N + 1))
    lam = mu[:, None] + mu[None, :]
    t = np.clip((2 * lam - a - b) / (b - a), -1, 1)
    qlam = sum(q.c[i] * np.cos(i * np.arccos(t)) for i in range(10))
    ref = sfft.idstn(sfft.dstn(v.reshape(N, N), type=1, norm="ortho") * qlam, type=1,
                     norm="ortho").ravel()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13


def test_newton_two_nodes_spec_example():
    """nodes {1,4} ⇒ q(z) = 7/6 - z/6; S:335-336 q(diag(1,4))(1,1) = (1, 1/2)."""
    q = newton.from_nodes([1.0, 4.0])
    z = np.array([0.0, 1.0, 4.0, 10.0])
    assert np.allclose(newton.evaluate(q, z), 7 / 6 - z / 6, atol=1e-15)
    import scipy.sparse as sp
    op = Operator(sp.csr_matrix(np.diag([1.0, 4.0]).astype(np.complex128)))
    out = newton.apply(q, op, np.array([1.0, 1.0]))
    assert np.allclose(out, [1.0, 0.5], atol=1e-15)


def test_newton_interpolation_property_lagrange():
    """q(θ_i) = θ_i^{-1/2} and agreement with the Lagrange form everywhere."""
    rng = np.random.default_rng(9)
    th = 3.0 + 2.0 * (rng.random(12) * np.exp(2j * np.pi * rng.random(12)))
    q = newton.from_nodes(th)
    assert np.abs(newton.evaluate(q, q.nodes) - q.nodes**-0.5).max() < 1e-10
    z = 3.0 + 1.5 * np.exp(1j * np.linspace(0, 2 * np.pi, 50))
    lag = np.zeros_like(z)
    for i, ti in enumerate(th):
        li = np.ones_like(z)
        for j, tj in enumerate(th):
            if j != i:
                li = li * (z - tj) / (ti - tj)
        lag = lag + ti**-0.5 * li
    assert np.abs(newton.evaluate(q, z) - lag).max() < 1e-9


def test_leja_order_properties():
    th = np.array([1.0, 2.0, 3.0, 4.0 + 0j, 2.5 + 1j])
    order = newton.leja_order(th)
    assert order[0] == 4.0
    # second point maximises distance to the first
    assert order[1] == 1.0
    assert sorted(map(complex, order), key=lambda c: (c.real, c.imag)) == \
        sorted(map(complex, th), key=lambda c: (c.real, c.imag))


def test_newton_apply_matches_dense_polynomial():
    """Newton apply vs dense evaluation Σ dd_j Π (A - θ_i) v."""
    rng = np.random.default_rng(1)
    n = 30
    M = rng.standard_normal((n, n)) / np.sqrt(n) + 3 * np.eye(n)
    import scipy.sparse as sp
    op = Operator(sp.csr_matrix(M.astype(np.complex128)))
    q = newton.from_nodes(np.linalg.eigvals(M[:8, :8]) + 0.0)
    v = rng.standard_normal(n) + 0j
    P = np.zeros((n, n), dtype=complex)
    prod = np.eye(n, dtype=complex)
    for j in range(q.deg + 1):
        P += q.dd[j] * prod
        prod = prod @ (M - q.nodes[j] * np.eye(n))
    assert np.linalg.norm(newton.apply(q, op, v) - P @ v) < 1e-11 * np.linalg.norm(P @ v)


def test_ritz_values_are_eigs_of_hessenberg_and_branch_check():
    rng = np.random.default_rng(2)
    n = 40
    M = np.diag(np.linspace(1, 10, n)) + 0.1 * rng.standard_normal((n, n))
    import scipy.sparse as sp
    op = Operator(sp.csr_matrix(M))
    H, ips = newton.arnoldi_plain(op, rng.standard_normal(n), n)
    th = np.sort_complex(newton.ritz_values(H[:n, :n]))
    ev = np.sort_complex(np.linalg.eigvals(M).astype(complex))
    assert np.abs(th - ev).max() < 1e-8                               # full space: Ritz = eig
    with pytest.raises(newton.BranchError):
        newton.ritz_values(np.diag([1.0, -2.0]))


# ---------------------------------------------------------------------------
# contour least-squares polynomial (§5.3)
# ---------------------------------------------------------------------------
def test_contour_ls_circle_equals_taylor_series():
    """On N equispaced points of a circle |z - c| = r the orthonormal basis is
    ((z - c)/r)^k / sqrt(N) and the least-squares fit of z^{-1/2} is the
    truncated Taylor series Σ binom(-1/2, k) c^{-1/2-k} (z - c)^k up to
    aliasing of order (r/c)^(N-d) (closed form)."""
    from scipy.special import binom
    from oracle import contour_ls
    c, r, N, deg = 3.0, 2.2, 128, 16
    q = contour_ls.construct(contour_ls.circle(c, r, N), deg)
    k = np.arange(deg + 1)
    t = binom(-0.5, k) * c ** (-0.5 - k)
    zz = c + 1.9 * np.exp(1j * np.linspace(0, 2 * np.pi, 37)) * np.linspace(0.1, 1, 37)
    taylor = np.polynomial.polynomial.polyval(zz - c, t)
    assert np.abs(contour_ls.evaluate(q, zz) - taylor).max() < 1e-12 * np.abs(taylor).max()
    assert contour_ls.certify(q) > 0


def test_contour_ls_normal_equations_and_lstsq():
    """General contour (an ellipse offset from 0): the residual z^{-1/2} - q is
    orthogonal to P_{d-1} in ⟨.,.⟩_ω (eq. polynomial_inner_product), and the fit
    values agree with numpy's least squares on a scaled monomial basis."""
    from oracle import contour_ls
    t = 2 * np.pi * np.arange(200) / 200
    z = 4.0 + 3.0 * np.cos(t) + 1.5j * np.sin(t)
    deg = 9
    q = contour_ls.construct(z, deg)
    f = z ** -0.5
    qz = contour_ls.evaluate(q, z)
    V = np.vander((z - 4.0) / 3.0, deg + 1, increasing=True)
    assert np.abs(V.conj().T @ (f - qz)).max() < 1e-12 * np.abs(f).sum()
    coef, *_ = np.linalg.lstsq(V, f, rcond=None)
    assert np.abs(V @ coef - qz).max() < 1e-12
    # q(A) v for A = diag(z) (the Arnoldi-like matrix process) equals
    # the fitted values
    import scipy.sparse as sp
    from oracle.spmv import Operator
    op = Operator(sp.diags(z).tocsr())
    assert np.abs(contour_ls.apply(q, op, np.ones(len(z))) - qz).max() < 1e-12
    assert op.mvms == deg


def test_contour_ls_wilson_converges():
    """The C5 family (Wilson-Dirac 4^4, m0 = -1.0) with the circle
    |z - (4 + m0)| = 2.2: left-preconditioned CGS2 reaches the
    R4 reference to 1e-8."""
    from oracle import contour_ls
    A, b, _ = configs.build("C5s")
    op = Operator(A.to_scipy())
    xr = reference.arnoldi_reference(op, b).x
    q = contour_ls.construct(contour_ls.circle(3.0, 2.2, 128), 16)
    res = krylov.run(op, b, q, func="invsqrt", krylov="cgs2", m_max=30, stop="true", tol=1e-8,
                     x_ref=xr)
    assert res.term == "converged" and res.m <= 6


def test_ritz_values_closed_form_partial_krylov():
    """Ritz node VALUES from a finite (d < n) Arnoldi run, pinned by closed
    forms:
    (i) the 1D Dirichlet Laplacian T_N = tridiag(-1, 2, -1) started from e_1:
        the Arnoldi/Lanczos basis is e_1..e_d, H_d = T_d, so the Ritz values are
        2 - 2 cos(k pi/(d+1)), k = 1..d, and ritz_newton's nodes are exactly
        those, Leja-ordered, with divided differences of z^{-1/2};
    (ii) b in a d-dimensional invariant subspace of a diagonal A: the d Ritz
        values are those d eigenvalues (the Krylov space is exhausted)."""
    import scipy.sparse as sp
    N, d = 200, 9
    T = sp.diags([-np.ones(N - 1), 2 * np.ones(N), -np.ones(N - 1)], [-1, 0, 1]).tocsr()
    e1 = np.zeros(N)
    e1[0] = 1.0
    H, _ = newton.arnoldi_plain(Operator(T), e1, d)
    theta = np.sort(newton.ritz_values(H[:d, :d]).real)
    exact = np.sort(2 - 2 * np.cos(np.arange(1, d + 1) * np.pi / (d + 1)))
    assert np.abs(theta - exact).max() < 1e-13
    q, mv, _ = newton.ritz_newton(Operator(T), e1, d - 1)
    assert mv == d
    assert np.abs(np.sort(q.nodes.real) - exact).max() < 1e-13
    assert np.abs(q.nodes.imag).max() < 1e-13
    assert abs(q.nodes[0].real - exact.max()) < 1e-13           # Leja: max modulus first
    # the interpolation property at the closed-form nodes (z^{-1/2} there)
    assert np.abs(newton.evaluate(q, exact) - exact ** -0.5).max() < 1e-10
    # (ii) invariant subspace
    lam = np.arange(1.0, 101.0)
    A = sp.diags(lam).tocsr()
    pick = np.array([3, 17, 42, 88]) - 1
    b = np.zeros(100)
    b[pick] = [1.0, -2.0, 0.5, 3.0]
    H2, _ = newton.arnoldi_plain(Operator(A), b, len(pick))
    th2 = np.sort(newton.ritz_values(H2[:len(pick), :len(pick)]).real)
    assert np.abs(th2 - lam[pick]).max() < 1e-10


def test_harmonic_ritz_values_closed_forms():
    """Harmonic Ritz values: (i) they are the reciprocals of
    the Ritz values of A^{-1} on A K_d(A, b), i.e. the eigenvalues of the
    d x d pencil (V^H A^H A V, V^H A^H V) -- checked against that definition
    with scipy's generalized eigensolver; (ii) for HPD A they are real and lie in
    [lambda_min, lambda_max] (bounded away from 0)."""
    import scipy.linalg as sla
    import scipy.sparse as sp
    from oracle import newton
    rng = np.random.default_rng(3)
    n = 40
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.linspace(0.3, 9.0, n)
    M = (Q * lam) @ Q.T + 0.3 * np.triu(rng.standard_normal((n, n)), 1)   # non-normal
    op = Operator(sp.csr_matrix(M))
    b = rng.standard_normal(n)
    d = 7
    H, _ = newton.arnoldi_plain(op, b, d)
    mu = newton.harmonic_ritz_values(H)
    # basis of K_d from the same Arnoldi process (oracle-independent rebuild)
    V = np.zeros((n, d))
    V[:, 0] = b / np.linalg.norm(b)
    for j in range(1, d):
        w = M @ V[:, j - 1]
        for _ in range(2):
            w -= V[:, :j] @ (V[:, :j].T @ w)
        V[:, j] = w / np.linalg.norm(w)
    AV = M @ V
    ref = sla.eigvals(AV.T @ AV, AV.T @ V)
    assert np.abs(np.sort_complex(mu) - np.sort_complex(ref)).max() < 1e-8 * np.abs(ref).max()
    # (ii) a symmetric positive definite A
    S = (Q * lam) @ Q.T
    ops = Operator(sp.csr_matrix(S))
    Hs, _ = newton.arnoldi_plain(ops, b, 9)
    mus = newton.harmonic_ritz_values(Hs)
    assert np.all(mus.real >= lam[0] - 1e-10) and np.all(mus.real <= lam[-1] + 1e-10)
    assert np.abs(mus.imag).max() < 1e-8


def test_ritz_polygon_contour():
    """Ritz-polygon contour: for Ritz values
    on a circle the polygon's points lie between the inscribed and the
    circumscribed circle of the hull; the minimum-distance rule keeps every
    point at |z| >= r_min; spacing is uniform to the step; a collinear (real)
    set gives the segment both ways; a set around 0 is rejected."""
    from oracle import contour_ls
    t = 2 * np.pi * np.arange(12) / 12
    th = 3.0 + 2.0 * np.exp(1j * t)
    z = contour_ls.ritz_polygon(th, 0.1, 0.01)
    r = np.abs(z - 3.0)
    assert r.max() <= 2.0 + 1e-12 and r.min() >= 2.0 * np.cos(np.pi / 12) - 1e-12
    d = np.abs(np.diff(z))
    assert d.max() <= 0.01 + 1e-12
    z2 = contour_ls.ritz_polygon(th, 1.5, 0.01)                 # cuts into the polygon
    assert np.abs(z2).min() >= 1.5 - 1e-12
    seg = contour_ls.ritz_polygon(np.array([0.5, 2.0, 7.0]), 0.1, 0.05)
    assert np.abs(seg.imag).max() == 0.0 and seg.real.min() == 0.5 and seg.real.max() <= 7.0
    with pytest.raises(ValueError):
        contour_ls.ritz_polygon(np.exp(1j * t), 0.1, 0.01)
    q = contour_ls.construct(z, 10)
    assert contour_ls.certify(q) > 0
