"""Pins for oracle/krylov.py (Algorithm 1) and oracle/reference.py: the paper's
Table 1 iteration counts, exactness at m = n, closed-form solutions (DST-I,
long-double similarity, free/pure-gauge Wilson), the paper's invariants, and the
Arnoldi relation."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from inputs import configs
from inputs import operators as ops
from oracle import chebyshev, dense, krylov, newton, reference
from oracle.spmv import Operator

from .conftest import GOLDEN


def _spd(n, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.linspace(0.2, 5.0, n)
    return (Q * lam) @ Q.T, lam


def test_exact_at_full_dimension_lanczos_and_cgs2():
    """m = n: the Krylov space is C^n, so f_n = A^{-1/2} b exactly (closed form
    via the eigendecomposition) -- this pins the left-preconditioning identity
    A^{-1/2}b = (A q(A)^2)^{-1/2} q(A) b end to end."""
    n = 24
    M, lam = _spd(n, 3)
    op = Operator(sp.csr_matrix(M))
    b = np.random.default_rng(5).standard_normal(n)
    ref = dense.invsqrt_dense(M).real @ b
    q = chebyshev.coefficients(lam[0], lam[-1], 3)
    for kry in ("lanczos", "cgs2"):
        res = krylov.run(op, b, q, func="invsqrt", krylov=kry, m_max=n)
        assert np.linalg.norm(res.x - ref) < 1e-9 * np.linalg.norm(ref), kry
    # sqrt: A^{1/2} b = A^{-1/2}(A b)
    res = krylov.run(op, b, q, func="sqrt", krylov="cgs2", m_max=n)
    ref = sla.sqrtm(M).real @ b
    assert np.linalg.norm(res.x - ref) < 1e-9 * np.linalg.norm(ref)


def test_spec_two_by_two_example():
    """A = diag(1,4), b = (1,1), deg-0 q: f_2 = (1, 1/2) exactly."""
    op = Operator(sp.csr_matrix(np.diag([1.0, 4.0])))
    q = chebyshev.ChebPoly(0.5, 5.0, np.array([0.7]))
    res = krylov.run(op, np.array([1.0, 1.0]), q, krylov="cgs2", m_max=2)
    assert np.allclose(res.x, [1.0, 0.5], atol=1e-14)


def test_arnoldi_relation_and_orthonormality():
    """(q(A))^2 A V_m = V_{m+1} H̄_m and V^H V = I (CGS2)."""
    N = 16
    A = ops.convdiff(N, 2, (20.0, 20.0))
    a, b_ = ops.convdiff_interval(N, 2, (20.0, 20.0))
    q = chebyshev.coefficients(a, b_, 5)
    op = Operator(A.to_scipy())
    b = np.random.default_rng(0).standard_normal(A.n)
    res = krylov.run(op, b, q, krylov="cgs2", m_max=12, keep_basis=True)
    V = res.V
    assert np.abs(V.T @ V - np.eye(13)).max() < 1e-12
    OpV = np.stack([chebyshev.apply(q, op, chebyshev.apply(q, op, op.matvec(V[:, j])))
                    for j in range(12)], axis=1)
    assert np.linalg.norm(OpV - V @ res.H) < 1e-10 * np.linalg.norm(res.H)
    # mvm count: deg for c, then (2 deg + 1) per step (PAPER.md:455 with d = deg+1)
    assert res.mvms == 5 + 12 * 11
    assert res.inner_products == sum(2 * j + 1 for j in range(1, 13))


def test_c1_converges_to_closed_form():
    """C1 (BASELINE configs[0]): true error against the DST-I closed form (R1)
    reaches 1e-10; m* recorded in DESIGN.md."""
    cfg = configs.CONFIGS["C1"]
    A, b, iv = configs.build("C1")
    op = Operator(A.to_scipy())
    xr = reference.laplacian_fAb(32, 2, b)
    q = chebyshev.coefficients(*iv, 4)
    res = krylov.find_m_star(op, b, q, func="invsqrt", krylov="lanczos", m_max=cfg.m_max,
                             tol=cfg.tol, x_ref=xr)
    assert res.term == "converged"
    assert res.m == 20
    assert res.mvms == 4 + 20 * 9
    # error decreases monotonically-ish and estimate tracks it
    errs = [h["err"] for h in res.history]
    assert errs[-1] <= 1e-10 and errs[0] > 1e-3


def test_c2_sqrt_closed_form_and_invariants():
    """C2 (configs[1]) at deg 20: x ≈ A^{1/2} b against the long-double
    similarity closed form (R2); invariant A^{-1/2}(A^{1/2} b) = b."""
    cfg = configs.CONFIGS["C2"]
    A, b, iv = configs.build("C2")
    op = Operator(A.to_scipy())
    p = cfg.params
    xr = reference.convdiff_fAb(p["N"], p["dim"], p["beta"], b, "sqrt")
    q = chebyshev.coefficients(*iv, 20)
    res = krylov.find_m_star(op, b, q, func="sqrt", krylov="cgs2", m_max=60, tol=1e-8, x_ref=xr)
    assert res.term == "converged" and res.history[-1]["err"] <= 1e-8
    back = krylov.run(op, res.x, q, func="invsqrt", krylov="cgs2", m_max=40, stop="est", tol=1e-11)
    # error amplification of A^{-1/2} on the 1e-8 error of x is ≲ sqrt(κ(A)) ≈ 49 (κ = 2403)
    assert np.linalg.norm(back.x - b) / np.linalg.norm(b) < 49 * 1e-8 * 2


def test_convdiff_closed_form_vs_dense():
    # moderate Péclet numbers keep cond(D) small enough for a dense sqrtm reference
    for N, dim, beta in ((10, 2, (5.0, 5.0)), (6, 3, (3.0, 3.0, 3.0))):
        A = ops.convdiff(N, dim, beta)
        M = A.to_scipy().toarray()
        b = np.random.default_rng(N).standard_normal(A.n)
        for func, ref in (("sqrt", sla.sqrtm(M) @ b),
                          ("invsqrt", np.linalg.solve(sla.sqrtm(M), b))):
            got = reference.convdiff_fAb(N, dim, beta, b, func)
            assert np.linalg.norm(got - ref.real) < 1e-11 * np.linalg.norm(ref)


def test_laplacian_closed_form_vs_dense():
    N = 7
    A = ops.laplacian(N, 3)
    M = A.to_scipy().toarray()
    b = np.random.default_rng(1).standard_normal(A.n)
    ref = dense.invsqrt_dense(M).real @ b
    assert np.linalg.norm(reference.laplacian_fAb(N, 3, b) - ref) < 1e-13 * np.linalg.norm(ref)


def test_wilson_free_and_pure_gauge_closed_form():
    """R3 against a dense inverse square root on a 3^4 lattice (m0 = 0.5: the
    free operator has the eigenvalue m0 at p = 0, so m0 must be > 0 here)."""
    L, m0 = 3, 0.5
    V = L**4
    b = np.random.default_rng(1).standard_normal(12 * V) + 0j
    eye = np.broadcast_to(np.eye(3, dtype=complex), (4, V, 3, 3)).copy()
    G = ops.haar_su3(np.random.default_rng(3), V)
    for links, Gt in ((eye, None), (reference.pure_gauge_links(G, L), G)):
        M = ops.wilson_dirac(L, m0, links=links).to_scipy().toarray()
        ref = np.linalg.solve(sla.sqrtm(M), b)
        got = reference.wilson_free_fAb(L, m0, b, G=Gt)
        assert np.linalg.norm(got - ref) < 1e-11 * np.linalg.norm(ref)


def test_c5_small_ritz_newton():
    """C5 family at 4^4 (Haar links, m0 = -1): Ritz-Newton q
    converges to the R4 reference; invariant D (D^{-1/2}(D^{-1/2} b)) = b."""
    cfg = configs.CONFIGS["C5s"]
    A, b, _ = configs.build("C5s")
    op = Operator(A.to_scipy())
    ref = reference.arnoldi_reference(op, b)
    assert ref.term == "converged"
    q, mv, ips = newton.ritz_newton(op, b, 16)
    assert mv == 17                                           # d extra mvms
    assert np.abs(newton.evaluate(q, q.nodes) - q.nodes**-0.5).max() < 1e-8
    assert np.all(q.nodes.real > 0)
    res = krylov.find_m_star(op, b, q, func="invsqrt", krylov="cgs2", m_max=cfg.m_max,
                             tol=cfg.tol, x_ref=ref.x)
    assert res.term == "converged" and res.m <= 5
    x1 = krylov.run(op, b, q, krylov="cgs2", m_max=12, stop="est", tol=1e-12).x
    x2 = krylov.run(op, x1, q, krylov="cgs2", m_max=12, stop="est", tol=1e-12).x
    assert np.linalg.norm(op.matvec(x2) - b) / np.linalg.norm(b) < 1e-9


def test_r4_reference_vs_dense():
    L = 3
    A = ops.wilson_dirac(L, -1.0, seed=11)
    b = np.random.default_rng(2).standard_normal(A.n) + 0j
    ref = reference.arnoldi_reference(Operator(A.to_scipy()), b)
    M = A.to_scipy().toarray()
    exact = np.linalg.solve(sla.sqrtm(M), b)
    assert np.linalg.norm(ref.x - exact) < 1e-12 * np.linalg.norm(exact)


@pytest.mark.slow
def _table1_setup():
    N = 100
    A = ops.laplacian(N, 3)
    a, bb = ops.laplacian_interval(N, 3)
    b = np.random.default_rng(0).standard_normal(N**3)
    b /= np.linalg.norm(b)
    return A, (a, bb), b, Operator(A.to_scipy()), reference.laplacian_fAb(N, 3, b)


def test_table1_iteration_counts_right_preconditioning():
    """PAPER.md:438-450, Table 1 rows d = 1, 4, 8, 16 at the paper's own scale
    (3D Laplacian 100^3, tol 1e-12, k = 64/d) with Algorithm 2 (right
    preconditioning) and the plain method for d = 1: iterations,
    mvms and inner products all three exactly (see golden file)."""
    g = json.load(open(os.path.join(GOLDEN, "table1_counts.json")))
    A, (a, bb), b, op, xr = _table1_setup()
    for row in g["rows"]:
        d = row["d"]
        q = None if d == 1 else chebyshev.coefficients(a, bb, d - 1)
        if q is not None:
            assert chebyshev.certify(q) > 0
        res = krylov.run(op, b, q, func="invsqrt", krylov="lanczos", m_max=600, stop="true",
                         tol=1e-12, check_every=64 // d, x_ref=xr, precond="right")
        assert res.m == row["iterations"], d
        assert res.mvms == row["mvms"], d
        assert res.inner_products == row["inner_products"], d


def test_table1_left_preconditioning_same_iterations():
    """Left preconditioning (Algorithm 1) at Table 1's d = 16: the same 28
    iterations, plus d-1 = 15 mvms for c = q(A)b."""
    A, (a, bb), b, op, xr = _table1_setup()
    q = chebyshev.coefficients(a, bb, 15)
    res = krylov.run(op, b, q, func="invsqrt", krylov="lanczos", m_max=200, stop="true",
                     tol=1e-12, check_every=4, x_ref=xr)
    assert res.m == 28
    assert res.mvms - 15 == 868
    assert res.inner_products == 56


@pytest.mark.parametrize("precond", ["left", "right", "plain"])
def test_two_pass_lanczos_closed_form(precond):
    """Two-pass Lanczos against the DST-I closed form
    (reference R1) on a 3D Laplacian: pass 1 stops on the estimate, pass 2
    regenerates the basis; the result must meet the tolerance against the
    closed form and need the same m as the one-pass method."""
    N = 14
    A = ops.laplacian(N, 3)
    a, bb = ops.laplacian_interval(N, 3)
    b = np.random.default_rng(41).standard_normal(N**3)
    xr = reference.laplacian_fAb(N, 3, b)
    op = Operator(A.to_scipy())
    q = None if precond == "plain" else chebyshev.coefficients(a, bb, 6)
    pre = "left" if precond == "plain" else precond
    one = krylov.run(op, b, q, func="invsqrt", krylov="lanczos", m_max=200, stop="est", tol=1e-10,
                     precond=pre)
    two = krylov.run_two_pass(op, b, q, func="invsqrt", precond=pre, m_max=200, stop="est",
                              tol=1e-10)
    assert two.m == one.m
    assert np.linalg.norm(two.x - xr) <= 1e-9 * np.linalg.norm(xr)
    assert np.allclose(two.H, one.H, rtol=0, atol=1e-12 * np.abs(one.H).max())
    # pass 2 repeats the operator applications of steps 1..m-1
    per_step = 1 if q is None else 2 * q.deg + 1
    start = 0 if (q is None or pre == "right") else q.deg
    final_q = q.deg if (q is not None and pre == "right") else 0
    assert two.mvms == start + one.m * per_step + (one.m - 1) * per_step + final_q


def test_right_preconditioning_nonhermitian_closed_form():
    """Algorithm 2 with CGS2 on the 2D convection-diffusion operator, sqrt via
    A^{-1/2}(Ab), against the long-double closed form R2."""
    N, beta = 24, (20.0, 20.0)
    A = ops.convdiff(N, 2, beta)
    a, bb = ops.convdiff_interval(N, 2, beta)
    b = np.random.default_rng(8).standard_normal(N**2)
    xr = reference.convdiff_fAb(N, 2, beta, b, "sqrt")
    op = Operator(A.to_scipy())
    q = chebyshev.coefficients(a, bb, 8)
    res = krylov.run(op, b, q, func="sqrt", krylov="cgs2", m_max=120, stop="true", tol=1e-9,
                     x_ref=xr, precond="right")
    assert res.term == "converged"
    left = krylov.run(op, b, q, func="sqrt", krylov="cgs2", m_max=120, stop="true", tol=1e-9,
                      x_ref=xr)
    assert abs(res.m - left.m) <= 2


@pytest.mark.parametrize("mu", [0.0, 0.3])
def test_sign_function_overlap_kernel_dense(mu):
    """sign(Q)b = Q (Q^2)^{-1/2} b for Q = Γ5 D_w(m_w = -1.4, mu)
    (Haar links on 3^4): the preconditioned Arnoldi result
    (Ritz-Newton q of Q^2) against the dense sign from the
    eigendecomposition, and the invariant sign(Q)^2 = I applied twice."""
    Qm = ops.overlap_kernel(3, -1.4, mu, seed=31)
    op = Operator(Qm.to_scipy())
    rng = np.random.default_rng(4)
    b = rng.standard_normal(Qm.n) + 1j * rng.standard_normal(Qm.n)
    S = dense.sign_dense(Qm.to_scipy().toarray())
    ref = S @ b
    from oracle.spmv import SquaredOperator
    q, _, _ = newton.ritz_newton(SquaredOperator(op), b, 7)
    res = krylov.run_sign(op, b, q, m_max=120, stop="est", tol=1e-12)
    assert res.term == "converged"
    assert np.linalg.norm(res.x - ref) <= 1e-9 * np.linalg.norm(ref)
    # (Q^2)^{-1/2} b itself
    inv = np.linalg.solve(Qm.to_scipy().toarray(), ref)          # Q^{-1} sign(Q) b
    assert np.linalg.norm(res.x_invsqrt_sq - inv) <= 1e-9 * np.linalg.norm(inv)
    twice = krylov.run_sign(op, res.x, q, m_max=120, stop="est", tol=1e-12).x
    assert np.linalg.norm(twice - b) <= 1e-8 * np.linalg.norm(b)
    # mvm unit of Table 2: 2 per application of Q^2
    per = 2 * (2 * q.deg + 1)
    assert res.mvms == 2 * q.deg + res.m * per + 1


def test_graph_laplacian_sqrt_implicit_desingularisation():
    """Ex. 6.3 setting: L = D_in - A is singular (zero column
    sums) with a simple eigenvalue 0; L^{1/2} b = L^{-1/2}(L b) with the
    Ritz-Newton q from L b works unchanged (Theorem 4.1): against
    the dense Schur square root (scipy.linalg.sqrtm) and the invariant
    L^{1/2}(L^{1/2} b) = L b."""
    A, b, _ = configs.build("C7s")
    S = A.to_scipy()
    assert abs(np.asarray(S.sum(axis=0))).max() == 0.0
    op = Operator(S)
    q, _, _ = newton.ritz_newton(op, op.matvec(b), 7)
    assert np.abs(q.nodes.imag).max() == 0.0 and q.nodes.real.min() > 0
    res = krylov.run(op, b, q, func="sqrt", krylov="cgs2", m_max=200, stop="est", tol=1e-11)
    assert res.term == "converged"
    ref = sla.sqrtm(S.toarray()) @ b
    assert np.linalg.norm(res.x - ref) <= 1e-8 * np.linalg.norm(ref)
    twice = krylov.run(op, res.x.real, q, func="sqrt", krylov="cgs2", m_max=200, stop="est",
                       tol=1e-11).x
    Lb = op.matvec(b)
    assert np.linalg.norm(twice - Lb) <= 1e-8 * np.linalg.norm(Lb)
