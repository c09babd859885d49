"""Generator invariants (inputs/): structure, symmetry/similarity, γ5-Hermiticity,
closed-form spectral intervals against dense eigenvalues."""
import numpy as np
import pytest

from inputs import configs
from inputs import operators as ops


def test_laplacian_structure():
    A = ops.laplacian(5, 3)
    assert A.n == 125
    # nnz = 7n - 2*N^2*dim (boundary faces)
    assert A.nnz == 7 * 125 - 2 * 25 * 3
    S = A.to_scipy()
    assert abs(S - S.T).max() == 0
    assert np.all(np.diff(A.col[A.row_ptr[0]:A.row_ptr[1]]) > 0)
    for i in range(A.n):
        seg = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
        assert np.all(np.diff(seg) > 0)
    lam = np.linalg.eigvalsh(S.toarray())
    a, b = ops.laplacian_interval(5, 3)
    assert abs(lam[0] - a) < 1e-12 and abs(lam[-1] - b) < 1e-12


def test_paper_interval_formula_3d():
    # [6(1-cos(pi/(N+1))), 12 - 6(1-cos(pi/(N+1)))]
    N = 100
    a, b = ops.laplacian_interval(N, 3)
    c = np.cos(np.pi / (N + 1))
    assert a == pytest.approx(6 * (1 - c), rel=1e-15)
    assert b == pytest.approx(12 - 6 * (1 - c), rel=1e-15)


def test_convdiff_structure_and_interval():
    N, beta = 6, (5.0, 5.0)  # mesh Péclet P = βh/2 < 1
    A = ops.convdiff(N, 2, beta, h=1.0 / 7)
    S = A.to_scipy().toarray()
    h = 1.0 / 7
    i = 2 + N * 3
    assert S[i, i] == pytest.approx(4 / h**2)
    assert S[i, i - 1] == pytest.approx(-1 / h**2 - 5 / (2 * h))
    assert S[i, i + 1] == pytest.approx(-1 / h**2 + 5 / (2 * h))
    assert S[i, i - N] == pytest.approx(-1 / h**2 - 5 / (2 * h))
    ev = np.linalg.eigvals(S)
    assert np.abs(ev.imag).max() < 1e-8 * np.abs(ev).max()
    a, b = ops.convdiff_interval(N, 2, beta, h=1.0 / 7)
    assert ev.real.min() == pytest.approx(a, rel=1e-10)
    assert ev.real.max() == pytest.approx(b, rel=1e-10)


def test_config_sizes():
    # nnz of C1 and C2 (C3-C5 checked on the GPU tests)
    A, b, iv = configs.build("C1")
    assert (A.n, A.nnz) == (1024, 4992)
    A, b, iv = configs.build("C2")
    assert (A.n, A.nnz) == (65536, 326656)


def test_haar_su3():
    U = ops.haar_su3(np.random.default_rng(0), 500)
    I = np.eye(3)
    assert np.abs(U @ np.swapaxes(U.conj(), 1, 2) - I).max() < 1e-13
    assert np.abs(np.linalg.det(U) - 1).max() < 1e-13
    # Haar: E|tr U|^2 = 1
    tr = np.abs(np.trace(U, axis1=1, axis2=2)) ** 2
    assert 0.8 < tr.mean() < 1.2


def test_wilson_structure_gamma5():
    L = 3
    A = ops.wilson_dirac(L, -1.0, seed=7)
    assert A.n == 12 * L**4
    assert np.all(np.diff(A.row_ptr) == 49)
    S = A.to_scipy().toarray()
    g5 = np.kron(np.eye(L**4), np.kron(ops.gamma5(), np.eye(3)))
    assert np.abs(g5 @ S @ g5 - S.conj().T).max() < 1e-14
    g = ops._gammas()
    for i in range(4):
        assert np.abs(g[i] - g[i].conj().T).max() == 0
        for j in range(4):
            ac = g[i] @ g[j] + g[j] @ g[i]
            assert np.abs(ac - 2 * (i == j) * np.eye(4)).max() < 1e-15
    # ‖D - (4+m0) I‖ ≤ 4 (each μ term (P- U T+ + P+ U^† T-) is unitary up to 1/2 factors)
    H = S - 3.0 * np.eye(A.n)
    assert np.linalg.norm(H, 2) <= 4.0 + 1e-10
    # field of values in C+ for m0 = -1 at this seed: λ_min((D + D^*)/2) > 0
    assert np.linalg.eigvalsh((S + S.conj().T) / 2).min() > 0


def test_overlap_kernel_conventions():
    """Q = Γ5 D_w: Γ5 = diag(1,1,-1,-1) on the spins
    (P:467); Q is Hermitian at mu = 0 (γ5-hermiticity of D_w) and
    Q(mu)^H = Q(-mu) with the chemical potential on the time links."""
    g5 = ops.gamma5()
    assert np.allclose(g5, np.diag([1, 1, -1, -1]))
    Q0 = ops.overlap_kernel(3, -1.4, 0.0, seed=2).to_scipy()
    assert abs(Q0 - Q0.conj().T).max() < 1e-14
    Qp = ops.overlap_kernel(3, -1.4, 0.3, seed=2).to_scipy()
    Qm = ops.overlap_kernel(3, -1.4, -0.3, seed=2).to_scipy()
    assert abs(Qp - Qp.conj().T).max() > 0.1
    assert abs(Qp.conj().T - Qm).max() < 1e-14
