"""Pins for oracle/dense.py: y = β0 H^{-1/2} e_1 against scipy.linalg.sqrtm + solve
(a different library routine: Schur-based) and closed forms."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import dense
from oracle.newton import BranchError


def test_diagonal_examples():
    # SPEC S:70-72 style: diag(4, 9): H^{-1/2} e1 = (1/2, 0)
    y = dense.invsqrt_e1(np.diag([4.0, 9.0]), 1.0, hermitian=True)
    assert np.allclose(y, [0.5, 0.0], atol=1e-16)
    y = dense.invsqrt_e1(np.diag([4.0, 9.0]), 3.0, hermitian=False)
    assert np.allclose(y, [1.5, 0.0], atol=1e-15)


@pytest.mark.parametrize("n", [1, 5, 30, 64])
def test_hermitian_vs_sqrtm(n):
    rng = np.random.default_rng(n)
    T = np.diag(rng.uniform(0.5, 3.0, n)) + np.diag(rng.uniform(0.05, 0.2, n - 1), 1) \
        + np.diag(np.zeros(n - 1), -1)
    T = np.triu(T) + np.triu(T, 1).T
    y = dense.invsqrt_e1(T, 2.0, hermitian=True)
    e1 = np.zeros(n)
    e1[0] = 1
    ref = 2.0 * np.linalg.solve(sla.sqrtm(T), e1)
    assert np.linalg.norm(y - ref.real) < 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("n", [2, 8, 40, 64])
def test_nonhermitian_vs_sqrtm(n):
    rng = np.random.default_rng(100 + n)
    H = np.triu(rng.standard_normal((n, n)) * 0.2, -1) + 2.0 * np.eye(n)
    y = dense.invsqrt_e1(H, 1.3, hermitian=False)
    e1 = np.zeros(n)
    e1[0] = 1
    ref = 1.3 * np.linalg.solve(sla.sqrtm(H), e1)
    assert np.isrealobj(y)
    assert np.linalg.norm(y - ref) < 1e-11 * np.linalg.norm(ref)
    Hc = H + 0.3j * np.triu(rng.standard_normal((n, n)), -1)
    yc = dense.invsqrt_e1(Hc, 1.0, hermitian=False)
    refc = np.linalg.solve(sla.sqrtm(Hc), e1)
    assert np.linalg.norm(yc - refc) < 1e-11 * np.linalg.norm(refc)


def test_inverse_sqrt_squares_to_inverse():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((20, 20)) * 0.3 + 3 * np.eye(20)
    X = dense.invsqrt_dense(A)
    assert np.linalg.norm(X @ X @ A - np.eye(20)) < 1e-12


def test_branch_cut_rejected():
    with pytest.raises(BranchError):
        dense.invsqrt_e1(np.diag([1.0, -1.0]), 1.0, hermitian=True)
    with pytest.raises(BranchError):
        dense.invsqrt_e1(np.array([[1.0, 2.0], [0.0, -3.0]]), 1.0, hermitian=False)
