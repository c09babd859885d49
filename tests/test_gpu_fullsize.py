"""Full BASELINE.json sizes, in the launch configuration bench.py times
(SELL-C-64 for fp64, SELL-C-32 for complex128, estimate stop at k = 1):
sampled outputs the oracle computes one by one (rows of A x), and properties
that hold at any size (true error against the closed forms R1/R2, the invariant
D (D^{-1/2} (D^{-1/2} b)) = b for the Wilson operator, P:115-124 branch
conditions on the Ritz nodes)."""
import numpy as np
import pytest

from inputs import configs
from oracle import reference

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_06684_b200 as pp  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return pp.Context(0)


def _sampled_spmv(ctx, A, M, rng, nsample=4096):
    x = rng.standard_normal(A.n)
    if np.iscomplexobj(A.val):
        x = x + 1j * rng.standard_normal(A.n)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    M.spmv(xd, yd)
    torch.cuda.synchronize()
    rows = np.sort(rng.choice(A.n, nsample, replace=False))
    rows = np.concatenate([rows, [0, A.n - 1]])
    y = yd.cpu().numpy()[rows]
    S = A.to_scipy()[rows]
    ref = S @ x
    scale = abs(S) @ np.abs(x)
    assert np.all(np.abs(y - ref) <= 1e-14 * scale)


def test_c4_fullsize(ctx):
    cfg = configs.CONFIGS["C4"]
    A, b, iv = configs.build("C4")
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=64))
    _sampled_spmv(ctx, A, M, np.random.default_rng(1))
    q = pp.Poly.chebyshev(*iv, 20)
    xg, rep = pp.run(ctx, M, q, torch.from_numpy(b).cuda(), func="sqrt", krylov="cgs2",
                     m_max=cfg.m_max, stop="est", tol=cfg.tol)
    torch.cuda.synchronize()
    xr = reference.convdiff_fAb(256, 3, (10.0, 10.0, 10.0), b, "sqrt")
    err = np.linalg.norm(xg.cpu().numpy() - xr) / np.linalg.norm(xr)
    assert rep.term == "converged" and rep.iterations <= 30
    # the estimate tracks the error; stopping at est <= 1e-8 leaves err ~ 1e-8
    assert err <= 3e-8, err
    assert rep.mvms == 20 + 1 + rep.iterations * 41


def test_c3_fullsize(ctx):
    cfg = configs.CONFIGS["C3"]
    A, b, iv = configs.build("C3")
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=64))
    _sampled_spmv(ctx, A, M, np.random.default_rng(2))
    xr = reference.laplacian_fAb(200, 3, b)
    for deg in cfg.degs:
        q = pp.Poly.chebyshev(*iv, deg)
        xg, rep = pp.run(ctx, M, q, torch.from_numpy(b).cuda(), func="invsqrt", krylov="lanczos",
                         m_max=cfg.m_max, stop="true", tol=cfg.tol, x_ref=torch.from_numpy(xr).cuda())
        torch.cuda.synchronize()
        err = np.linalg.norm(xg.cpu().numpy() - xr) / np.linalg.norm(xr)
        assert rep.term == "converged" and err <= 1e-8
        # m* at the paper's own kind of workload (52 / 27 / 14 with another seed)
        assert abs(rep.iterations - {10: 52, 20: 27, 40: 14}[deg]) <= 2


def test_c5_fullsize_invariant(ctx):
    cfg = configs.CONFIGS["C5"]
    A, b, _ = configs.build("C5")
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=32))
    _sampled_spmv(ctx, A, M, np.random.default_rng(3))
    bd = torch.from_numpy(b).cuda()
    q = pp.Poly.ritz_newton(ctx, M, bd, 16)
    nodes = q.export()["nodes"]
    assert np.all(nodes.real > 0)
    assert np.abs(q.eval(nodes) - nodes ** -0.5).max() < 1e-8
    x1, rep1 = pp.run(ctx, M, q, bd, func="invsqrt", krylov="cgs2", m_max=cfg.m_max, stop="est",
                      tol=1e-12)
    x2, rep2 = pp.run(ctx, M, q, x1.clone(), func="invsqrt", krylov="cgs2", m_max=cfg.m_max,
                      stop="est", tol=1e-12)
    torch.cuda.synchronize()
    res = A.to_scipy() @ x2.cpu().numpy() - b
    assert np.linalg.norm(res) / np.linalg.norm(b) <= 1e-9
    assert rep1.iterations <= 8


def test_c6_fullsize_sign_involution(ctx):
    """sign(Q)b for the 16^4 overlap kernel (bench C6): sign(Q)(sign(Q) b) = b
    (sign(Q)^2 = I) in the bench's launch configuration, Ritz values of Q^2 off
    the branch cut, and the (Q^2)^{-1/2} b iterate satisfies Q^2 f ~ ... via
    sign: Q f = sign(Q) b."""
    cfg = configs.CONFIGS["C6"]
    A, b, _ = configs.build("C6")
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=32))
    _sampled_spmv(ctx, A, M, np.random.default_rng(6))
    bd = torch.from_numpy(b).cuda()
    q = pp.Poly.ritz_newton(ctx, M, bd, 15, power=2)
    nodes = q.export()["nodes"]
    assert not np.any((np.abs(nodes.imag) < 1e-12 * np.abs(nodes)) & (nodes.real <= 0))
    s1, r1 = pp.run(ctx, M, q, bd, func="sign", krylov="cgs2", m_max=cfg.m_max, stop="est",
                    tol=1e-12)
    s2, r2 = pp.run(ctx, M, q, s1.clone(), func="sign", krylov="cgs2", m_max=cfg.m_max,
                    stop="est", tol=1e-12)
    assert r1.term == "converged" and r2.term == "converged"
    torch.cuda.synchronize()
    assert np.linalg.norm(s2.cpu().numpy() - b) <= 1e-9 * np.linalg.norm(b)


def test_c7_fullsize_sqrt_invariant(ctx):
    """L^{1/2} b for the synthetic 281,903-node graph Laplacian (bench C7, global
    SELL-32 sorting, forward-basis Newton chain): L^{1/2}(L^{1/2} b) = L b
    (Theorem 4.1's setting) with the Ritz q from L b."""
    cfg = configs.CONFIGS["C7"]
    A, b, _ = configs.build("C7")
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=32, sigma=32 * ((A.n + 31) // 32)))
    _sampled_spmv(ctx, A, M, np.random.default_rng(7))
    bd = torch.from_numpy(b).cuda()
    Lb = torch.empty_like(bd)
    M.spmv(bd, Lb)
    q = pp.Poly.ritz_newton(ctx, M, Lb, 15).set_newton_eval("basis")
    assert np.all(q.export()["nodes"].real > 0)
    x1, r1 = pp.run(ctx, M, q, bd, func="sqrt", krylov="cgs2", m_max=250, stop="est", tol=1e-10,
                    check_every=2)
    x2, r2 = pp.run(ctx, M, q, x1.clone(), func="sqrt", krylov="cgs2", m_max=250, stop="est",
                    tol=1e-10, check_every=2)
    assert r1.term == "converged" and r2.term == "converged"
    torch.cuda.synchronize()
    Lbh = Lb.cpu().numpy()
    # bar: 10x what the oracle itself reaches with this stopping rule (estimate
    # 1e-10 at k = 2): 9.0e-5 at full size (m = 186 / 148), because on this
    # strongly non-normal operator the paper's estimate is optimistic (at
    # n = 20000 the oracle's est 1e-10 is a true error of 4e-8) and the
    # composition doubles it; a wrong result would be O(1) off
    assert np.linalg.norm(x2.cpu().numpy() - Lbh) <= 9e-4 * np.linalg.norm(Lbh)
