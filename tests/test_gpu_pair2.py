"""Paired chain SpMVs (kernels.cu sellp_pair_kernel): two consecutive Clenshaw
steps b_i, b_{i-1} (§5.1) in one persistent launch that sweeps
both as a wavefront.  Each row's multiply-adds are the single-step kernel's,
so q(A)x and whole runs must be bitwise equal to the unpaired path
(PPF_PAIR2=0), for chain lengths odd and even, ragged sizes whose last block
and last slice are partial, bandwidths of 1..several blocks, and handout
slacks from 0 (step-2 items wait on freshly handed-out step-1 items) to
beyond the block count (all step-1 items first).  The run-level case also
checks the oracle bar (x to 1e-10, same m*) on the paired path."""
import numpy as np
import pytest

from inputs import configs
from inputs import operators as ops
from oracle import chebyshev, krylov, reference
from oracle.spmv import Operator

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_06684_b200 as pp  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return pp.Context(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


SHAPES = [
    (13, 3, None),                 # n = 2197: 3 blocks, last one partial, halo 1
    (200, 2, None),                # n = 40000: halo 1 block
    (47, 3, (10.0, 5.0, 2.5)),     # n = 103823, ragged, convection: halo 3 blocks
    (64, 3, None),                 # n = 262144: 256 full blocks, halo 4
]


@pytest.mark.parametrize("slack", [None, "0", "1", "100000"])
@pytest.mark.parametrize("deg", [2, 3, 7, 20])
@pytest.mark.parametrize("shape", SHAPES)
def test_pair_chain_bitwise(ctx, shape, deg, slack, monkeypatch):
    N, dim, beta = shape
    A = ops.laplacian(N, dim) if beta is None else ops.convdiff(N, 3, beta)
    plan = pp.Plan.from_csr(A, fmt="sell", C_=64)
    assert plan.encoding()[0] == "pair8"
    M = pp.Matrix(ctx, plan)
    x = np.random.default_rng(N + deg).standard_normal(A.n)
    q = pp.Poly.chebyshev(0.5, 20.0, deg)
    if slack is not None:
        monkeypatch.setenv("PPF_PAIR2_SLACK", slack)
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PPF_PAIR2", flag)
        # repeated applications: the sync words must reset between launches
        res[flag] = [host(q.apply(ctx, M, dev(x))) for _ in range(3)]
    for r in res["0"] + res["1"]:
        assert np.array_equal(r, res["0"][0])
    # and against a plain numpy Clenshaw (the chain's own definition)
    S = A.to_scipy()
    a, b = 0.5, 20.0
    c = chebyshev.coefficients(a, b, deg)
    al, be = 2.0 / (b - a), -(a + b) / (b - a)
    b1 = np.zeros_like(x)
    b2 = np.zeros_like(x)
    for k in range(deg, 0, -1):
        b0 = 2 * (al * (S @ b1) + be * b1) - b2 + c[k] * x
        b2, b1 = b1, b0
    ref = al * (S @ b1) + be * b1 - b2 + c[0] * x
    assert np.linalg.norm(res["1"][0] - ref) <= 1e-12 * np.linalg.norm(ref)


def _reference(cfg, b):
    p = cfg.params
    if cfg.family == "laplacian":
        return reference.laplacian_fAb(p["N"], p["dim"], b, cfg.func)
    return reference.convdiff_fAb(p["N"], p["dim"], p["beta"], b, cfg.func)


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("name,deg", [("C3s", 10), ("C3s", 20), ("C4s", 5), ("C4s", 20)])
def test_pair_run_bitwise_and_oracle(ctx, name, deg, graphs, monkeypatch):
    """Scaled C3/C4 runs to the true error (Lanczos / CGS2, invsqrt / sqrt):
    paired and unpaired runs give the same m, mvms, H and x bitwise (also
    under the step graph, which captures the paired launches and replays
    them), and the paired run meets the oracle bar (same m*, x to 1e-10)."""
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    xr = _reference(cfg, b)
    res_o = krylov.find_m_star(Operator(A.to_scipy()), b, chebyshev.coefficients(*iv, deg),
                               func=cfg.func, krylov=cfg.krylov, m_max=cfg.m_max, tol=cfg.tol,
                               x_ref=xr)
    assert res_o.term == "converged"
    plan = pp.Plan.from_csr(A, fmt="sell", C_=64)
    assert plan.encoding()[0] == "pair8"
    M = pp.Matrix(ctx, plan)
    q = pp.Poly.chebyshev(*iv, deg)
    out = {}
    ctx.set_graphs(graphs)
    try:
        for flag in ("0", "1"):
            monkeypatch.setenv("PPF_PAIR2", flag)
            xg, rep = pp.run(ctx, M, q, dev(b), func=cfg.func, krylov=cfg.krylov, m_max=cfg.m_max,
                             stop="true", tol=cfg.tol, x_ref=dev(xr))
            out[flag] = (host(xg), pp.hessenberg(ctx, False)[0], rep.iterations, rep.mvms)
    finally:
        ctx.set_graphs(True)
    assert out["0"][2] == out["1"][2] == res_o.m
    assert out["0"][3] == out["1"][3] == res_o.mvms
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])
    rel = np.linalg.norm(out["1"][0] - res_o.x) / np.linalg.norm(res_o.x)
    print(f"{name} deg {deg} paired: m = {out['1'][2]}, |dx|/|x| = {rel:.2e} (bar 1e-10)")
    assert rel <= 1e-10
