"""The resident step loop (kernels.cu: resident_steps_kernel; one CTA runs the
steps while the host decides the checkpoints from H columns in a mapped block)
against the oracle and against the launched path, for every small-operator
shape it takes: Lanczos and CGS2, real and complex, Chebyshev, Newton-Horner
and the forward Newton basis (the chain's second output), estimate stop with
k = 1 and k = 4 (steps run past a checkpoint), fixed m, sqrt and invsqrt."""
import numpy as np
import pytest

from inputs import configs
from inputs import operators as ops
from oracle import chebyshev, krylov, newton
from oracle.spmv import Operator

from .rounding import measured_bars

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_06684_b200 as pp  # noqa: E402



def _case(name):
    if name == "cd2":   # 2D convection-diffusion 40^2: CGS2, sqrt, Chebyshev
        A = ops.convdiff(40, 2, (20.0, 20.0))
        b = np.random.default_rng(5).standard_normal(A.n)
        return A, b, ops.convdiff_interval(40, 2, (20.0, 20.0)), "sqrt", "cgs2", "cheb", 1e-8
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    return A, b, iv, cfg.func, cfg.krylov, "cheb" if cfg.poly == "chebyshev" else "ritz", cfg.tol


@pytest.mark.parametrize("name,deg,stop,k", [("C1", 4, "est", 1), ("C1", 4, "fixed", 1),
                                             ("C1", 7, "est", 4), ("cd2", 6, "est", 1),
                                             ("cd2", 6, "fixed", 1), ("C5s", 16, "est", 1),
                                             ("C7s", 7, "est", 4)])
def test_resident_matches_oracle_and_launched(name, deg, stop, k, monkeypatch):
    A, b, iv, func, kry, poly, tol = _case(name)
    op = Operator(A.to_scipy())
    if poly == "cheb":
        qo = chebyshev.coefficients(*iv, deg)
    else:
        start = op.matvec(b) if name == "C7s" else b
        qo = newton.ritz_newton(op, start, deg)[0]
        if name == "C7s":
            qo.nodes, qo.dd = qo.nodes.real.astype(complex), qo.dd.real.astype(complex)
    m_max = 14 if stop == "fixed" else 200
    res_o = krylov.run(op, b, qo, func=func, krylov=kry, m_max=m_max, stop=stop, tol=tol,
                       check_every=k)
    if not np.iscomplexobj(b):
        res_o.x = res_o.x.real
        res_o.H = res_o.H.real
    ctx = pp.Context(0)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=32))
    if poly == "cheb":
        q = pp.Poly.chebyshev(*iv, deg)
    else:
        q = pp.Poly.newton(qo.nodes, qo.dd)
        if name == "C7s":
            q.set_newton_eval("basis")
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("PPF_RESIDENT", flag)
        x, rep = pp.run(ctx, M, q, torch.from_numpy(b).cuda(), func=func, krylov=kry, m_max=m_max,
                        stop=stop, tol=tol, check_every=k)
        torch.cuda.synchronize()
        out[flag] = (x.cpu().numpy(), rep, pp.hessenberg(ctx, np.iscomplexobj(b))[0],
                     pp.history(ctx))
    # bars: 1e-11 / 1e-10, or 10x the oracle's own gap under a rounding-only
    # perturbation (every mat-vec rounded once, tests/rounding.py; reading Q19)
    def rerun(op2):
        r = krylov.run(op2, b, qo, func=func, krylov=kry, m_max=res_o.m)
        if not np.iscomplexobj(b):
            r.x, r.H = r.x.real, r.H.real
        return r
    h_bar, x_bar, hg, xg = measured_bars(res_o, rerun, A.to_scipy())
    for flag, (x, rep, H, hist) in out.items():
        assert rep.iterations == res_o.m, (flag, rep.iterations, res_o.m)
        assert rep.mvms == res_o.mvms
        e_x = np.linalg.norm(x - res_o.x) / np.linalg.norm(res_o.x)
        e_h = np.abs(H - res_o.H).max() / np.abs(res_o.H).max()
        print(f"resident={flag}: H gap {e_h:.2e} (bar {h_bar:.1e}), x gap {e_x:.2e} (bar {x_bar:.1e})")
        assert e_x <= x_bar
        assert e_h <= h_bar
        if stop == "est":
            assert [h["m"] for h in hist] == [h["m"] for h in res_o.history]
    # the resident run launched one step kernel instead of ~5 per step
    assert out["1"][1].kernel_launches < out["0"][1].kernel_launches
