"""Memory-safety checks of our own (compute-sanitizer is not available on the
GPU pool): guard bands and run-to-run determinism.

* Guard bands: b, x and the ppf_run workspace are carved out of ONE device
  buffer with 64 KB canary zones (0xA5 bytes) before, between and after them,
  the matrix likewise; after the run every canary byte must be intact (an
  out-of-bounds store by a kernel -- a ragged tail, a bulk copy, a SELL slice
  past n -- would land in one), and x must still match the oracle.
* Determinism: the TMA/mbarrier-ring sweeps, the flat sweeps, the sell2
  prefetch/PDL SpMV and the peer-memory reductions have no atomics in their
  arithmetic, so a shared-memory race or a stage released too early shows up
  as run-to-run differences: repeated runs must be bitwise identical.
Cases span the kernels: SELL-32 / SELL-64 / CSR, real and complex, Lanczos,
tiled and flat CGS2, ragged sizes."""
import numpy as np
import pytest

from inputs import configs
from inputs import operators as ops
from oracle import chebyshev, krylov, newton
from oracle.spmv import Operator

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_06684_b200 as pp  # noqa: E402
from paper_2401_06684_b200 import api  # noqa: E402

GUARD = 65536
CANARY = 0xA5


class _Work:
    def __init__(self, buf, nbytes):
        self.buf, self.nbytes = buf, nbytes


def _carve(sizes):
    """One uint8 device buffer: guard | seg_0 | guard | seg_1 | ... | guard
    (256-B aligned segments).  Returns (buffer, [(offset, size)])."""
    off, segs = GUARD, []
    for s in sizes:
        segs.append((off, s))
        off += (s + 255) // 256 * 256 + GUARD
    buf = torch.full((off,), CANARY, dtype=torch.uint8, device="cuda")
    return buf, segs


def _guards_intact(buf, segs):
    h = buf.cpu().numpy()
    mask = np.ones(len(h), dtype=bool)
    for o, s in segs:
        mask[o:o + s] = False
    bad = np.flatnonzero(mask & (h != CANARY))
    return bad


CASES = [
    ("C2", 5, 30, "sell", 32, "0"),     # wide CGS2 (2-D tensor-map ring), 31 columns
    ("C2", 5, 30, "sell", 32, "w0"),    # tiled CGS2 (TMA ring), 2 column tiles
    ("C2", 5, 30, "sell", 32, "1"),     # flat CGS2
    ("C4s", 20, 12, "sell", 64, "0"),   # sell2 (C = 64, prefetch, PDL), sqrt
    ("C3s", 10, 20, "csr", 32, None),   # CSR kernel, Lanczos
    ("odd", 3, 6, "sell", 64, "0"),     # n = 1001: ragged SELL slice and CGS chunk
    ("C5s", 16, 4, "sell", 32, None),   # complex, Ritz-Newton setup on the device
]


def _problem(name, deg):
    if name == "odd":
        A = ops.convdiff(1001, 1, (5.0,))
        b = np.random.default_rng(3).standard_normal(A.n)
        return configs.CONFIGS["C4s"], A, b, ops.convdiff_interval(1001, 1, (5.0,))
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    return cfg, A, b, iv


@pytest.mark.parametrize("name,deg,m,fmt,C_,flat", CASES)
def test_guard_bands(ctx_dev, monkeypatch, name, deg, m, fmt, C_, flat):
    if flat is not None:
        monkeypatch.setenv("PPF_CGS_FLAT", flat[-1])
        monkeypatch.setenv("PPF_CGS_WIDE", "0" if flat.startswith("w") else "1")
    cfg, A, b, iv = _problem(name, deg)
    ctx = pp.Context(0)
    plan = pp.Plan.from_csr(A, fmt=fmt, C_=C_)
    cplx = np.iscomplexobj(b)
    sc = 16 if cplx else 8
    mbytes = plan.device_bytes()
    ritz = cfg.poly == "ritz"
    func = cfg.func if name != "odd" else "sqrt"
    kry = cfg.krylov if name != "odd" else "cgs2"
    opts = api.make_opts(func=func, krylov=kry, m_max=m, stop="fixed")
    # workspace size needs a matrix handle: a throw-away matrix first
    M0 = pp.Matrix(ctx, plan)
    q0 = (pp.Poly.chebyshev(*iv, deg) if not ritz else
          pp.Poly.ritz_newton(ctx, M0, torch.from_numpy(b).cuda(), deg))
    wbytes = api.Workspace(ctx, M0, q0, opts).nbytes
    rbytes = pp.Poly.ritz_workspace(ctx, M0, deg).numel() if ritz else 0
    M0.close()
    buf, segs = _carve([mbytes, A.n * sc, A.n * sc, wbytes, max(rbytes, 256)])
    (mo, _), (bo, _), (xo, _), (wo, _), (ro, _) = segs
    dt = torch.complex128 if cplx else torch.float64
    bview = buf[bo:bo + A.n * sc].view(dt)
    xview = buf[xo:xo + A.n * sc].view(dt)
    bview.copy_(torch.from_numpy(b))
    # the matrix uploaded into its carved segment
    import ctypes as C
    h = C.c_void_p()
    api.check(api._lib().ppf_mat_create(ctx.h, plan.h, C.c_void_p(buf.data_ptr() + mo), mbytes,
                                        C.byref(h)))
    M = pp.Matrix.__new__(pp.Matrix)
    M.ctx, M.dtype, M.info, M.h, M.buf = ctx, plan.dtype, plan.info(), h, buf
    M.n_local = A.n
    if ritz:
        q = pp.Poly.ritz_newton(ctx, M, bview, deg, work=buf[ro:ro + rbytes])
    else:
        q = pp.Poly.chebyshev(*iv, deg)
    _, rep = pp.run(ctx, M, q, bview, xview, work=_Work(buf[wo:wo + wbytes], wbytes), func=func,
                    krylov=kry, m_max=m, stop="fixed")
    torch.cuda.synchronize()
    bad = _guards_intact(buf, segs)
    assert len(bad) == 0, f"{len(bad)} canary bytes overwritten, first at offset {bad[0]}"
    op = Operator(A.to_scipy())
    qo = newton.ritz_newton(op, b, deg)[0] if ritz else chebyshev.coefficients(*iv, deg)
    r = krylov.run(op, b, qo, func=func, krylov=kry, m_max=m)
    x = xview.cpu().numpy()
    assert np.linalg.norm(x - r.x) <= 1e-10 * np.linalg.norm(r.x)
    M.close()


@pytest.fixture(scope="module")
def ctx_dev():
    assert torch.cuda.is_available()
    return 0


@pytest.mark.parametrize("name,deg,m,C_,flat", [("C2", 5, 40, 32, "0"), ("C2", 5, 40, 32, "1"),
                                                ("C2", 5, 40, 32, "w0"),
                                                ("C4s", 20, 14, 64, "0"), ("C5s", 16, 4, 32, None)])
def test_bitwise_repeatable(ctx_dev, monkeypatch, name, deg, m, C_, flat):
    """Ten runs of the same problem: x and H bitwise identical (a shared-memory
    race in the bulk-copy ring or an early stage release would show here)."""
    if flat is not None:
        monkeypatch.setenv("PPF_CGS_FLAT", flat[-1])
        monkeypatch.setenv("PPF_CGS_WIDE", "0" if flat.startswith("w") else "1")
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    ctx = pp.Context(0)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=C_))
    bd = torch.from_numpy(b).cuda()
    q = pp.Poly.ritz_newton(ctx, M, bd, deg) if cfg.poly == "ritz" else pp.Poly.chebyshev(*iv, deg)
    ref = None
    for _ in range(10):
        x, rep = pp.run(ctx, M, q, bd, func=cfg.func, krylov=cfg.krylov, m_max=m, stop="fixed")
        torch.cuda.synchronize()
        got = (x.cpu().numpy().tobytes(), pp.hessenberg(ctx, np.iscomplexobj(b))[0].tobytes())
        if ref is None:
            ref = got
        assert got == ref
