"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same
seeded inputs.  Bars (BASELINE.json north_star, reading Q19):
  x:  ||x_gpu - x_oracle|| / ||x_oracle|| <= 1e-10 after the same m steps,
  H:  max|H_gpu - H_oracle| / max|H_oracle| <= 1e-11,
  m*: the same iteration count to reach the stated tolerance.
Kernel-level parity (SpMV, fused chain) uses 1e-13 relative (fp64 rounding of
a few hundred terms).  Sizes span several slices/tiles and a ragged tail."""
import numpy as np
import pytest

from inputs import configs
from inputs import operators as ops
from inputs.operators import CSR
from oracle import chebyshev, krylov, newton, reference
from oracle.spmv import Operator

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_06684_b200 as pp  # noqa: E402
from paper_2401_06684_b200 import api  # noqa: E402

X_TOL, H_TOL = 1e-10, 1e-11


@pytest.fixture(scope="module")
def ctx():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return pp.Context(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def ragged_matrix(n, seed, complex_=False):
    """Random sparse matrix with row lengths 0..40 (empty rows included)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 41, n)
    lens[rng.random(n) < 0.05] = 0
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens]).astype(np.int64)
    vals = rng.standard_normal(len(cols))
    if complex_:
        vals = vals + 1j * rng.standard_normal(len(cols))
    return CSR(n, rp, cols, vals)


FORMATS = [("sell", 32, 1), ("sell", 64, 1), ("sell", 32, 128), ("csr", 32, 1)]


@pytest.mark.parametrize("idx", ["8", "16", "32"])
@pytest.mark.parametrize("fmt,C_,sig", FORMATS)
@pytest.mark.parametrize("which", ["lap3", "convdiff3", "ragged", "ragged_c", "wilson", "wide_cols"])
def test_spmv_parity(ctx, fmt, C_, sig, which, idx, monkeypatch):
    """Every format against SciPy; SELL-64 fp64 with the pair codes (idx 8:
    PPF_PAIR8, the default for the stencils; the ragged/random matrices fall
    back), SELL-32/64 with the 16-bit column deltas (PPF_IDX16, the default
    where every (slice, column) spans <= 65535 columns) and with 32-bit
    indices; "wide_cols" has columns spread over 200,000 so the plan must
    fall back to 32-bit indices."""
    monkeypatch.setenv("PPF_IDX16", "0" if idx == "32" else "1")
    monkeypatch.setenv("PPF_PAIR8", "1" if idx == "8" else "0")
    if idx != "32" and not (fmt == "sell" and sig == 1):
        pytest.skip("16-bit deltas / pair codes exist for SELL without sorting")
    if idx == "8" and C_ != 64:
        pytest.skip("pair codes: SELL-64 fp64")
    if which == "lap3":
        A = ops.laplacian(13, 3)            # 2197 rows: ragged tail for C = 32 and 64
    elif which == "convdiff3":
        A = ops.convdiff(11, 3, (10.0, 10.0, 10.0))
    elif which == "ragged":
        A = ragged_matrix(3001, 1)
    elif which == "ragged_c":
        A = ragged_matrix(1999, 2, complex_=True)
    elif which == "wide_cols":
        A = ragged_matrix(200_000, 5)
    else:
        A = ops.wilson_dirac(3, -1.0, seed=4)
    if np.iscomplexobj(A.val) and C_ == 64:
        pytest.skip("C = 64 is the fp64 two-rows-per-lane layout")
    plan = pp.Plan.from_csr(A, fmt=fmt, C_=C_, sigma=sig)
    if idx == "8" and which in ("lap3", "convdiff3"):
        assert plan.encoding() == ("pair8", 8)
    M = pp.Matrix(ctx, plan)
    rng = np.random.default_rng(7)
    x = rng.standard_normal(A.n)
    if np.iscomplexobj(A.val):
        x = x + 1j * rng.standard_normal(A.n)
    xd = dev(x)
    yd = torch.full_like(xd, float("nan"))
    M.spmv(xd, yd)
    ref = A.to_scipy() @ x
    got = host(yd)
    absA = abs(A.to_scipy()) @ np.abs(x)
    assert np.all(np.abs(got - ref) <= 1e-14 * absA + 1e-300)


@pytest.mark.parametrize("ks", [1, 2, 4])
@pytest.mark.parametrize("shape", [(13, 3, None), (64, 2, None), (19, 3, (10.0, 10.0, 10.0)),
                                   (47, 3, (10.0, 5.0, 2.5)), (1, 3, None), (2, 2, None)])
def test_pair_codes_bitwise(ctx, shape, ks):
    """The pair-code layout does the explicit layout's multiply-adds in the
    same order on the same values and columns: the SpMV and the fused
    Clenshaw chain (z, u, x epilogue terms) must be bitwise identical across
    pair8 / delta16 / explicit, for sizes spanning many 64-row slices with a
    ragged last slice, a 1-row and a 4-row matrix, warps split per slice, and
    an anisotropic convection (distinct values per direction)."""
    N, dim, beta = shape
    A = ops.laplacian(N, dim) if beta is None else ops.convdiff(N, 3, beta)
    rng = np.random.default_rng(N * 10 + dim)
    x = rng.standard_normal(A.n)
    outs = {}
    for enc in ("pair8", "delta16", "explicit"):
        plan = pp.Plan.from_csr(A, fmt="sell", C_=64)
        if enc != "pair8":
            try:
                plan.set_encoding(enc)
            except RuntimeError:
                assert enc == "delta16"
                continue
        else:
            assert plan.encoding()[0] == "pair8"
        M = pp.Matrix(ctx, plan)
        M.set_split(ks)
        yd = torch.full_like(dev(x), float("nan"))
        M.spmv(dev(x), yd)
        a, b = 0.5, 20.0
        q = pp.Poly.chebyshev(a, b, 7)
        outs[enc] = (host(yd), host(q.apply(ctx, M, dev(x))))
    ref = A.to_scipy() @ x
    absA = abs(A.to_scipy()) @ np.abs(x)
    for enc, (y, c) in outs.items():
        assert np.array_equal(y, outs["explicit"][0]), enc
        assert np.array_equal(c, outs["explicit"][1]), enc
    assert np.all(np.abs(outs["pair8"][0] - ref) <= 1e-14 * absA + 1e-300)


@pytest.mark.parametrize("tile", ["4x2", "8x1", "2x4"])
@pytest.mark.parametrize("shape", [(64, 3, (10.0, 10.0, 10.0)), (47, 3, (10.0, 5.0, 2.5)), (90, 2, None),
                                   (21, 3, None)])
def test_pair_codes_slice_schedule_bitwise(ctx, shape, tile, monkeypatch):
    """The slice schedule (ppf_plan_slice_schedule: blocks take tiles of slices
    that gather from one another) only reorders which warp computes which
    slice: SpMV and the fused Clenshaw chain are bitwise those of the in-order
    launch and of the explicit layout, for aligned and ragged grids, 2-D and
    3-D, and every tile shape."""
    N, dim, beta = shape
    A = ops.laplacian(N, dim) if beta is None else ops.convdiff(N, 3, beta)
    rng = np.random.default_rng(N + dim)
    x = rng.standard_normal(A.n)
    outs = {}
    for name, env in (("tiled", tile), ("inorder", "0")):
        monkeypatch.setenv("PPF_SELLP_TILE", env)
        plan = pp.Plan.from_csr(A, fmt="sell", C_=64)
        assert plan.encoding()[0] == "pair8"
        assert (len(plan.slice_schedule()) > 0) == (name == "tiled")
        M = pp.Matrix(ctx, plan)
        yd = torch.full_like(dev(x), float("nan"))
        M.spmv(dev(x), yd)
        q = pp.Poly.chebyshev(0.5, 20.0, 7)
        outs[name] = (host(yd), host(q.apply(ctx, M, dev(x))))
    assert np.array_equal(outs["tiled"][0], outs["inorder"][0])
    assert np.array_equal(outs["tiled"][1], outs["inorder"][1])
    ref = A.to_scipy() @ x
    absA = abs(A.to_scipy()) @ np.abs(x)
    assert np.all(np.abs(outs["tiled"][0] - ref) <= 1e-14 * absA + 1e-300)


@pytest.mark.parametrize("scaled", ["1", "0"])
@pytest.mark.parametrize("ctab", ["1", "0"])
@pytest.mark.parametrize("nvals", [2, 3, 10, 40])
def test_pair_codes_table_sizes(ctx, nvals, ctab, scaled, monkeypatch):
    """Pair tables beyond the 32 entries passed as a kernel parameter are
    held in shared memory (and PPF_SELLP_CTAB=0 forces that path for small
    ones): a banded matrix (offsets -3..3, ragged n = 5003) whose values are
    drawn from `nvals` levels -- 7 * nvals pairs + padding: 15 (codes
    uploaded as record byte offsets unless PPF_SELLP_SCALED=0), 22 (parameter
    table), 71 (shared-memory table), 281 (over the 256-entry table: the
    deltas) -- against the explicit layout (bitwise) and SciPy."""
    monkeypatch.setenv("PPF_SELLP_CTAB", ctab)
    monkeypatch.setenv("PPF_SELLP_SCALED", scaled)
    n = 5003
    rng = np.random.default_rng(nvals)
    levels = rng.standard_normal(nvals)
    offs = np.arange(-3, 4)
    rows, cols = [], []
    for o in offs:
        r = np.arange(max(0, -o), min(n, n - o))
        rows.append(r)
        cols.append(r + o)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    vals = levels[rng.integers(0, nvals, len(rows))]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    A = CSR(n, rp, cols.astype(np.int64), vals)
    plan = pp.Plan.from_csr(A, fmt="sell", C_=64)
    enc, ntab = plan.encoding()
    assert (enc == "pair8") == (7 * nvals + 1 <= 256), (enc, ntab)
    if enc == "pair8":
        assert ntab == 7 * nvals + 1
    x = rng.standard_normal(n)
    M = pp.Matrix(ctx, plan)
    yd = torch.full_like(dev(x), float("nan"))
    M.spmv(dev(x), yd)
    Me = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=64).set_encoding("explicit"))
    ye = torch.full_like(dev(x), float("nan"))
    Me.spmv(dev(x), ye)
    assert np.array_equal(host(yd), host(ye))
    ref = A.to_scipy() @ x
    assert np.all(np.abs(host(yd) - ref) <= 1e-14 * (abs(A.to_scipy()) @ np.abs(x)))


@pytest.mark.parametrize("ks", [1, 2, 4, 8])
@pytest.mark.parametrize("C_", [32, 64])
@pytest.mark.parametrize("which", ["ragged", "ragged_c", "wilson", "lap3"])
def test_spmv_split_parity(ctx, ks, C_, which):
    """KS warps per SELL slice (ppf_mat_set_split): the parts' partial sums are
    combined in part order; every row must still match the oracle SpMV, for
    slices whose width is not a multiple of KS and slices narrower than KS."""
    if which == "ragged":
        A = ragged_matrix(3001, 11)
    elif which == "ragged_c":
        A = ragged_matrix(1999, 12, complex_=True)
    elif which == "wilson":
        A = ops.wilson_dirac(4, -1.0, seed=5)   # 3072 rows, 49 entries each
    else:
        A = ops.laplacian(13, 3)
    if np.iscomplexobj(A.val) and C_ == 64:
        pytest.skip("C = 64 is the fp64 two-rows-per-lane layout")
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=C_, sigma=1))
    assert M.set_split(ks) == ks
    rng = np.random.default_rng(17)
    x = rng.standard_normal(A.n)
    if np.iscomplexobj(A.val):
        x = x + 1j * rng.standard_normal(A.n)
    xd = dev(x)
    yd = torch.full_like(xd, float("nan"))
    M.spmv(xd, yd)
    ref = A.to_scipy() @ x
    absA = abs(A.to_scipy()) @ np.abs(x)
    assert np.all(np.abs(host(yd) - ref) <= 1e-14 * absA + 1e-300)
    assert M.set_split(0) >= 1


def powerlaw_matrix(n, seed, complex_=False):
    """Heavy-tailed row lengths (Zipf-like, a few rows of 300-1500 entries,
    empty rows included) -- after a whole-matrix sigma sort the leading
    slices are wide enough to take the SELL kernel's one-block-per-slice path
    (sell_heavy_prefix)."""
    rng = np.random.default_rng(seed)
    lens = np.minimum((rng.pareto(1.2, n) * 3).astype(np.int64), n // 2)
    lens[rng.choice(n, 40, replace=False)] = rng.integers(300, 1500, 40)
    lens[rng.random(n) < 0.03] = 0
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens]).astype(np.int64)
    vals = rng.standard_normal(len(cols))
    if complex_:
        vals = vals + 1j * rng.standard_normal(len(cols))
    return CSR(n, rp, cols, vals)


@pytest.mark.parametrize("ks", [1, 2, 4])
@pytest.mark.parametrize("complex_", [False, True])
def test_spmv_heavy_slices_parity(ctx, ks, complex_):
    """Power-law rows, whole-matrix sigma sort: the leading (heavy) slices get
    a block of 8 warps each, the rest KS warps; every row matches the oracle
    SpMV, and so does the forward-Newton-basis chain (second output) on it."""
    n = 4099
    A = powerlaw_matrix(n, 21 + ks, complex_)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=32, sigma=32 * ((n + 31) // 32)))
    assert M.set_split(ks) == ks
    rng = np.random.default_rng(ks)
    x = rng.standard_normal(n) + (1j * rng.standard_normal(n) if complex_ else 0)
    yd = torch.full_like(dev(x), float("nan"))
    M.spmv(dev(x), yd)
    ref = A.to_scipy() @ x
    absA = abs(A.to_scipy()) @ np.abs(x)
    assert np.all(np.abs(host(yd) - ref) <= 1e-14 * absA + 1e-300)
    # forward Newton basis (the chain's second output) on the same slices
    th = 40.0 + 10.0 * rng.random(6)
    qo = newton.from_nodes(th.astype(complex))
    q = pp.Poly.newton(qo.nodes, qo.dd).set_newton_eval("basis")
    got = host(q.apply(ctx, M, dev(x)))
    ref = newton.apply(qo, Operator(A.to_scipy()), x.astype(complex))
    if not complex_:
        ref = ref.real
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_auto_split_choice(ctx):
    """The automatic split: KS = 1 for narrow rows and for matrices with many
    slices; a few-slice matrix with wide rows is split."""
    A = ops.wilson_dirac(4, -1.0, seed=5)     # 96 slices of 49 entries
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=32, sigma=1))
    assert M.set_split(0) == 4
    L = ops.laplacian(13, 3)
    M2 = pp.Matrix(ctx, pp.Plan.from_csr(L, fmt="sell", C_=64, sigma=1))
    assert M2.set_split(0) == 1


@pytest.mark.parametrize("fmt", ["sell", "csr"])
@pytest.mark.parametrize("deg", [0, 1, 2, 3, 7, 20])
def test_chebyshev_chain_parity(ctx, fmt, deg):
    """Fused Clenshaw chain vs the oracle's forward recurrence, and
    against the DST-I closed form q(A)v = S q(Λ) S v."""
    N = 17
    A = ops.laplacian(N, 3)
    a, b = ops.laplacian_interval(N, 3)
    qo = chebyshev.coefficients(a, b, deg)
    q = pp.Poly.chebyshev(a, b, deg)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt=fmt))
    v = np.random.default_rng(deg).standard_normal(A.n)
    got = host(q.apply(ctx, M, dev(v)))
    ref = chebyshev.apply(qo, Operator(A.to_scipy()), v)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("deg", [1, 2, 5, 16])
def test_newton_chain_parity(ctx, deg):
    """Fused Newton-Horner chain vs the oracle's forward Newton basis,
    with the oracle's q imported (no value flows from the CUDA path)."""
    A = ops.wilson_dirac(3, -1.0, seed=9)
    rng = np.random.default_rng(3)
    th = 3.0 + 1.5 * rng.random(deg + 1) * np.exp(2j * np.pi * rng.random(deg + 1))
    qo = newton.from_nodes(th)
    q = pp.Poly.newton(qo.nodes, qo.dd)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    v = rng.standard_normal(A.n) + 1j * rng.standard_normal(A.n)
    got = host(q.apply(ctx, M, dev(v)))
    ref = newton.apply(qo, Operator(A.to_scipy()), v)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def _reference(cfg, A, b):
    p = cfg.params
    if cfg.family == "laplacian":
        return reference.laplacian_fAb(p["N"], p["dim"], b, cfg.func)
    if cfg.family == "convdiff":
        return reference.convdiff_fAb(p["N"], p["dim"], p["beta"], b, cfg.func)
    return reference.arnoldi_reference(Operator(A.to_scipy()), b, func=cfg.func).x


def _clenshaw_np(q, op, v):
    """Test-local Clenshaw evaluation of a Chebyshev q (numpy): a rounding
    perturbation of the oracle's forward recurrence, same mathematics."""
    al, be = 2 / (q.b - q.a), -(q.a + q.b) / (q.b - q.a)
    d = q.deg
    if d == 0:
        return q.c[0] * v
    b1 = q.c[d] * v
    b2 = np.zeros_like(v)
    for k in range(d - 1, 0, -1):
        b1, b2 = q.c[k] * v + 2 * (al * op.matvec(b1) + be * b1) - b2, b1
    return q.c[0] * v + (al * op.matvec(b1) + be * b1) - b2


def h_tolerance(A, b, q, **kw):
    """H-parity bar: 1e-11 (north_star), raised only where the Arnoldi process
    itself amplifies rounding beyond it.  The amplification is measured, not
    assumed: two oracle runs that differ only in the rounding of q(A)v
    (forward recurrence vs Clenshaw) -- e.g. C2 deg 20 (cond(D) = 4e8,
    SURVEY F3) gives 1.2e-10.  The bar is then 10x that oracle-vs-oracle gap."""
    if not isinstance(q, chebyshev.ChebPoly):
        return H_TOL
    op = Operator(A.to_scipy())
    r1 = krylov.run(op, b, q, stop="fixed", **kw)
    orig = krylov.apply_q
    try:
        krylov.apply_q = _clenshaw_np
        r2 = krylov.run(op, b, q, stop="fixed", **kw)
    finally:
        krylov.apply_q = orig
    gap = np.abs(r1.H - r2.H).max() / np.abs(r1.H).max()
    return max(H_TOL, 10 * gap)


def _compare(ctx, res_o, x_gpu, rep, complex_, h_tol=H_TOL):
    assert rep.iterations == res_o.m
    assert np.linalg.norm(x_gpu - res_o.x) <= X_TOL * np.linalg.norm(res_o.x)
    Hg, beta0 = pp.hessenberg(ctx, complex_)
    Ho = res_o.H
    assert Hg.shape == Ho.shape
    assert np.abs(Hg - Ho).max() <= h_tol * np.abs(Ho).max()
    assert beta0 == pytest.approx(res_o.beta0, rel=1e-13)


CASES = [("C1", 4), ("C2", 5), ("C2", 10), ("C2", 20), ("C3s", 10), ("C3s", 20), ("C4s", 20),
         ("C4s", 5)]


@pytest.mark.parametrize("name,deg", CASES)
@pytest.mark.parametrize("cgs", ["flat", "wide", "tiled"])
def test_run_parity_true_error(ctx, name, deg, cgs, monkeypatch):
    """End to end at the same m*: both sides stop at the first m whose true
    error (vs the closed form) is <= tol (reading Q11)."""
    monkeypatch.setenv("PPF_CGS_FLAT", "1" if cgs == "flat" else "0")
    monkeypatch.setenv("PPF_CGS_WIDE", "1" if cgs == "wide" else "0")
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    xr = _reference(cfg, A, b)
    qo = chebyshev.coefficients(*iv, deg)
    res_o = krylov.find_m_star(Operator(A.to_scipy()), b, qo, func=cfg.func, krylov=cfg.krylov,
                               m_max=cfg.m_max, tol=cfg.tol, x_ref=xr)
    assert res_o.term == "converged"
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    q = pp.Poly.chebyshev(*iv, deg)
    xg, rep = pp.run(ctx, M, q, dev(b), func=cfg.func, krylov=cfg.krylov, m_max=cfg.m_max,
                     stop="true", tol=cfg.tol, x_ref=dev(xr))
    assert rep.term == "converged"
    htol = h_tolerance(A, b, qo, func=cfg.func, krylov=cfg.krylov, m_max=res_o.m)
    _compare(ctx, res_o, host(xg), rep, False, htol)
    assert rep.mvms == res_o.mvms
    assert rep.inner_products == res_o.inner_products


@pytest.mark.parametrize("name,deg,C_", [("C2", 10, 64), ("C2", 5, 32), ("C2", 20, 32), ("C3s", 10, 64),
                                         ("C4s", 20, 64)])
@pytest.mark.parametrize("cgs", ["flat", "wide", "tiled"])
def test_run_parity_estimate_stop(ctx, name, deg, C_, cgs, monkeypatch):
    """The paper's practical criterion: both stop at the same m
    (C2 also in SELL-32, the layout bench.py times it in)."""
    monkeypatch.setenv("PPF_CGS_FLAT", "1" if cgs == "flat" else "0")
    monkeypatch.setenv("PPF_CGS_WIDE", "1" if cgs == "wide" else "0")
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    qo = chebyshev.coefficients(*iv, deg)
    res_o = krylov.run(Operator(A.to_scipy()), b, qo, func=cfg.func, krylov=cfg.krylov,
                       m_max=cfg.m_max, stop="est", tol=cfg.tol)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=C_))
    xg, rep = pp.run(ctx, M, pp.Poly.chebyshev(*iv, deg), dev(b), func=cfg.func,
                     krylov=cfg.krylov, m_max=cfg.m_max, stop="est", tol=cfg.tol)
    htol = h_tolerance(A, b, qo, func=cfg.func, krylov=cfg.krylov, m_max=res_o.m)
    _compare(ctx, res_o, host(xg), rep, False, htol)
    hist = pp.history(ctx)
    assert [h["m"] for h in hist] == [h["m"] for h in res_o.history]
    for hg, ho in zip(hist, res_o.history):
        if ho["est"] is not None:
            assert hg["est"] == pytest.approx(ho["est"], rel=1e-6, abs=1e-13)


@pytest.mark.parametrize("fmt,C_,sig", FORMATS)
def test_run_parity_formats_fixed_m(ctx, fmt, C_, sig):
    cfg = configs.CONFIGS["C4s"]
    A, b, iv = configs.build("C4s")
    qo = chebyshev.coefficients(*iv, 5)
    res_o = krylov.run(Operator(A.to_scipy()), b, qo, func="sqrt", krylov="cgs2", m_max=9)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt=fmt, C_=C_, sigma=sig))
    xg, rep = pp.run(ctx, M, pp.Poly.chebyshev(*iv, 5), dev(b), func="sqrt", krylov="cgs2",
                     m_max=9, stop="fixed")
    _compare(ctx, res_o, host(xg), rep, False)


def test_c5_small_parity_shared_q(ctx):
    """C5 family (complex128, Wilson-Dirac 4^4): H- and x-parity with the
    oracle's Ritz-Newton q imported into the library (reading Q19)."""
    cfg = configs.CONFIGS["C5s"]
    A, b, _ = configs.build("C5s")
    op = Operator(A.to_scipy())
    qo, _, _ = newton.ritz_newton(op, b, 16)
    xr = reference.arnoldi_reference(op, b).x
    res_o = krylov.find_m_star(op, b, qo, func="invsqrt", krylov="cgs2", m_max=cfg.m_max,
                               tol=cfg.tol, x_ref=xr)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    q = pp.Poly.newton(qo.nodes, qo.dd)
    xg, rep = pp.run(ctx, M, q, dev(b), func="invsqrt", krylov="cgs2", m_max=cfg.m_max,
                     stop="true", tol=cfg.tol, x_ref=dev(xr))
    _compare(ctx, res_o, host(xg), rep, True)


def test_c5_small_library_ritz(ctx):
    """The library's own Ritz construction on the device: nodes agree
    with the oracle's as multisets (rounding-dependent at ~1e-11, F6), the
    interpolation property holds, and the run reaches the same m*."""
    cfg = configs.CONFIGS["C5s"]
    A, b, _ = configs.build("C5s")
    op = Operator(A.to_scipy())
    qo, _, _ = newton.ritz_newton(op, b, 16)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    bd = dev(b)
    q = pp.Poly.ritz_newton(ctx, M, bd, 16)
    ex = q.export()
    a_sorted = np.sort_complex(ex["nodes"])
    o_sorted = np.sort_complex(qo.nodes)
    assert np.abs(a_sorted - o_sorted).max() < 1e-8
    assert np.abs(q.eval(ex["nodes"]) - ex["nodes"] ** -0.5).max() < 1e-8
    xr = reference.arnoldi_reference(op, b).x
    res_o = krylov.find_m_star(op, b, qo, func="invsqrt", krylov="cgs2", m_max=cfg.m_max,
                               tol=cfg.tol, x_ref=xr)
    xg, rep = pp.run(ctx, M, q, bd, func="invsqrt", krylov="cgs2", m_max=cfg.m_max,
                     stop="true", tol=cfg.tol, x_ref=dev(xr))
    assert rep.iterations == res_o.m
    # own q on each side: the nodes differ at ~1e-11 (F6), the iterate only at
    # rounding level -- held to the north_star bar
    e_x = np.linalg.norm(host(xg) - res_o.x) / np.linalg.norm(res_o.x)
    print(f"C5s own-Ritz x gap {e_x:.2e} (bar {X_TOL:g})")
    assert e_x <= X_TOL


def test_library_ritz_closed_form(ctx):
    """The library's device Ritz construction against a closed form:
    the 1D Laplacian T_N from e_1 gives H_d = T_d, Ritz values
    2 - 2 cos(k pi/(d+1)); nodes Leja-ordered, max modulus first, real."""
    import scipy.sparse as sp
    N, d = 4096, 9
    T = sp.diags([-np.ones(N - 1), 2 * np.ones(N), -np.ones(N - 1)], [-1, 0, 1]).tocsr()
    A = CSR(N, T.indptr.astype(np.int64), T.indices.astype(np.int64), T.data.astype(np.float64))
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    e1 = np.zeros(N)
    e1[0] = 1.0
    q = pp.Poly.ritz_newton(ctx, M, dev(e1), d - 1)
    nodes = q.export()["nodes"]
    exact = np.sort(2 - 2 * np.cos(np.arange(1, d + 1) * np.pi / (d + 1)))
    assert np.abs(np.sort(nodes.real) - exact).max() < 1e-13
    assert np.abs(nodes.imag).max() == 0.0
    assert abs(nodes[0].real - exact.max()) < 1e-13


def test_run_host_matches_device(ctx):
    A, b, iv = configs.build("C1")
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    q = pp.Poly.chebyshev(*iv, 4)
    xd, rep_d = pp.run(ctx, M, q, dev(b), krylov="lanczos", m_max=20)
    bh = torch.from_numpy(b).pin_memory()
    xh = torch.empty_like(bh).pin_memory()
    _, rep_h = pp.run_host(ctx, M, q, bh, xh, krylov="lanczos", m_max=20)
    assert np.array_equal(host(xd), xh.numpy())
    assert rep_h.iterations == rep_d.iterations == 20


def test_edge_m1_deg0_and_breakdown(ctx):
    # m_max = 1 and deg 0 (plain Lanczos / Arnoldi, Table 1 d = 1)
    A, b, iv = configs.build("C1")
    for kry in ("lanczos", "cgs2"):
        for deg, m in ((0, 1), (0, 30), (3, 1)):
            qo = chebyshev.coefficients(*iv, deg)
            res_o = krylov.run(Operator(A.to_scipy()), b, qo, krylov=kry, m_max=m)
            M = pp.Matrix(ctx, pp.Plan.from_csr(A))
            xg, rep = pp.run(ctx, M, pp.Poly.chebyshev(*iv, deg), dev(b), krylov=kry, m_max=m)
            assert rep.iterations == m
            assert np.linalg.norm(host(xg) - res_o.x) <= X_TOL * np.linalg.norm(res_o.x)
    # breakdown: A with 3 distinct eigenvalues -> Krylov space exhausted at m = 3 (reading Q9)
    n = 300
    d = np.repeat([1.0, 2.0, 4.0], 100)
    rp = np.arange(n + 1, dtype=np.int64)
    Ad = CSR(n, rp, np.arange(n, dtype=np.int64), d)
    bb = np.random.default_rng(0).standard_normal(n)
    M = pp.Matrix(ctx, pp.Plan.from_csr(Ad))
    q = pp.Poly.chebyshev(1.0, 4.0, 2)
    for kry in ("lanczos", "cgs2"):
        xg, rep = pp.run(ctx, M, q, dev(bb), krylov=kry, m_max=10, stop="est", tol=1e-14)
        assert rep.term == "breakdown" and rep.iterations == 3
        assert np.linalg.norm(host(xg) - bb / np.sqrt(d)) <= 1e-12 * np.linalg.norm(bb)


def test_branch_errors(ctx):
    # Ritz values on the negative axis -> PPF_EBRANCH
    n = 64
    Ad = CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64),
             -np.linspace(1, 2, n) + 0j)
    M = pp.Matrix(ctx, pp.Plan.from_csr(Ad))
    with pytest.raises(api.L.PPFError) as e:
        pp.Poly.ritz_newton(ctx, M, dev(np.ones(n, dtype=complex)), 3)
    assert e.value.status == 5


@pytest.mark.parametrize("name,deg,kry", [("C2", 10, "cgs2"), ("C1", 4, "lanczos"), ("C4s", 5, "cgs2")])
def test_graph_replay_bitwise(ctx, name, deg, kry):
    """The CUDA-graph replay of the step's q(A)q(A) chain (ppf_ctx_set_graphs)
    launches the same kernels in the same order: x and H bitwise equal to the
    direct launches, and equal to the oracle within the usual bars."""
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    q = pp.Poly.chebyshev(*iv, deg)
    out = {}
    for on in (True, False):
        ctx.set_graphs(on)
        x, rep = pp.run(ctx, M, q, dev(b), func=cfg.func, krylov=kry, m_max=cfg.m_max, stop="est",
                        tol=cfg.tol)
        out[on] = (host(x), pp.hessenberg(ctx, False)[0], rep)
    ctx.set_graphs(True)
    assert np.array_equal(out[True][0], out[False][0])
    assert np.array_equal(out[True][1], out[False][1])
    assert out[True][2].iterations == out[False][2].iterations
    assert out[True][2].mvms == out[False][2].mvms
    # (launch counts differ by the work run ahead of the final checkpoint and
    # discarded: the look-ahead SpMVs, or a whole step when the host's f(H_m)
    # was the slower side -- a timing-dependent choice, so not compared)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 65, 257])
@pytest.mark.parametrize("kry", ["lanczos", "cgs2"])
@pytest.mark.parametrize("cgs", ["flat", "wide", "tiled"])
def test_tiny_and_ragged_sizes(ctx, n, kry, cgs, monkeypatch):
    """Sizes below one SELL slice (64 rows), one CGS2 chunk (256 rows) and
    ragged tails just past them: the run must match the oracle, including the
    bulk-copy tail of the CGS2 sweeps (one padding element for odd n)."""
    monkeypatch.setenv("PPF_CGS_FLAT", "1" if cgs == "flat" else "0")
    monkeypatch.setenv("PPF_CGS_WIDE", "1" if cgs == "wide" else "0")
    rng = np.random.default_rng(n)
    main = 2.0 + rng.random(n)
    off = 0.3 * rng.random(max(n - 1, 0))
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in ((i - 1, off[i - 1] if i > 0 else 0), (i, main[i]), (i + 1, off[i] if i + 1 < n else 0)):
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
                vals.append(v)
    import scipy.sparse as sp
    S = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    A = CSR(n, S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data.astype(np.float64))
    lam = np.linalg.eigvalsh(S.toarray())
    a, bb = 0.9 * lam.min(), 1.1 * lam.max()
    b = rng.standard_normal(n)
    m = min(n, 6)
    qo = chebyshev.coefficients(a, bb, 3)
    res_o = krylov.run(Operator(S), b, qo, krylov=kry, m_max=m)
    for fmt, C_ in (("sell", 64), ("sell", 32), ("csr", 32)):
        M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt=fmt, C_=C_))
        xg, rep = pp.run(ctx, M, pp.Poly.chebyshev(a, bb, 3), dev(b), krylov=kry, m_max=m)
        assert rep.iterations == res_o.m
        assert np.linalg.norm(host(xg) - res_o.x) <= X_TOL * np.linalg.norm(res_o.x)
