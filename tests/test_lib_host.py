"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/ppf.h declares, and its host-side logic (plan construction, Chebyshev
coefficients + certificate, polynomial evaluation, the host dense kernel K10)
agrees with the independent oracle.  No GPU calls are made here."""
import os
import re

import numpy as np
import pytest
import scipy.linalg as sla

from inputs import configs
from inputs import operators as ops
from oracle import chebyshev, contour_ls, dense, newton

from .conftest import ROOT

pp = pytest.importorskip("paper_2401_06684_b200")
from paper_2401_06684_b200 import _lib  # noqa: E402
from paper_2401_06684_b200.api import Plan, Poly, dense_invsqrt_e1  # noqa: E402


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "ppf.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(ppf_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 30
    lib = _lib.load()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding declares all of them
    assert names <= set(_lib.SIGNATURES), names - set(_lib.SIGNATURES)
    assert lib.ppf_abi_version() == 3


def test_no_batch_memcpy_in_sources():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2401_06684_b200", "csrc")):
        for f in files:
            src = open(os.path.join(dirpath, f)).read()
            assert "BatchAsync" not in src


@pytest.mark.parametrize("name,deg", [("C1", 4), ("C2", 5), ("C2", 20), ("C3", 40), ("C4", 20)])
def test_chebyshev_coefficients_match_oracle(name, deg):
    cfg = configs.CONFIGS[name]
    p = cfg.params
    if cfg.family == "laplacian":
        a, b = ops.laplacian_interval(p["N"], p["dim"])
    else:
        a, b = ops.convdiff_interval(p["N"], p["dim"], p["beta"])
    q = Poly.chebyshev(a, b, deg).export()
    ref = chebyshev.coefficients(a, b, deg)
    assert q["kind"] == "chebyshev" and q["deg"] == deg
    assert np.abs(q["c"] - ref.c).max() <= 1e-13 * np.abs(ref.c).max()
    z = chebyshev.certificate_points(a, b)
    got = Poly.chebyshev(a, b, deg).eval(z)
    assert np.abs(got.real - chebyshev.evaluate(ref, z)).max() <= 1e-12 * np.abs(ref.c).sum()


def test_chebyshev_golden_c1():
    # SURVEY §8(c) golden host-side values for C1 (interpolant on the closed-form interval)
    a, b = ops.laplacian_interval(32, 2)
    c = Poly.chebyshev(a, b, 4).export()["c"]
    assert c[0] == pytest.approx(0.83970316174, abs=1e-10)
    assert c[1] == pytest.approx(-0.777096031927, abs=1e-11)


def test_chebyshev_invalid_arguments():
    with pytest.raises(_lib.PPFError) as e:
        Poly.chebyshev(0.0, 1.0, 3)
    assert e.value.status == _lib.PPF_OK + 1  # EINVAL
    with pytest.raises(_lib.PPFError):
        Poly.chebyshev(2.0, 1.0, 3)
    with pytest.raises(_lib.PPFError):
        Poly.chebyshev(1.0, 2.0, -1)


@pytest.mark.parametrize("name,deg", [("C1", 4), ("C3", 10), ("C4", 20)])
def test_poly_certify_chebyshev(name, deg):
    """ppf_poly_certify: on the default grid the minimum is
    the oracle's certificate of the same polynomial; on real and complex point
    sets it is min Re q there (the oracle's evaluation)."""
    iv = configs.build(name)[2] if name == "C1" else None
    if iv is None:
        cfg = configs.CONFIGS[name]
        p = cfg.params
        iv = (ops.laplacian_interval(p["N"], p["dim"]) if cfg.family == "laplacian"
              else ops.convdiff_interval(p["N"], p["dim"], p["beta"]))
    q = Poly.chebyshev(*iv, deg)
    qo = chebyshev.coefficients(*iv, deg)
    assert q.certify() == pytest.approx(chebyshev.certify(qo), rel=1e-12)
    pts = np.linspace(iv[0], iv[1], 333)
    assert q.certify(pts) == pytest.approx(chebyshev.evaluate(qo, pts).min(), rel=1e-12)
    zc_ = pts + 0.01j * (iv[1] - iv[0])
    assert q.certify(zc_) == pytest.approx(q.eval(zc_).real.min(), rel=1e-14)


def test_poly_certify_failure_and_contour():
    """The certificate fails (PPF_EBRANCH, minimum reported) where q has a zero:
    the degree-3 interpolant of z^{-1/2} on [1, 9] at points beyond the
    interval; the least-squares q's certificate equals the value
    ppf_poly_contour_ls reported."""
    q = Poly.chebyshev(1.0, 9.0, 3)
    zs = np.linspace(1.0, 60.0, 400)
    vals = chebyshev.evaluate(chebyshev.coefficients(1.0, 9.0, 3), zs)
    assert vals.min() <= 0.0          # the oracle says q has a zero past b
    with pytest.raises(_lib.PPFError) as e:
        q.certify(zs)
    assert e.value.status == 5 and e.value.min_re == pytest.approx(vals.min(), rel=1e-12)
    z = contour_ls.circle(3.0, 2.2, 128)
    ql = Poly.contour_ls(z, 6)
    assert ql.certify(z) == ql.min_re
    assert ql.min_re == pytest.approx(contour_ls.certify(contour_ls.construct(z, 6)), rel=1e-10)
    with pytest.raises(_lib.PPFError) as e:
        ql.certify()                  # no default points for a Newton-form q
    assert e.value.status == 1


def test_newton_import_eval_matches_oracle():
    rng = np.random.default_rng(0)
    th = 3 + 2 * rng.random(10) * np.exp(2j * np.pi * rng.random(10))
    qo = newton.from_nodes(th)
    q = Poly.newton(qo.nodes, qo.dd)
    z = 3 + 1.8 * np.exp(1j * np.linspace(0, 2 * np.pi, 64))
    assert np.abs(q.eval(z) - newton.evaluate(qo, z)).max() < 1e-11
    assert np.abs(q.eval(qo.nodes) - qo.nodes ** -0.5).max() < 1e-10
    ex = q.export()
    assert np.array_equal(ex["nodes"], qo.nodes) and np.array_equal(ex["dd"], qo.dd)


@pytest.mark.parametrize("contour", ["circle", "ellipse"])
@pytest.mark.parametrize("deg", [0, 4, 16])
def test_contour_ls_matches_oracle(contour, deg):
    """ppf_poly_contour_ls (host, Newton form on Leja contour points) vs the
    oracle's least-squares polynomial (Arnoldi-like recurrence) at
    points inside and on the contour; the certificate min Re q."""
    if contour == "circle":
        z = contour_ls.circle(3.0, 2.2, 128)
    else:
        t = 2 * np.pi * np.arange(150) / 150
        z = 4.0 + 3.0 * np.cos(t) + 1.5j * np.sin(t)
    qo = contour_ls.construct(z, deg)
    q = Poly.contour_ls(z, deg)
    zz = np.concatenate([z, 0.5 * z + 0.5 * z.mean()])
    ref = contour_ls.evaluate(qo, zz)
    assert np.abs(q.eval(zz) - ref).max() < 1e-11 * np.abs(ref).max()
    assert q.min_re == pytest.approx(contour_ls.certify(qo), rel=1e-10)


@pytest.mark.parametrize("case", ["circle", "cut", "real", "cloud"])
def test_contour_from_ritz_matches_oracle(case):
    """ppf_contour_from_ritz (host C++) against the oracle's ritz_polygon: the
    same construction, so the same points to rounding."""
    from paper_2401_06684_b200.api import contour_from_ritz
    t = 2 * np.pi * np.arange(12) / 12
    rng = np.random.default_rng(5)
    th, r_min, step = {
        "circle": (3.0 + 2.0 * np.exp(1j * t), 0.1, 0.01),
        "cut": (3.0 + 2.0 * np.exp(1j * t), 1.5, 0.01),
        "real": (np.array([0.5, 2.0, 7.0]), 0.1, 0.05),
        "cloud": (4 + rng.standard_normal(30) + 1j * rng.standard_normal(30), 0.2, 0.02),
    }[case]
    z = contour_from_ritz(th, r_min, step)
    zo = contour_ls.ritz_polygon(th, r_min, step)
    assert z.shape == zo.shape
    assert np.abs(z - zo).max() < 1e-12


def test_contour_ls_rejects_branch_cut():
    # a circle around 0: the contour meets (-inf, 0]
    with pytest.raises(_lib.PPFError):
        Poly.contour_ls(contour_ls.circle(0.0, 1.0, 64), 4)


@pytest.mark.parametrize("m", [1, 2, 7, 25, 60])
def test_dense_tridiagonal_matches_oracle(m):
    rng = np.random.default_rng(m)
    T = np.diag(rng.uniform(0.3, 2.0, m))
    off = rng.uniform(0.01, 0.3, m - 1)
    T += np.diag(off, 1) + np.diag(off, -1)
    y = dense_invsqrt_e1(T, 1.7, hermitian=True)
    ref = dense.invsqrt_e1(T, 1.7, hermitian=True)
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("m", [1, 3, 12, 40, 75])
def test_dense_schur_matches_oracle(m):
    rng = np.random.default_rng(100 + m)
    H = np.triu(rng.standard_normal((m, m)) * 0.3, -1) + 2.5 * np.eye(m)
    y = dense_invsqrt_e1(H, 0.9, hermitian=False)
    ref = dense.invsqrt_e1(H, 0.9, hermitian=False)
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    Hc = H + 0.4j * np.triu(rng.standard_normal((m, m)), -1)
    yc = dense_invsqrt_e1(Hc, 0.9, hermitian=False)
    refc = 0.9 * np.linalg.solve(sla.sqrtm(Hc), np.eye(m)[:, 0])
    assert np.linalg.norm(yc - refc) <= 1e-11 * np.linalg.norm(refc)


@pytest.mark.parametrize("m", [2, 3, 7, 25, 60, 130])
@pytest.mark.parametrize("kind", ["real_eigs", "complex_pairs", "stiff"])
def test_dense_real_schur_matches_oracle(m, kind):
    """Real Hessenberg H (a real operator's Arnoldi matrix): the library's real
    Schur route (Francis double shift, quasi-triangular square root) against
    the oracle's eigendecomposition, with real eigenvalues, complex pairs and a
    wide spectrum; and against the complex Schur route of the same matrix."""
    rng = np.random.default_rng(7 * m + len(kind))
    H = np.triu(rng.standard_normal((m, m)), -1)
    if kind == "real_eigs":
        H = np.triu(rng.random((m, m)), -1) * 0.2 + np.diag(np.linspace(0.5, 3.0, m))
    elif kind == "complex_pairs":
        H += np.diag(np.full(m, 2.0 * np.sqrt(m)))
    else:
        H = (np.triu(rng.random((m, m)), 1) * 0.3 + np.diag(rng.random(m - 1) * 0.01, -1)
             + np.diag(np.geomspace(0.05, 5e3, m)))
    ev = np.linalg.eigvals(H)
    assert not np.any((np.abs(ev.imag) < 1e-12) & (ev.real <= 0))
    y = dense_invsqrt_e1(H, 0.7, hermitian=False)
    ref = dense.invsqrt_e1(H.astype(np.complex128), 0.7, hermitian=False)
    assert np.linalg.norm(y - ref) <= 1e-11 * np.linalg.norm(ref)
    yc = dense_invsqrt_e1(H.astype(np.complex128), 0.7, hermitian=False)
    assert np.linalg.norm(y - yc) <= 1e-11 * np.linalg.norm(yc)


@pytest.mark.parametrize("m", [30, 60])
def test_dense_real_schur_nearly_symmetric(m):
    """CGS2-Arnoldi matrix of a symmetric operator (C1, plain method): a real
    Hessenberg with converged 2x2 blocks whose off-diagonals are ~1e-15 --
    the case that needs the cancellation-free 2x2 standardisation."""
    from oracle import krylov
    from oracle.spmv import Operator
    A, b, iv = configs.build("C1")
    r = krylov.run(Operator(A.to_scipy()), b, chebyshev.coefficients(*iv, 0), krylov="cgs2",
                   m_max=m)
    H = r.H[:m, :m].real.copy()
    y = dense_invsqrt_e1(H, r.beta0, hermitian=False)
    assert np.linalg.norm(y - r.y) <= 1e-12 * np.linalg.norm(r.y)


def test_dense_real_schur_branch_cut():
    H = np.array([[1.0, 2.0, 0.0], [1.0, -3.0, 1.0], [0.0, 0.5, 2.0]])
    assert np.any(np.linalg.eigvals(H).real < 0)
    with pytest.raises(_lib.PPFError):
        dense_invsqrt_e1(H, 1.0, hermitian=False)


def test_dense_branch_cut_rejected():
    with pytest.raises(_lib.PPFError) as e:
        dense_invsqrt_e1(np.diag([1.0, -2.0]), 1.0, hermitian=True)
    assert e.value.status == 5
    with pytest.raises(_lib.PPFError):
        dense_invsqrt_e1(np.array([[1.0, 1.0], [0.0, -4.0]]), 1.0, hermitian=False)


def test_plan_sell_layout_sizes():
    A = ops.laplacian(10, 3)
    for fmt, C_, sig in (("sell", 32, 1), ("sell", 64, 1), ("sell", 32, 64), ("csr", 32, 1)):
        p = Plan.from_csr(A, fmt=fmt, C_=C_, sigma=sig)
        info = p.info()
        assert info["n_local"] == A.n and info["nnz"] == A.nnz and info["halo_total"] == 0
        if fmt == "csr":
            assert info["stored"] == A.nnz
        else:
            assert A.nnz <= info["stored"] <= 7 * (A.n + C_)
        # 8-byte values + 4-byte indices, or one byte per entry where the
        # SELL-64 plan stores the stencil's entries as pair codes
        ib = p.index_bits()
        assert ib == (8 if (fmt, C_, sig) == ("sell", 64, 1) else 32)   # fp64 operator
        per = {32: 12, 16: 10, 8: 1}[ib]
        assert p.device_bytes() >= info["stored"] * per
        if ib == 8:
            assert p.device_bytes() < info["stored"] * 2


def test_plan_rejects_bad_input():
    A = ops.laplacian(4, 2)
    bad = A.col.copy()
    bad[3], bad[4] = bad[4], bad[3]
    with pytest.raises(_lib.PPFError):
        Plan(A.row_ptr, bad, A.val, n_global=A.n)
    with pytest.raises(_lib.PPFError):
        Plan(A.row_ptr, A.col, A.val, n_global=A.n, fmt="sell", C_=48)
    rp = A.row_ptr.copy()
    rp[5] = rp[4] - 1
    with pytest.raises(_lib.PPFError):
        Plan(rp, A.col, A.val, n_global=A.n)


def test_plan_halo_lists_two_slabs():
    """Row-slab sharding: the halo of a z-slab of the 3D Laplacian
    is exactly the neighbouring z-plane."""
    N = 6
    A = ops.laplacian(N, 3)
    bounds = [0, 3 * N * N, N**3]
    for rank in (0, 1):
        lo, hi = bounds[rank], bounds[rank + 1]
        rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
        sl = slice(A.row_ptr[lo], A.row_ptr[hi])
        p = Plan(rp, A.col[sl], A.val[sl], row_bounds=bounds, rank=rank)
        peer = 1 - rank
        got = p.halo_recv(peer)
        plane = np.arange(N * N) + (3 * N * N if rank == 0 else 2 * N * N)
        assert np.array_equal(got, plane)
        assert len(p.halo_recv(rank)) == 0
        assert p.info()["halo_total"] == N * N


def test_pair_codes_per_slab():
    """Each rank's plan codes its own diagonal block: the z-slabs of a 3D
    convection-diffusion stencil both get pair codes (the off-slab neighbours
    go to the halo block, so a slab may have fewer pairs than the whole
    matrix), the device layout is ~1 byte per diagonal-block entry, and the
    halo lists are those of the explicit layout."""
    N = 12
    A = ops.convdiff(N, 3, (10.0, 10.0, 10.0))
    bounds = [0, 5 * N * N, N**3]
    for rank in (0, 1):
        lo, hi = bounds[rank], bounds[rank + 1]
        rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
        sl = slice(A.row_ptr[lo], A.row_ptr[hi])
        p = Plan(rp, A.col[sl], A.val[sl], row_bounds=bounds, rank=rank, fmt="sell", C_=64)
        enc, ntab = p.encoding()
        assert enc == "pair8" and 7 <= ntab <= 13, (enc, ntab)
        halo = p.halo_recv(1 - rank)
        p.set_encoding("explicit")
        assert np.array_equal(p.halo_recv(1 - rank), halo)
        assert len(halo) == N * N


def test_real_pair_form_same_polynomial():
    """ppf_poly_set_newton_eval("pairs") on a Newton q with conjugate-pair nodes
    (the Ritz values of the real, convection-dominated C8s operator): the
    reordered real form is the same polynomial as the oracle's Newton form
    (evaluated at points off the nodes) and still interpolates z^{-1/2}."""
    from oracle.spmv import Operator
    A, b, _ = configs.build("C8s")
    qo, _, _ = newton.ritz_newton(Operator(A.to_scipy()), b, 9)
    assert np.abs(qo.nodes.imag).max() > 1.0
    q = Poly.newton(qo.nodes, qo.dd).set_newton_eval("pairs")
    ex = q.export()
    nodes = ex["nodes"]
    # pairs adjacent: every complex node is followed by its conjugate
    i = 0
    while i < len(nodes):
        if abs(nodes[i].imag) > 0:
            assert nodes[i + 1] == np.conj(nodes[i])
            i += 2
        else:
            i += 1
    z = nodes.real.mean() + np.abs(nodes).max() * 0.3 * np.exp(1j * np.linspace(0, 6, 40))
    ref = newton.evaluate(qo, z)
    assert np.abs(q.eval(z) - ref).max() <= 1e-9 * np.abs(ref).max()
    assert np.abs(q.eval(qo.nodes) - qo.nodes ** -0.5).max() <= 1e-8 * np.abs(qo.nodes ** -0.5).max()


def test_fake_nccl_test_library_links():
    """The multi-process NCCL-path test (test_gpu_multirank, transport "nccl")
    links the product objects with tests/native/fake_nccl.cpp; it must build
    here and export the NCCL entry points the library calls."""
    import subprocess
    from tests.native import build_fake
    path = build_fake.build()
    syms = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True,
                          text=True).stdout
    for s in ("ncclCommInitRank", "ncclSend", "ncclRecv", "ncclAllReduce", "ncclGroupEnd",
              "ppf_run"):
        assert f" {s}\n" in syms


def test_header_is_plain_c_and_links(tmp_path):
    """include/ppf.h is a C header (no C++ in the signatures): a C99 program
    includes it, links against libppf.so and calls the host-only entry points
    (ABI version, status strings, the Chebyshev polynomial of P:323-335)."""
    import subprocess
    from paper_2401_06684_b200 import _lib
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "abi.c"
    src.write_text(r"""
#include <stdio.h>
#include "ppf.h"
int main(void) {
  ppf_poly* q = NULL;
  double ab[2];
  int kind = -1, deg = -1;
  if (ppf_abi_version() != PPF_ABI_VERSION) return 1;
  if (ppf_poly_chebyshev(0.5, 8.0, 6, &q) != PPF_OK) return 2;
  if (ppf_poly_export(q, &kind, &deg, ab, NULL, NULL) != PPF_OK) return 3;
  ppf_poly_destroy(q);
  if (kind != PPF_POLY_CHEBYSHEV || deg != 6 || ab[0] != 0.5 || ab[1] != 8.0) return 4;
  if (ppf_poly_chebyshev(-1.0, 8.0, 6, &q) != PPF_EINVAL) return 5;
  printf("%s|%s\n", ppf_status_string(PPF_EINVAL), ppf_last_error());
  return 0;
}
""")
    exe = tmp_path / "abi"
    libdir = os.path.dirname(_lib.LIB_PATH)
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                        str(src), "-o", str(exe), "-L", libdir, "-l:libppf.so",
                        f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "EINVAL" in r.stdout.upper() or "INVAL" in r.stdout.upper()


def test_plan_index_bits_choice(monkeypatch):
    """ppf_plan_index_bits: the SELL-64 fp64 plan stores 16-bit column deltas
    relative to the row when every slice-column spans <= 65535 (stencils,
    including the 256^3 conv-diff of C4 whose offsets reach N^2 = 65536 but
    span at most N^2 - 1 within one slice-column), 32-bit indices otherwise
    (columns spread over 200,000) or when PPF_IDX16=0."""
    monkeypatch.setenv("PPF_PAIR8", "0")
    A = ops.convdiff(40, 3, (10.0, 10.0, 10.0))
    assert Plan.from_csr(A, fmt="sell", C_=64).index_bits() == 16
    assert Plan.from_csr(A, fmt="sell", C_=32).index_bits() == 32          # fp64 SELL-32: no
    W = ops.wilson_dirac(4, -1.0, seed=5)                                   # complex SELL-32: yes
    assert Plan.from_csr(W, fmt="sell", C_=32).index_bits() == 16
    assert Plan.from_csr(W, fmt="sell", C_=32, sigma=64).index_bits() == 32
    monkeypatch.setenv("PPF_IDX16", "0")
    assert Plan.from_csr(A, fmt="sell", C_=64).index_bits() == 32
    monkeypatch.delenv("PPF_IDX16")
    n = 200_000
    i = np.arange(n, dtype=np.int64)
    cols = np.sort(np.stack([i, (i * 7919) % n, (i * 104729 + 17) % n], axis=1), axis=1)
    keep = np.ones_like(cols, dtype=bool)
    keep[:, 1:] = cols[:, 1:] != cols[:, :-1]            # distinct, sorted per row
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=rp[1:])
    from inputs.operators import CSR
    R = CSR(n, rp, cols[keep], np.ones(int(rp[-1])))
    assert Plan.from_csr(R, fmt="sell", C_=64).index_bits() == 32


def test_plan_pair_codes_choice(monkeypatch):
    """ppf_plan_encoding: SELL-64 fp64 without sorting stores each entry as an
    8-bit code into a table of (col - row, value) pairs when there are at most
    256 distinct pairs, padding (0, 0.0) included: the constant-coefficient
    stencils (7 pairs + padding); complex, sorted, SELL-32, CSR and
    variable-coefficient operators keep the wider layouts.  PPF_PAIR8=0 and
    ppf_plan_set_encoding select a wider one; an unavailable one is EINVAL."""
    from inputs.operators import CSR
    for A in (ops.convdiff(40, 3, (10.0, 10.0, 10.0)), ops.laplacian(30, 3), ops.laplacian(32, 2)):
        p = Plan.from_csr(A, fmt="sell", C_=64)
        enc, ntab = p.encoding()
        nd = 2 * (3 if A.n in (64000, 27000) else 2) + 1     # distinct diagonals
        assert enc == "pair8" and ntab == nd + 1, (enc, ntab)
        assert p.index_bits() == 8
        stored = p.info()["stored"]
        b8 = p.device_bytes()
        p.set_encoding("delta16")
        assert p.encoding() == ("delta16", 0) and p.index_bits() == 16
        assert p.device_bytes() >= 10 * stored > 5 * b8
        p.set_encoding("explicit")
        assert p.index_bits() == 32 and p.device_bytes() >= 12 * stored
        p.set_encoding("pair8")                      # back: still available
        assert p.device_bytes() == b8
    A = ops.convdiff(20, 3, (10.0, 10.0, 10.0))
    assert Plan.from_csr(A, fmt="sell", C_=32).encoding()[0] == "explicit"
    assert Plan.from_csr(A, fmt="csr").encoding()[0] == "explicit"
    W = ops.wilson_dirac(4, -1.0, seed=5)
    pw = Plan.from_csr(W, fmt="sell", C_=32)
    assert pw.encoding()[0] == "delta16"
    with pytest.raises(RuntimeError):
        pw.set_encoding("pair8")
    # variable coefficients: 257+ distinct values -> the deltas
    V = CSR(A.n, A.row_ptr, A.col, A.val * (1.0 + 1e-3 * (np.arange(A.nnz) % 300)))
    assert Plan.from_csr(V, fmt="sell", C_=64).encoding()[0] == "delta16"
    # exactly 256 distinct pairs (padding included) still fits; 257 does not
    n = 64 * 8
    rp = np.arange(n + 1, dtype=np.int64)
    for k in (256, 257):
        vals = 1.0 + (np.arange(n) % k)                  # k values on the diagonal
        D = CSR(n, rp, np.arange(n, dtype=np.int64), vals)
        enc = Plan.from_csr(D, fmt="sell", C_=64).encoding()
        # a diagonal matrix has no padding: k pairs
        assert (enc[0] == "pair8") == (k <= 256)
        if enc[0] == "pair8":
            assert enc[1] == k
    monkeypatch.setenv("PPF_PAIR8", "0")
    assert Plan.from_csr(ops.laplacian(30, 3), fmt="sell", C_=64).encoding()[0] == "delta16"


def test_pair_code_slice_schedule(monkeypatch):
    """ppf_plan_slice_schedule: with PPF_SELLP_TILE=TYxTZ every slice appears
    exactly once, 8 entries per block, and the live warps of a block are slices
    G1 = N / 64 (y-neighbours) and G2 = N^2 / 64 (z-neighbours) apart; a 2-D
    stencil (one far offset) gets tiles of 8 along y; ragged sizes (N not a
    multiple of 64) still cover every slice once; PPF_SELLP_TILE=0, a wider
    layout or a small block give the in-order launch (empty schedule)."""
    monkeypatch.setenv("PPF_SELLP_TILE", "4x2")
    N = 64
    A = ops.convdiff(N, 3, (10.0, 10.0, 10.0))
    p = Plan.from_csr(A, fmt="sell", C_=64)
    s = p.slice_schedule()
    ns = N**3 // 64
    assert len(s) % 8 == 0 and len(s) == ns           # N = 64: no dead warps
    assert np.array_equal(np.sort(s), np.arange(ns))
    blk = s.reshape(-1, 8)
    G1, G2 = N // 64, N * N // 64
    assert np.array_equal(blk[:, 1] - blk[:, 0], np.full(len(blk), G1))
    assert np.array_equal(blk[:, 4] - blk[:, 0], np.full(len(blk), G2))
    p.set_encoding("delta16")
    assert len(p.slice_schedule()) == 0
    for tile in ("8x1", "2x4", "1x8"):
        monkeypatch.setenv("PPF_SELLP_TILE", tile)
        s = Plan.from_csr(A, fmt="sell", C_=64).slice_schedule()
        assert np.array_equal(np.sort(s[s >= 0]), np.arange(ns)), tile
    monkeypatch.setenv("PPF_SELLP_TILE", "4x2")
    for B in (ops.convdiff(40, 3, (10.0, 10.0, 10.0)), ops.laplacian(30, 3), ops.laplacian(100, 2)):
        s = Plan.from_csr(B, fmt="sell", C_=64).slice_schedule()
        nsb = (B.n + 63) // 64
        assert len(s) % 8 == 0 and len(s) >= nsb
        assert np.array_equal(np.sort(s[s >= 0]), np.arange(nsb))
        assert (s >= -1).all() and (s.reshape(-1, 8) >= 0).any(axis=1).all()   # no empty block
    s2 = Plan.from_csr(ops.laplacian(100, 2), fmt="sell", C_=64).slice_schedule().reshape(-1, 8)
    full = (s2 >= 0).all(axis=1)
    assert full.any() and (np.diff(s2[full], axis=1) == round(100 / 64)).all()   # 8 along y
    assert len(Plan.from_csr(ops.laplacian(32, 2), fmt="sell", C_=64).slice_schedule()) == 0  # 16 slices
    monkeypatch.setenv("PPF_SELLP_TILE", "0")
    assert len(Plan.from_csr(A, fmt="sell", C_=64).slice_schedule()) == 0
