"""Thin Python binding over the C ABI (include/ppf.h), same names as the calls.

Argument marshalling only: every step of the hot path runs inside libppf.so.
PyTorch provides device memory and streams.  Citations: PAPER.md lines (P:n).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import check


def _lib():
    return L.load()


def _torch():
    import torch
    return torch


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _stream_handle(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Context:
    """ppf_ctx_create: one per GPU/rank, bound to a CUDA stream."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None,
                 stream=None):
        torch = _torch()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        check(_lib().ppf_ctx_create(device, rank, nranks, idbuf, _stream_handle(self.stream),
                                    C.byref(h)))
        self.h = h
        self.rank, self.nranks = rank, nranks

    def set_graphs(self, on: bool):
        """ppf_ctx_set_graphs: CUDA-graph replay of the step's q(A)q(A) chain."""
        check(_lib().ppf_ctx_set_graphs(self.h, int(bool(on))))

    def set_transport(self, exchange, allreduce_sum):
        """ppf_ctx_set_transport: host-side halo exchange / sum over ranks.

        exchange(send: ndarray, send_counts: list, recv: ndarray, recv_counts: list)
        fills ``recv`` (float64, per-peer segments in peer order); allreduce_sum(buf)
        sums ``buf`` (float64) over all ranks in place.  Exceptions -> nonzero."""
        nr = self.nranks

        def _ex(user, send, sc, recv, rc):
            try:
                scount = [int(sc[p]) for p in range(nr)]
                rcount = [int(rc[p]) for p in range(nr)]
                s_arr = np.ctypeslib.as_array(send, shape=(max(1, sum(scount)),))[: sum(scount)]
                r_arr = np.ctypeslib.as_array(recv, shape=(max(1, sum(rcount)),))[: sum(rcount)]
                exchange(s_arr, scount, r_arr, rcount)
                return 0
            except Exception:  # pragma: no cover - reported as PPF_ENCCL
                import traceback
                traceback.print_exc()
                return 1

        def _ar(user, buf, count):
            try:
                allreduce_sum(np.ctypeslib.as_array(buf, shape=(int(count),)))
                return 0
            except Exception:  # pragma: no cover
                import traceback
                traceback.print_exc()
                return 1

        self._transport = L.Transport(None, L.EXCHANGE_FN(_ex), L.ALLREDUCE_FN(_ar))
        check(_lib().ppf_ctx_set_transport(self.h, C.byref(self._transport)))

    def close(self):
        if self.h:
            _lib().ppf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def contour_from_ritz(theta, r_min: float, step: float) -> np.ndarray:
    """ppf_contour_from_ritz: the Ritz-polygon contour (complex points)."""
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.complex128))
    n = C.c_int()
    check(_lib().ppf_contour_from_ritz(th.ctypes.data_as(C.c_void_p), len(th), float(r_min),
                                       float(step), 0, None, C.byref(n)))
    out = np.empty(n.value, dtype=np.complex128)
    check(_lib().ppf_contour_from_ritz(th.ctypes.data_as(C.c_void_p), len(th), float(r_min),
                                       float(step), n.value, out.ctypes.data_as(C.c_void_p),
                                       C.byref(n)))
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_lib().ppf_nccl_unique_id(buf))
    return buf.raw


class Plan:
    """ppf_plan_create: host conversion of this rank's CSR slab (no GPU needed)."""

    def __init__(self, row_ptr, col, val, n_global: int | None = None, row_bounds=None, rank: int = 0,
                 fmt: str = "sell", C_: int = 32, sigma: int = 1):
        val = np.ascontiguousarray(val)
        self.dtype = L.C128 if np.iscomplexobj(val) else L.R64
        val = val.astype(np.complex128 if self.dtype == L.C128 else np.float64, copy=False)
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int64)
        n_local = len(row_ptr) - 1
        if row_bounds is None:
            row_bounds = [0, n_local if n_global is None else n_global]
        row_bounds = np.ascontiguousarray(row_bounds, dtype=np.int64)
        self.nranks = len(row_bounds) - 1
        self.rank = rank
        self.n_global = int(row_bounds[-1])
        self.row_bounds = row_bounds
        h = C.c_void_p()
        f = {"sell": L.FMT_SELL, "csr": L.FMT_CSR}[fmt]
        check(_lib().ppf_plan_create(self.dtype, self.n_global, self.nranks, rank,
                                     _ptr(row_bounds, C.c_int64), _ptr(row_ptr, C.c_int64),
                                     _ptr(col, C.c_int64), val.ctypes.data_as(C.c_void_p), f, C_,
                                     sigma, C.byref(h)))
        self.h = h

    @classmethod
    def from_csr(cls, A, **kw):
        """From an ``inputs.CSR`` (whole matrix, one rank)."""
        return cls(A.row_ptr, A.col, A.val, n_global=A.n, **kw)

    def device_bytes(self) -> int:
        b = C.c_size_t()
        check(_lib().ppf_plan_device_bytes(self.h, C.byref(b)))
        return b.value

    def info(self):
        n, z, s, h = (C.c_int64() for _ in range(4))
        check(_lib().ppf_plan_info(self.h, C.byref(n), C.byref(z), C.byref(s), C.byref(h)))
        return dict(n_local=n.value, nnz=z.value, stored=s.value, halo_total=h.value)

    def index_bits(self) -> int:
        """ppf_plan_index_bits: 8 (pair codes), 16 (column deltas) or 32."""
        b = C.c_int()
        check(_lib().ppf_plan_index_bits(self.h, C.byref(b)))
        return b.value

    ENCODINGS = ("explicit", "delta16", "pair8")

    def encoding(self) -> tuple[str, int]:
        """ppf_plan_encoding: (layout name, pair-table size or 0)."""
        e, t = C.c_int(), C.c_int()
        check(_lib().ppf_plan_encoding(self.h, C.byref(e), C.byref(t)))
        return self.ENCODINGS[e.value], t.value

    def slice_schedule(self) -> np.ndarray:
        """ppf_plan_slice_schedule: slice of warp w of block b at [8 b + w] (-1: none);
        empty = slices in order."""
        cnt = C.c_int64()
        check(_lib().ppf_plan_slice_schedule(self.h, None, 0, C.byref(cnt)))
        out = np.empty(cnt.value, dtype=np.int32)
        if cnt.value:
            check(_lib().ppf_plan_slice_schedule(
                self.h, out.ctypes.data_as(C.POINTER(C.c_int32)), cnt.value, C.byref(cnt)))
        return out

    def set_encoding(self, enc: str) -> "Plan":
        """ppf_plan_set_encoding: select a wider layout than the one chosen."""
        check(_lib().ppf_plan_set_encoding(self.h, self.ENCODINGS.index(enc)))
        return self

    def halo_recv(self, peer: int) -> np.ndarray:
        cnt = C.c_int64()
        check(_lib().ppf_plan_halo_count(self.h, peer, C.byref(cnt)))
        out = np.empty(cnt.value, dtype=np.int64)
        check(_lib().ppf_plan_halo_recv(self.h, peer, _ptr(out, C.c_int64)))
        return out

    def set_halo_send(self, peer: int, local_rows):
        rows = np.ascontiguousarray(local_rows, dtype=np.int64)
        check(_lib().ppf_plan_set_halo_send(self.h, peer, len(rows), _ptr(rows, C.c_int64)))

    def close(self):
        if self.h:
            _lib().ppf_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Matrix:
    """ppf_mat_create: upload a plan into a caller-owned (torch) device buffer."""

    def __init__(self, ctx: Context, plan: Plan):
        torch = _torch()
        nbytes = plan.device_bytes()
        self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{ctx.device}")
        self.ctx = ctx
        self.dtype = plan.dtype
        self.info = plan.info()
        self.n_local = self.info["n_local"]
        h = C.c_void_p()
        check(_lib().ppf_mat_create(ctx.h, plan.h, C.c_void_p(self.buf.data_ptr()), nbytes,
                                    C.byref(h)))
        self.h = h

    def torch_dtype(self):
        torch = _torch()
        return torch.complex128 if self.dtype == L.C128 else torch.float64

    def spmv(self, x, y):
        """y = A x (device tensors of n_local entries)."""
        check(_lib().ppf_spmv(self.ctx.h, self.h, C.c_void_p(x.data_ptr()),
                              C.c_void_p(y.data_ptr())))

    def peer_window(self) -> bytes:
        """ppf_mat_peer_window: allocate this rank's peer-memory window; returns its
        PPF_PEER_DESC_BYTES descriptor for the caller to all-gather."""
        buf = C.create_string_buffer(L.PEER_DESC_BYTES)
        check(_lib().ppf_mat_peer_window(self.h, buf))
        return buf.raw

    def peer_connect(self, descs):
        """ppf_mat_peer_connect: `descs` = every rank's descriptor in rank order
        (None returns the matrix to NCCL / the host transport)."""
        if descs is None:
            check(_lib().ppf_mat_peer_connect(self.h, None))
            return
        blob = b"".join(bytes(d) for d in descs)
        assert all(len(d) == L.PEER_DESC_BYTES for d in descs)
        check(_lib().ppf_mat_peer_connect(self.h, C.create_string_buffer(blob, len(blob))))

    def set_split(self, sell_ks: int = 0) -> int:
        """ppf_mat_set_split: warps per SELL slice (0 = automatic); returns the value in force."""
        out = C.c_int()
        check(_lib().ppf_mat_set_split(self.h, int(sell_ks), C.byref(out)))
        return out.value

    def close(self):
        if self.h:
            _lib().ppf_mat_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Poly:
    """Host polynomial object (ppf_poly_*)."""

    def __init__(self, h):
        self.h = h

    @classmethod
    def chebyshev(cls, a: float, b: float, deg: int) -> "Poly":
        """P:323-335 with reading Q2 (Chebyshev interpolant, positivity certificate)."""
        h = C.c_void_p()
        check(_lib().ppf_poly_chebyshev(float(a), float(b), int(deg), C.byref(h)))
        return cls(h)

    @classmethod
    def ritz_newton(cls, ctx: Context, A: Matrix, start, deg: int, power: int = 1,
                    harmonic: bool = False, work=None) -> "Poly":
        """Ritz values of deg+1 device Arnoldi steps with A^power
        (power 2: the operator of func "invsqrt_sq" / "sign") from ``start``.
        ``work``: optional uint8 device tensor from ``ritz_workspace`` (allocated
        here otherwise)."""
        if work is None:
            work = cls.ritz_workspace(ctx, A, deg)
        h = C.c_void_p()
        check(_lib().ppf_poly_ritz_newton_pow(ctx.h, A.h, C.c_void_p(start.data_ptr()), deg,
                                              int(power), int(bool(harmonic)),
                                              C.c_void_p(work.data_ptr()), work.numel(), C.byref(h)))
        return cls(h)

    @staticmethod
    def ritz_workspace(ctx: Context, A: Matrix, deg: int):
        """ppf_ritz_workspace_bytes + the device scratch of the Ritz setup."""
        torch = _torch()
        nb = C.c_size_t()
        check(_lib().ppf_ritz_workspace_bytes(ctx.h, A.h, deg, C.byref(nb)))
        return torch.empty(max(nb.value, 256), dtype=torch.uint8, device=f"cuda:{ctx.device}")

    def set_newton_eval(self, mode: str) -> "Poly":
        """ppf_poly_set_newton_eval: "horner" (default), "basis" or "pairs"
        (real conjugate-pair form for real operators)."""
        check(_lib().ppf_poly_set_newton_eval(self.h, {"horner": 0, "basis": 1, "pairs": 2}[mode]))
        return self

    @classmethod
    def contour_ls(cls, points, deg: int) -> "Poly":
        """least-squares q on the contour points (complex array)."""
        z = np.ascontiguousarray(np.asarray(points, dtype=np.complex128))
        h = C.c_void_p()
        mr = C.c_double()
        check(_lib().ppf_poly_contour_ls(_ptr(z.view(np.float64), C.c_double), len(z), int(deg),
                                         C.byref(mr), C.byref(h)))
        p = cls(h)
        p.min_re = mr.value
        return p

    @classmethod
    def newton(cls, nodes, dd) -> "Poly":
        nodes = np.ascontiguousarray(nodes, dtype=np.complex128)
        dd = np.ascontiguousarray(dd, dtype=np.complex128)
        h = C.c_void_p()
        check(_lib().ppf_poly_import(L.POLY_NEWTON, len(nodes) - 1, None,
                                     dd.ctypes.data_as(C.c_void_p),
                                     nodes.ctypes.data_as(C.c_void_p), C.byref(h)))
        return cls(h)

    @classmethod
    def chebyshev_coeffs(cls, a: float, b: float, c) -> "Poly":
        c = np.ascontiguousarray(c, dtype=np.float64)
        ab = np.array([a, b], dtype=np.float64)
        h = C.c_void_p()
        check(_lib().ppf_poly_import(L.POLY_CHEBYSHEV, len(c) - 1, _ptr(ab, C.c_double),
                                     c.ctypes.data_as(C.c_void_p), None, C.byref(h)))
        return cls(h)

    def export(self) -> dict:
        kind, deg = C.c_int(), C.c_int()
        check(_lib().ppf_poly_export(self.h, C.byref(kind), C.byref(deg), None, None, None))
        d = deg.value
        if kind.value == L.POLY_CHEBYSHEV:
            ab = np.empty(2)
            c = np.empty(d + 1)
            check(_lib().ppf_poly_export(self.h, None, None, _ptr(ab, C.c_double),
                                         c.ctypes.data_as(C.c_void_p), None))
            return {"kind": "chebyshev", "deg": d, "a": ab[0], "b": ab[1], "c": c}
        dd = np.empty(d + 1, dtype=np.complex128)
        nodes = np.empty(d + 1, dtype=np.complex128)
        check(_lib().ppf_poly_export(self.h, None, None, None, dd.ctypes.data_as(C.c_void_p),
                                     nodes.ctypes.data_as(C.c_void_p)))
        return {"kind": "newton", "deg": d, "nodes": nodes, "dd": dd}

    def eval(self, z) -> np.ndarray:
        z = np.ascontiguousarray(np.atleast_1d(z), dtype=np.complex128)
        out = np.empty_like(z)
        check(_lib().ppf_poly_eval(self.h, len(z), z.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
                                   out.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def certify(self, points=None) -> float:
        """ppf_poly_certify: min Re q over the
        points (real or complex array; None = the Chebyshev default grid of
        P:420).  Raises PPFError(PPF_EBRANCH) unless the minimum is > 0 (the
        minimum is then in the exception's ``min_re``)."""
        mr = C.c_double()
        if points is None:
            st = _lib().ppf_poly_certify(self.h, None, 0, L.R64, C.byref(mr))
        else:
            z = np.ascontiguousarray(np.atleast_1d(points))
            cplx = np.iscomplexobj(z)
            z = z.astype(np.complex128 if cplx else np.float64, copy=False)
            st = _lib().ppf_poly_certify(self.h, z.ctypes.data_as(C.c_void_p), len(z),
                                         L.C128 if cplx else L.R64, C.byref(mr))
        try:
            check(st)
        except L.PPFError as e:
            e.min_re = mr.value
            raise
        return mr.value

    def apply(self, ctx: Context, A: Matrix, x, y=None):
        """y = q(A) x: the fused SpMV chain (P:332 Clenshaw / P:354 Newton-Horner)."""
        torch = _torch()
        nb = C.c_size_t()
        check(_lib().ppf_poly_apply_bytes(ctx.h, A.h, C.byref(nb)))
        work = torch.empty(nb.value, dtype=torch.uint8, device=x.device)
        if y is None:
            y = torch.empty_like(x)
        check(_lib().ppf_poly_apply(ctx.h, A.h, self.h, C.c_void_p(x.data_ptr()),
                                    C.c_void_p(y.data_ptr()), C.c_void_p(work.data_ptr()),
                                    nb.value))
        # the chain runs on ctx.stream: keep the caching allocator from handing
        # out the scratch (and a freshly allocated y) before it has finished
        if ctx.stream != torch.cuda.current_stream(x.device):
            work.record_stream(ctx.stream)
            y.record_stream(ctx.stream)
        return y

    def close(self):
        if self.h:
            _lib().ppf_poly_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class RunReport:
    iterations: int
    term: str
    mvms: int
    inner_products: int
    est: float
    err: float
    beta0: float
    seconds_total: float
    seconds_host_dense: float
    kernel_launches: int
    seconds_device: float = float("nan")


_TERM = {L.CONVERGED: "converged", L.MAX_ITER: "max_iter", L.BREAKDOWN: "breakdown"}
_FUNC = {"invsqrt": L.INVSQRT, "sqrt": L.SQRT, "invsqrt_sq": L.INVSQRT_SQ, "sign": L.SIGN}
_KRY = {"lanczos": L.LANCZOS, "cgs2": L.ARNOLDI_CGS2, "lanczos2p": L.LANCZOS_2PASS}
_PREC = {"left": L.PREC_LEFT, "right": L.PREC_RIGHT}
_STOP = {"fixed": L.STOP_FIXED_M, "est": L.STOP_EST, "true": L.STOP_TRUE_ERR}


def make_opts(func="invsqrt", krylov="cgs2", m_max=60, stop="fixed", tol=1e-8, check_every=1,
              x_ref=None, breakdown_rtol=0.0, record_history=True, precond="left") -> L.Opts:
    o = L.Opts()
    o.func = _FUNC[func]
    o.krylov = _KRY[krylov]
    o.m_max = int(m_max)
    o.stop = _STOP[stop]
    o.tol = float(tol)
    o.check_every = int(check_every)
    o.x_ref = C.c_void_p(x_ref.data_ptr()) if x_ref is not None else None
    o.breakdown_rtol = float(breakdown_rtol)
    o.record_history = int(bool(record_history))
    o.precond = _PREC[precond]
    return o


class Workspace:
    """Caller-owned device scratch for ppf_run (sized by ppf_workspace_bytes)."""

    def __init__(self, ctx: Context, A: Matrix, q: Poly, opts: L.Opts):
        torch = _torch()
        nb = C.c_size_t()
        check(_lib().ppf_workspace_bytes(ctx.h, A.h, _qh(q), C.byref(opts), C.byref(nb)))
        self.nbytes = nb.value
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=f"cuda:{ctx.device}")


def _qh(q):
    """ppf_poly handle, or NULL for the plain (unpreconditioned, d = 1) method."""
    return None if q is None else q.h


def _report(r: L.Report) -> RunReport:
    return RunReport(r.iterations, _TERM.get(r.term, str(r.term)), r.mvms, r.inner_products, r.est,
                     r.err, r.beta0, r.seconds_total, r.seconds_host_dense, r.kernel_launches,
                     r.seconds_device)


def run(ctx: Context, A: Matrix, q: Poly, b, x=None, work: Workspace | None = None, **opt_kw):
    """ppf_run: Algorithm 1 + f(H_m) + x = V_m y_m; b, x device tensors."""
    torch = _torch()
    opts = make_opts(**opt_kw)
    if work is None:
        work = Workspace(ctx, A, q, opts)
    if x is None:
        x = torch.empty_like(b)
    rep = L.Report()
    check(_lib().ppf_run(ctx.h, A.h, _qh(q), C.byref(opts), C.c_void_p(b.data_ptr()),
                         C.c_void_p(x.data_ptr()), C.c_void_p(work.buf.data_ptr()), work.nbytes,
                         C.byref(rep)))
    return x, _report(rep)


def run_host(ctx: Context, A: Matrix, q: Poly, b_host, x_host, work: Workspace | None = None,
             **opt_kw):
    """ppf_run_host: the same with host (ideally pinned) buffers; x_host filled on return."""
    opts = make_opts(**opt_kw)
    if work is None:
        work = Workspace(ctx, A, q, opts)
    rep = L.Report()
    check(_lib().ppf_run_host(ctx.h, A.h, _qh(q), C.byref(opts), C.c_void_p(b_host.data_ptr()),
                              C.c_void_p(x_host.data_ptr()), C.c_void_p(work.buf.data_ptr()),
                              work.nbytes, C.byref(rep)))
    return x_host, _report(rep)


def history(ctx: Context):
    cnt = C.c_int()
    check(_lib().ppf_history(ctx.h, 0, C.byref(cnt), None, None, None, None))
    n = cnt.value
    m = (C.c_int * max(n, 1))()
    est = np.empty(max(n, 1))
    err = np.empty(max(n, 1))
    mv = (C.c_longlong * max(n, 1))()
    check(_lib().ppf_history(ctx.h, n, C.byref(cnt), m, _ptr(est, C.c_double), _ptr(err, C.c_double),
                             mv))
    return [{"m": m[i], "est": float(est[i]), "err": float(err[i]), "mvms": mv[i]} for i in range(n)]


def hessenberg(ctx: Context, complex_: bool):
    m = C.c_int()
    beta0 = C.c_double()
    check(_lib().ppf_hessenberg(ctx.h, 0, None, C.byref(m), C.byref(beta0)))
    mm = m.value
    H = np.zeros((mm, mm + 1), dtype=np.complex128 if complex_ else np.float64)  # column-major
    check(_lib().ppf_hessenberg(ctx.h, mm + 1, H.ctypes.data_as(C.c_void_p), None, None))
    return H.T.copy(), beta0.value


def dense_invsqrt_e1(H: np.ndarray, beta0: float, hermitian: bool) -> np.ndarray:
    """ppf_dense_invsqrt_e1 (host K10), for tests."""
    m = H.shape[0]
    cplx = np.iscomplexobj(H)
    Hf = np.asfortranarray(H, dtype=np.complex128 if cplx else np.float64)
    y = np.empty(m, dtype=Hf.dtype)
    check(_lib().ppf_dense_invsqrt_e1(L.C128 if cplx else L.R64, m, Hf.ctypes.data_as(C.c_void_p),
                                      m, float(beta0), int(hermitian), y.ctypes.data_as(C.c_void_p)))
    return y


def profile_enable(ctx: Context, on: bool = True):
    """ppf_profile_enable: event-time every hot-path kernel launch (resets counters)."""
    check(_lib().ppf_profile_enable(ctx.h, int(bool(on))))


def profile_read(ctx: Context) -> dict:
    """ppf_profile_read for the three kernel classes."""
    out = {}
    for cls, name in ((0, "spmv"), (1, "ortho"), (2, "other")):
        n = C.c_longlong()
        ms = C.c_double()
        by = C.c_double()
        check(_lib().ppf_profile_read(ctx.h, cls, C.byref(n), C.byref(ms), C.byref(by)))
        out[name] = {"launches": n.value, "ms": ms.value, "bytes": by.value}
    return out


class _CudaBuf:
    """Exposes a raw device pointer to torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, n: int, complex_: bool):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": "<c16" if complex_ else "<f8",
            "data": (ptr, False), "version": 2, "strides": None}


def halo_pack(ctx: Context, A: Matrix, x):
    """ppf_halo_pack: gather this rank's boundary entries of x into the send buffer."""
    check(_lib().ppf_halo_pack(ctx.h, A.h, C.c_void_p(x.data_ptr())))


def halo_buffers(A: Matrix, send_total: int, recv_total: int):
    """ppf_halo_buffers as torch views (no copy) of the device send / recv buffers."""
    torch = _torch()
    s, r = C.c_void_p(), C.c_void_p()
    check(_lib().ppf_halo_buffers(A.h, C.byref(s), C.byref(r)))
    cplx = A.dtype == L.C128
    dev = torch.device(f"cuda:{A.ctx.device}")
    sb = torch.as_tensor(_CudaBuf(s.value or 0, send_total, cplx), device=dev) if send_total else None
    rb = torch.as_tensor(_CudaBuf(r.value or 0, recv_total, cplx), device=dev) if recv_total else None
    return sb, rb


def spmv_local(ctx: Context, A: Matrix, x, y):
    """ppf_spmv_local: y = A x from local x and the current receive buffer."""
    check(_lib().ppf_spmv_local(ctx.h, A.h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr())))
