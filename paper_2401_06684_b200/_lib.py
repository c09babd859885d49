"""ctypes declarations of the C ABI in include/ppf.h (argument marshalling only).

Loading fails loudly if the in-tree ``libppf.so`` is missing: there is no CPU
fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libppf.so")

PPF_OK = 0
PEER_DESC_BYTES = 2048   # include/ppf.h PPF_PEER_DESC_BYTES
STATUS = {0: "PPF_OK", 1: "PPF_EINVAL", 2: "PPF_ECUDA", 3: "PPF_ENCCL", 4: "PPF_EWORKSPACE",
          5: "PPF_EBRANCH", 6: "PPF_EDENSE", 7: "PPF_ESTATE"}
R64, C128 = 0, 1
INVSQRT, SQRT, INVSQRT_SQ, SIGN = 0, 1, 2, 3
LANCZOS, ARNOLDI_CGS2, LANCZOS_2PASS = 0, 1, 2
PREC_LEFT, PREC_RIGHT = 0, 1
STOP_FIXED_M, STOP_EST, STOP_TRUE_ERR = 0, 1, 2
CONVERGED, MAX_ITER, BREAKDOWN = 0, 1, 2
POLY_CHEBYSHEV, POLY_NEWTON = 0, 1
FMT_SELL, FMT_CSR = 0, 1

vp = C.c_void_p
i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)


class Opts(C.Structure):
    _fields_ = [("func", C.c_int), ("krylov", C.c_int), ("m_max", C.c_int), ("stop", C.c_int),
                ("tol", C.c_double), ("check_every", C.c_int), ("x_ref", vp),
                ("breakdown_rtol", C.c_double), ("record_history", C.c_int),
                ("precond", C.c_int)]


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                          C.POINTER(C.c_double), C.POINTER(C.c_int64))
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)


class Transport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("exchange", EXCHANGE_FN), ("allreduce_sum", ALLREDUCE_FN)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("term", C.c_int), ("mvms", C.c_longlong),
                ("inner_products", C.c_longlong), ("est", C.c_double), ("err", C.c_double),
                ("beta0", C.c_double), ("seconds_total", C.c_double),
                ("seconds_host_dense", C.c_double), ("kernel_launches", C.c_longlong),
                ("seconds_device", C.c_double)]


# name -> (restype, argtypes)
SIGNATURES = {
    "ppf_status_string": (C.c_char_p, [C.c_int]),
    "ppf_last_error": (C.c_char_p, []),
    "ppf_abi_version": (C.c_int, []),
    "ppf_nccl_unique_id": (C.c_int, [vp]),
    "ppf_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
    "ppf_ctx_destroy": (None, [vp]),
    "ppf_plan_create": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_int, i64p, i64p, i64p, vp,
                                  C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "ppf_plan_device_bytes": (C.c_int, [vp, C.POINTER(C.c_size_t)]),
    "ppf_plan_info": (C.c_int, [vp, i64p, i64p, i64p, i64p]),
    "ppf_plan_halo_count": (C.c_int, [vp, C.c_int, i64p]),
    "ppf_plan_index_bits": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "ppf_plan_encoding": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ppf_plan_slice_schedule": (C.c_int, [vp, C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_int64)]),
    "ppf_plan_set_encoding": (C.c_int, [vp, C.c_int]),
    "ppf_plan_halo_recv": (C.c_int, [vp, C.c_int, i64p]),
    "ppf_plan_set_halo_send": (C.c_int, [vp, C.c_int, C.c_int64, i64p]),
    "ppf_plan_destroy": (None, [vp]),
    "ppf_mat_create": (C.c_int, [vp, vp, vp, C.c_size_t, C.POINTER(vp)]),
    "ppf_spmv": (C.c_int, [vp, vp, vp, vp]),
    "ppf_mat_set_split": (C.c_int, [vp, C.c_int, C.POINTER(C.c_int)]),
    "ppf_ctx_set_transport": (C.c_int, [vp, C.POINTER(Transport)]),
    "ppf_ctx_set_graphs": (C.c_int, [vp, C.c_int]),
    "ppf_mat_destroy": (None, [vp]),
    "ppf_halo_pack": (C.c_int, [vp, vp, vp]),
    "ppf_halo_buffers": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp)]),
    "ppf_spmv_local": (C.c_int, [vp, vp, vp, vp]),
    "ppf_poly_chebyshev": (C.c_int, [C.c_double, C.c_double, C.c_int, C.POINTER(vp)]),
    "ppf_ritz_workspace_bytes": (C.c_int, [vp, vp, C.c_int, C.POINTER(C.c_size_t)]),
    "ppf_poly_ritz_newton": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_size_t, C.POINTER(vp)]),
    "ppf_poly_set_newton_eval": (C.c_int, [vp, C.c_int]),
    "ppf_contour_from_ritz": (C.c_int, [vp, C.c_int, C.c_double, C.c_double, C.c_int, vp,
                                        C.POINTER(C.c_int)]),
    "ppf_poly_contour_ls": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(vp)]),
    "ppf_poly_ritz_newton_pow": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, C.c_size_t,
                                           C.POINTER(vp)]),
    "ppf_poly_import": (C.c_int, [C.c_int, C.c_int, dblp, vp, vp, C.POINTER(vp)]),
    "ppf_poly_export": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), dblp, vp, vp]),
    "ppf_poly_eval": (C.c_int, [vp, C.c_int, dblp, dblp]),
    "ppf_poly_certify": (C.c_int, [vp, vp, C.c_int, C.c_int, dblp]),
    "ppf_poly_destroy": (None, [vp]),
    "ppf_poly_apply_bytes": (C.c_int, [vp, vp, C.POINTER(C.c_size_t)]),
    "ppf_poly_apply": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_size_t]),
    "ppf_workspace_bytes": (C.c_int, [vp, vp, vp, C.POINTER(Opts), C.POINTER(C.c_size_t)]),
    "ppf_run": (C.c_int, [vp, vp, vp, C.POINTER(Opts), vp, vp, vp, C.c_size_t, C.POINTER(Report)]),
    "ppf_run_host": (C.c_int, [vp, vp, vp, C.POINTER(Opts), vp, vp, vp, C.c_size_t,
                               C.POINTER(Report)]),
    "ppf_history": (C.c_int, [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), dblp, dblp,
                              C.POINTER(C.c_longlong)]),
    "ppf_hessenberg": (C.c_int, [vp, C.c_int, vp, C.POINTER(C.c_int), dblp]),
    "ppf_profile_enable": (C.c_int, [vp, C.c_int]),
    "ppf_mat_peer_window": (C.c_int, [vp, vp]),
    "ppf_mat_peer_connect": (C.c_int, [vp, vp]),
    "ppf_profile_read": (C.c_int, [vp, C.c_int, C.POINTER(C.c_longlong), dblp, dblp]),
    "ppf_dense_invsqrt_e1": (C.c_int, [C.c_int, C.c_int, vp, C.c_int, C.c_double, C.c_int, vp]),
}


class PPFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load():
    """Load the in-tree libppf.so (built by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != PPF_OK:
        msg = load().ppf_last_error().decode(errors="replace")
        raise PPFError(status, msg)
