"""ctypes binding of the C ABI in include/qpb200.h — argument marshalling only.

Every step of the hot path runs inside ``libqpb200.so`` (sm_100a kernels).
If the library is missing or no CUDA device is present the calls raise; there
is no CPU fallback.  The function names mirror the C ABI."""
from __future__ import annotations

import ctypes as C
import os

from ._build import LIB

QP_OK = 0
ERRORS = {0: "ok", -1: "invalid argument", -2: "unsupported shape", -3: "pointer not 4-byte aligned",
          -4: "CUDA error", -5: "out of device memory", -6: "backward called before solve",
          -7: "unsupported option"}
QP_CONVERGED, QP_MAX_ITER, QP_NUMERICAL_FAILURE = 0, 2, 3
QP_IMPLICIT, QP_EXPLICIT = 0, 1
QP_MEM_DEVICE, QP_MEM_HOST, QP_MEM_HOST_ASYNC = 0, 1, 2
QP_RELAX_NEWTON, QP_RELAX_CHORD = 0, 2


class QpDims(C.Structure):
    _fields_ = [("batch", C.c_int32), ("n", C.c_int32), ("m_eq", C.c_int32), ("p", C.c_int32),
                ("bstride_Q", C.c_int64), ("bstride_q", C.c_int64), ("bstride_A", C.c_int64),
                ("bstride_b", C.c_int64), ("bstride_G", C.c_int64), ("bstride_h", C.c_int64)]


class QpConfig(C.Structure):
    _fields_ = [("tol", C.c_float), ("max_iter", C.c_int32), ("sigma", C.c_float), ("tau", C.c_float),
                ("kappa_relax", C.c_float), ("relax_ktol", C.c_float), ("relax_max_iter", C.c_int32),
                ("formulation", C.c_int32), ("pivot_floor_rel", C.c_float), ("mem_kind", C.c_int32),
                ("relax_tol", C.c_float), ("relax_mode", C.c_int32), ("chord_max", C.c_int32),
                ("chord_rho", C.c_float)]


class QpInfo(C.Structure):
    _fields_ = [("path", C.c_int32), ("threads", C.c_int32), ("smem_bytes", C.c_int32),
                ("ctas_per_sm", C.c_int32), ("kkt_dim", C.c_int32), ("launches_solve", C.c_int32),
                ("launches_backward", C.c_int32), ("workspace_bytes", C.c_int64),
                ("partition_cap", C.c_int32), ("handed_solve", C.c_int32), ("handed_backward", C.c_int32),
                ("relax_mode", C.c_int32), ("chord_steps", C.c_int32)]


EXPORTS = ("qp_config_default", "qp_create", "qp_set_stream", "qp_get_info", "qp_max_kkt_dim",
           "qp_solve_batched", "qp_backward_batched", "qp_last_flops", "qp_destroy", "qp_error_string",
           "qp_debug_tc_syrk", "qp_debug_check_guards")

_lib = None


class QPError(RuntimeError):
    pass


def load(path: str | None = None):
    """Load libqpb200.so (raises if it was not built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("QPB200_LIB") or LIB  # QPB200_LIB: experiment with an alternate build
    if not os.path.exists(p):
        raise QPError(f"CUDA library {p} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(p)
    V = C.c_void_p
    L.qp_config_default.argtypes = [C.POINTER(QpConfig)]
    L.qp_create.argtypes = [C.POINTER(V), C.POINTER(QpDims), C.POINTER(QpConfig), C.c_int, V]
    L.qp_set_stream.argtypes = [V, V]
    L.qp_get_info.argtypes = [V, C.POINTER(QpInfo)]
    L.qp_max_kkt_dim.argtypes = [C.c_int32]
    L.qp_max_kkt_dim.restype = C.c_int32
    L.qp_solve_batched.argtypes = [V] * 13
    L.qp_backward_batched.argtypes = [V] * 10
    L.qp_destroy.argtypes = [V]
    L.qp_last_flops.argtypes = [V, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.qp_debug_tc_syrk.argtypes = [V, V, V, C.c_int32, C.c_int32, V, V]
    L.qp_debug_tc_syrk.restype = C.c_int
    L.qp_debug_check_guards.argtypes = [V, C.POINTER(C.c_int64)]
    L.qp_debug_check_guards.restype = C.c_int
    L.qp_error_string.argtypes = [C.c_int]
    L.qp_error_string.restype = C.c_char_p
    for f in ("qp_config_default", "qp_create", "qp_set_stream", "qp_get_info", "qp_solve_batched",
              "qp_backward_batched", "qp_destroy", "qp_last_flops"):
        getattr(L, f).restype = C.c_int
    if path is None:
        _lib = L
    return L


def check(rc: int, what: str):
    if rc != QP_OK:
        raise QPError(f"{what} failed: {ERRORS.get(rc, rc)} ({rc})")


def default_config() -> QpConfig:
    c = QpConfig()
    check(load().qp_config_default(C.byref(c)), "qp_config_default")
    return c


def qp_create(dims: QpDims, cfg: QpConfig, device: int, stream: int | None):
    h = C.c_void_p()
    check(load().qp_create(C.byref(h), C.byref(dims), C.byref(cfg), device, C.c_void_p(stream or 0)), "qp_create")
    return h


def qp_set_stream(h, stream: int | None):
    check(load().qp_set_stream(h, C.c_void_p(stream or 0)), "qp_set_stream")


def qp_get_info(h) -> QpInfo:
    info = QpInfo()
    check(load().qp_get_info(h, C.byref(info)), "qp_get_info")
    return info


def qp_solve_batched(h, Q, q, A, b, G, h_, x, s, z, y, iters, status):
    args = [C.c_void_p(v or 0) for v in (Q, q, A, b, G, h_, x, s, z, y, iters, status)]
    check(load().qp_solve_batched(h, *args), "qp_solve_batched")


def qp_backward_batched(h, dl_dx, dQ, dq, dA, db, dG, dh, relax_iters, status):
    args = [C.c_void_p(v or 0) for v in (dl_dx, dQ, dq, dA, db, dG, dh, relax_iters, status)]
    check(load().qp_backward_batched(h, *args), "qp_backward_batched")


def qp_last_flops(h):
    a, b = C.c_double(), C.c_double()
    check(load().qp_last_flops(h, C.byref(a), C.byref(b)), "qp_last_flops")
    return a.value, b.value


def qp_debug_tc_syrk(G, om, Q, n, p, H, stream=None):
    check(load().qp_debug_tc_syrk(C.c_void_p(G), C.c_void_p(om), C.c_void_p(Q), n, p, C.c_void_p(H),
                                  C.c_void_p(stream or 0)), "qp_debug_tc_syrk")


def qp_destroy(h):
    load().qp_destroy(h)


def qp_debug_check_guards(h) -> int:
    """Guard words overwritten in the ctx workspaces (QPB200_GUARD mode)."""
    n = C.c_int64()
    check(load().qp_debug_check_guards(h, C.byref(n)), "qp_debug_check_guards")
    return n.value
