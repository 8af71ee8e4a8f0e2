"""CPU oracle — TEST INFRASTRUCTURE ONLY.

ctypes front-end of ``oracle/qp_oracle.cpp`` (a plain scalar-loop C++
implementation of Alg. 1/2/3 of arxiv 2605.17913 and of the standard
Mehrotra arm).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2605_17913_b200`` (the CUDA path);
both are fed by ``paper_2605_17913_b200.generators``, which holds no solver
arithmetic.

Parity status of every oracle function is listed in DESIGN.md §4 ("pins");
nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qp_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

SOLVER_K14_GEPP, SOLVER_M_LDL, SOLVER_NORMAL_CHOL, SOLVER_M_PART = 0, 1, 2, 3
FORM_IMPLICIT, FORM_EXPLICIT = 0, 1
ST_CONVERGED, ST_MAX_ITER, ST_NUMERICAL_FAILURE = 0, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle shared library with g++ (no BLAS, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", _SRC, "-o", _LIB]
        subprocess.run(cmd, check=True)
    return _LIB


class OracleCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int32), ("sigma", C.c_double),
                ("tau", C.c_double), ("kappa_relax", C.c_double), ("relax_ktol", C.c_double),
                ("relax_max_iter", C.c_int32), ("kkt_solver", C.c_int32),
                ("formulation", C.c_int32), ("pivot_floor_rel", C.c_double), ("relax_tol", C.c_double),
                ("partition_cap", C.c_int32), ("relax_mode", C.c_int32),
                ("chord_max", C.c_int32), ("chord_rho", C.c_double)]


@dataclass
class Cfg:
    """Solver settings (DESIGN.md §2 readings Q2-Q5, Q12, Q22)."""
    tol: float = 1e-5
    max_iter: int = 100
    sigma: float = 0.1
    tau: float = 0.99
    kappa_relax: float = 1e-4
    relax_ktol: float = 1e-4
    relax_max_iter: int = 50
    kkt_solver: int = SOLVER_M_PART
    formulation: int = FORM_IMPLICIT
    pivot_floor_rel: float = float(np.sqrt(np.finfo(np.float32).eps))
    relax_tol: float = 1e-6
    partition_cap: int = -1  # SOLVER_M_PART: reading Q12c (-1 = keep every v_i > 0)
    relax_mode: int = 0      # 0: Alg. 2 by exact Newton (Q6); 1: chord steps with Alg. 1's factor (N2(i)); 2: guarded chord (Q26)
    chord_max: int = 8       # relax_mode 2: most chord steps
    chord_rho: float = 0.5   # relax_mode 2: contraction a chord step must reach

    @staticmethod
    def f64(**kw) -> "Cfg":
        base = dict(tol=1e-10, relax_ktol=1e-10, relax_tol=1e-12, kkt_solver=SOLVER_K14_GEPP,
                    pivot_floor_rel=float(np.sqrt(np.finfo(np.float64).eps)))
        base.update(kw)
        return Cfg(**base)

    @staticmethod
    def f32(**kw) -> "Cfg":
        return Cfg(**kw)

    def c(self) -> OracleCfg:
        return OracleCfg(self.tol, self.max_iter, self.sigma, self.tau, self.kappa_relax,
                         self.relax_ktol, self.relax_max_iter, self.kkt_solver, self.formulation,
                         self.pivot_floor_rel, self.relax_tol, self.partition_cap, self.relax_mode,
                         self.chord_max, self.chord_rho)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            _lib = C.CDLL(_LIB)
            _declare(_lib)
    return _lib


def _declare(L):
    P = C.c_void_p
    ll = C.c_longlong
    for suf, ft in (("f64", C.c_double), ("f32", C.c_float)):
        f = getattr(L, f"oracle_solve_{suf}")
        f.argtypes = [C.POINTER(OracleCfg), C.c_int, C.c_int, C.c_int, C.c_int] + [P, ll] * 6 + [P] * 6 + [C.c_int]
        f.restype = C.c_int
        f = getattr(L, f"oracle_backward_{suf}")
        f.argtypes = ([C.POINTER(OracleCfg), C.c_int, C.c_int, C.c_int, C.c_int] + [P, ll] * 6 +
                      [P] * 5 + [P] * 6 + [P] * 4 + [P, P, C.c_int])
        f.restype = C.c_int
        f = getattr(L, f"oracle_retract_{suf}")
        f.argtypes = [C.c_int, P, ft, P, P, P, P, P]
        f.restype = None
        f = getattr(L, f"oracle_linesearch_{suf}")
        f.argtypes = [C.c_int, P, P, P, P, ft]
        f.restype = ft
        f = getattr(L, f"oracle_init_{suf}")
        f.argtypes = [C.c_int] * 3 + [P] * 10
        f.restype = C.c_int
        f = getattr(L, f"oracle_newton_step_{suf}")
        f.argtypes = [C.c_int] * 3 + [P] * 10 + [ft, C.c_int, ft, C.c_int] + [P] * 7
        f.restype = C.c_int
        f = getattr(L, f"oracle_ldl_{suf}")
        f.argtypes = [C.c_int, C.c_int, ft, P, P, P]
        f.restype = C.c_int
        f = getattr(L, f"oracle_residuals_{suf}")
        f.argtypes = [C.c_int] * 3 + [P] * 10 + [P] * 5
        f.restype = None
    L.oracle_hardware_threads.restype = C.c_int


def _dt(prec: str):
    return (np.float64, "f64") if prec == "f64" else (np.float32, "f32")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _prep(batch, name, dt):
    arr = np.ascontiguousarray(getattr(batch, name), dtype=dt)
    shared = batch.shared.get(name, False)
    per = int(np.prod(arr.shape[1:])) if arr.ndim > 1 else 1
    return arr, (0 if shared else per)


def hardware_threads() -> int:
    return int(lib().oracle_hardware_threads())


def solve(batch, cfg: Cfg, prec: str = "f64", nthreads: int | None = None):
    """Alg. 1 over a QPBatch.  Returns dict(x, y, z, s, iters, status)."""
    L = lib()
    dt, suf = _dt(prec)
    B, n, m, p = batch.batch, batch.n, batch.m, batch.p
    arrs = [_prep(batch, k, dt) for k in ("Q", "q", "A", "b", "G", "h")]
    x = np.zeros((B, n), dt); y = np.zeros((B, m), dt); z = np.zeros((B, p), dt); s = np.zeros((B, p), dt)
    it = np.zeros(B, np.int32); st = np.zeros(B, np.int32)
    c = cfg.c()
    args = []
    for a, stride in arrs:
        args += [_ptr(a), stride]
    nt = nthreads if nthreads is not None else max(1, os.cpu_count() or 1)
    getattr(L, f"oracle_solve_{suf}")(C.byref(c), B, n, m, p, *args, _ptr(x), _ptr(y), _ptr(z), _ptr(s),
                                      _ptr(it), _ptr(st), nt)
    return dict(x=x, y=y, z=z, s=s, iters=it, status=st)


def backward(batch, sol: dict, cfg: Cfg, prec: str = "f64", dl_dx=None, nthreads: int | None = None):
    """Alg. 2 + Alg. 3 from a solution.  Per-problem gradients (shared fields
    are NOT summed here) and the relaxed point."""
    L = lib()
    dt, suf = _dt(prec)
    B, n, m, p = batch.batch, batch.n, batch.m, batch.p
    arrs = [_prep(batch, k, dt) for k in ("Q", "q", "A", "b", "G", "h")]
    xs = [np.ascontiguousarray(sol[k], dtype=dt) for k in ("x", "y", "z", "s")]
    dl = np.ascontiguousarray(batch.dl_dx if dl_dx is None else dl_dx, dtype=dt)
    g = dict(dQ=np.zeros((B, n, n), dt), dq=np.zeros((B, n), dt), dA=np.zeros((B, m, n), dt),
             db=np.zeros((B, m), dt), dG=np.zeros((B, p, n), dt), dh=np.zeros((B, p), dt))
    rel = dict(x=np.zeros((B, n), dt), y=np.zeros((B, m), dt), z=np.zeros((B, p), dt), s=np.zeros((B, p), dt))
    it = np.zeros(B, np.int32); st = np.zeros(B, np.int32)
    c = cfg.c()
    args = []
    for a, stride in arrs:
        args += [_ptr(a), stride]
    nt = nthreads if nthreads is not None else max(1, os.cpu_count() or 1)
    getattr(L, f"oracle_backward_{suf}")(
        C.byref(c), B, n, m, p, *args, *[_ptr(a) for a in xs], _ptr(dl),
        *[_ptr(g[k]) for k in ("dQ", "dq", "dA", "db", "dG", "dh")],
        *[_ptr(rel[k]) for k in ("x", "y", "z", "s")], _ptr(it), _ptr(st), nt)
    return g | dict(relaxed=rel, relax_iters=it, status=st)


def retract(v, kappa, prec="f64"):
    L = lib()
    dt, suf = _dt(prec)
    v = np.ascontiguousarray(v, dtype=dt).ravel()
    out = [np.zeros_like(v) for _ in range(5)]
    getattr(L, f"oracle_retract_{suf}")(len(v), _ptr(v), dt(kappa), *[_ptr(o) for o in out])
    return dict(zip(("z", "s", "dp", "dm", "c"), out))


def linesearch(s, z, ds, dz, tau, prec="f64"):
    L = lib()
    dt, suf = _dt(prec)
    a = [np.ascontiguousarray(t, dtype=dt).ravel() for t in (s, z, ds, dz)]
    return float(getattr(L, f"oracle_linesearch_{suf}")(len(a[0]), *[_ptr(t) for t in a], dt(tau)))


def _one(prob, dt):
    return [np.ascontiguousarray(prob[k], dtype=dt) for k in ("Q", "q", "A", "b", "G", "h")]


def initialize(prob, n, m, p, prec="f64"):
    L = lib()
    dt, suf = _dt(prec)
    data = _one(prob, dt)
    x, y, z, s = np.zeros(n, dt), np.zeros(m, dt), np.zeros(p, dt), np.zeros(p, dt)
    rc = getattr(L, f"oracle_init_{suf}")(n, m, p, *[_ptr(a) for a in data], _ptr(x), _ptr(y), _ptr(z), _ptr(s))
    return dict(x=x, y=y, z=z, s=s, ok=(rc == 0))


def newton_step(prob, n, m, p, x, y, z, s, kappa_target, solver=SOLVER_K14_GEPP, floor_rel=1e-8, prec="f64",
                partition_cap=-1):
    L = lib()
    dt, suf = _dt(prec)
    data = _one(prob, dt)
    it = [np.ascontiguousarray(a, dtype=dt) for a in (x, y, z, s)]
    dx, dy, dz, ds, dv = np.zeros(n, dt), np.zeros(m, dt), np.zeros(p, dt), np.zeros(p, dt), np.zeros(p, dt)
    dk = np.zeros(1, dt); ka = np.zeros(1, dt)
    nf = getattr(L, f"oracle_newton_step_{suf}")(n, m, p, *[_ptr(a) for a in data], *[_ptr(a) for a in it],
                                                dt(kappa_target), solver, dt(floor_rel), partition_cap,
                                                *[_ptr(a) for a in (dx, dy, dz, ds, dv, dk, ka)])
    return dict(dx=dx, dy=dy, dz=dz, ds=ds, dv=dv, dk=float(dk[0]), kappa=float(ka[0]), nfloor=nf)


def residuals(prob, n, m, p, x, y, z, s, prec="f64"):
    L = lib()
    dt, suf = _dt(prec)
    data = _one(prob, dt)
    it = [np.ascontiguousarray(a, dtype=dt) for a in (x, y, z, s)]
    out = [np.zeros(n, dt), np.zeros(m, dt), np.zeros(p, dt), np.zeros(p, dt), np.zeros(p, dt)]
    getattr(L, f"oracle_residuals_{suf}")(n, m, p, *[_ptr(a) for a in data], *[_ptr(a) for a in it],
                                          *[_ptr(o) for o in out])
    return dict(zip(("rt", "re", "ri", "rz", "rs"), out))


def ldl(M, npos, floor_rel, rhs, prec="f64"):
    """Unpivoted signed LDLᵀ of M (first npos pivots positive, the rest
    negative; a pivot on the wrong side of ±θ, θ = floor_rel·max|diag|, is set
    to ±θ and counted — reading Q12) and the solve of M x = rhs with that
    factor.  Returns dict(L (unit lower), D, x, nfloor)."""
    L_ = lib()
    dt, suf = _dt(prec)
    M = np.array(M, dtype=dt, order="C")
    N = M.shape[0]
    D = np.zeros(N, dt)
    x = np.array(rhs, dtype=dt)
    nf = getattr(L_, f"oracle_ldl_{suf}")(N, npos, dt(floor_rel), _ptr(M), _ptr(D), _ptr(x))
    Lm = np.tril(M, -1) + np.eye(N, dtype=dt)
    return dict(L=Lm, D=D, x=x, nfloor=nf)
