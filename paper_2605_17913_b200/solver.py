"""PyTorch-facing wrapper of the C ABI: tensors in, tensors out.

PyTorch supplies device memory and the stream; the work runs in
``libqpb200.so``.  ``QPSolver`` owns one ``qp_ctx``; ``QPFunction`` is the
autograd layer (forward = Alg. 1, backward = Alg. 2 + Alg. 3)."""
from __future__ import annotations

import numpy as np
import torch

from . import capi

FIELDS = ("Q", "q", "A", "b", "G", "h")
GRADS = ("dQ", "dq", "dA", "db", "dG", "dh")


def _per(name, n, m, p):
    return {"Q": (n, n), "q": (n,), "A": (m, n), "b": (m,), "G": (p, n), "h": (p,)}[name]


class QPSolver:
    """Batched solver for B QPs of fixed (n, m, p).

    ``shared``: names of data fields given WITHOUT a batch dimension (stride 0
    in the C ABI); their gradients come back batch-summed."""

    def __init__(self, batch: int, n: int, m: int, p: int, shared=(), device: int = 0,
                 mem: str = "device", formulation: str = "implicit", **cfg):
        self.B, self.n, self.m, self.p = batch, n, m, p
        self.shared = frozenset(shared)
        self.device = device
        self.mem = mem
        strides = {}
        for f in FIELDS:
            strides[f] = 0 if f in self.shared else int(np.prod(_per(f, n, m, p)))
        self.dims = capi.QpDims(batch, n, m, p, *[strides[f] for f in FIELDS])
        c = capi.default_config()
        for k, v in cfg.items():
            setattr(c, k, v)
        c.formulation = capi.QP_EXPLICIT if formulation == "explicit" else capi.QP_IMPLICIT
        # "host": host buffers, each call returns with its results in host memory;
        # "host_async": host buffers, the caller synchronises the device (copies
        # and kernels of consecutive calls overlap)
        c.mem_kind = {"device": capi.QP_MEM_DEVICE, "host": capi.QP_MEM_HOST,
                      "host_async": capi.QP_MEM_HOST_ASYNC}[mem]
        self.cfg = c
        self._saved = None
        self.generation = 0  # number of solve calls; the C ctx differentiates the LAST one
        if batch == 0:  # empty batch: nothing to solve, no ctx (the C ABI takes B >= 1)
            self.h = None
            return
        stream = torch.cuda.current_stream(device).cuda_stream if mem == "device" else None
        self.h = capi.qp_create(self.dims, c, device, stream)

    def info(self) -> dict:
        if self.h is None:
            return {}
        i = capi.qp_get_info(self.h)
        return {k: getattr(i, k) for k, _ in i._fields_}

    def last_flops(self):
        """(solve, backward) algorithmic flops of the last calls."""
        if self.h is None:
            return (0.0, 0.0)
        return capi.qp_last_flops(self.h)

    def close(self):
        h, self.h = getattr(self, "h", None), None
        if h and capi is not None and getattr(capi, "qp_destroy", None) is not None:  # not at interpreter exit
            capi.qp_destroy(h)

    __del__ = close

    # -- helpers ---------------------------------------------------------------
    def _shape(self, f):
        per = _per(f, self.n, self.m, self.p)
        return per if f in self.shared else (self.B, *per)

    def _check(self, f, t):
        exp = self._shape(f)
        if tuple(t.shape) != tuple(exp):
            raise ValueError(f"{f}: expected shape {exp}, got {tuple(t.shape)}")
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError(f"{f}: need contiguous float32")
        if self.mem == "device" and (not t.is_cuda or t.device.index != self.device):
            raise ValueError(f"{f}: must live on cuda:{self.device}")
        if self.mem != "device" and t.is_cuda:
            raise ValueError(f"{f}: host mode takes CPU tensors")

    def _alloc(self, shape, dtype=torch.float32):
        if self.B == 0:  # empty outputs; shared-field gradients are sums over no problems
            dev = f"cuda:{self.device}" if self.mem == "device" else "cpu"
            return torch.zeros(shape, dtype=dtype, device=dev)
        if self.mem == "device":
            return torch.empty(shape, dtype=dtype, device=f"cuda:{self.device}")
        return torch.empty(shape, dtype=dtype, pin_memory=True)  # no staging copy

    @staticmethod
    def _ptr(t):
        return t.data_ptr() if (t is not None and t.numel() > 0) else None

    # -- API -----------------------------------------------------------------
    def solve(self, Q, q, A, b, G, h, out=None):
        data = dict(Q=Q, q=q, A=A, b=b, G=G, h=h)
        for f, t in data.items():
            self._check(f, t)
        if self.mem == "device" and self.h is not None:
            capi.qp_set_stream(self.h, torch.cuda.current_stream(self.device).cuda_stream)
        B, n, m, p = self.B, self.n, self.m, self.p
        if out is None:
            out = dict(x=self._alloc((B, n)), s=self._alloc((B, p)), z=self._alloc((B, p)), y=self._alloc((B, m)),
                       iters=self._alloc((B,), torch.int32), status=self._alloc((B,), torch.int32))
        P = self._ptr
        if self.B == 0:
            self._saved = (data, out)
            self.generation += 1
            return out
        capi.qp_solve_batched(self.h, *[P(data[f]) for f in FIELDS], P(out["x"]), P(out["s"]), P(out["z"]),
                              P(out["y"]), P(out["iters"]), P(out["status"]))
        self._saved = (data, out)  # keep alive for backward (C-ABI contract)
        self.generation += 1
        return out

    def backward(self, dl_dx, out=None, need=GRADS):
        self._check_dl(dl_dx)
        if self.mem == "device" and self.h is not None:
            capi.qp_set_stream(self.h, torch.cuda.current_stream(self.device).cuda_stream)
        if out is None:
            out = {}
            for g, f in zip(GRADS, FIELDS):
                if g in need:
                    out[g] = self._alloc(self._shape(f))
            out["relax_iters"] = self._alloc((self.B,), torch.int32)
            out["status"] = self._alloc((self.B,), torch.int32)
        P = self._ptr
        if self.B == 0:
            if self._saved is None:
                raise RuntimeError("QP_ERR_NOT_SOLVED: backward before solve")
            return out
        capi.qp_backward_batched(self.h, P(dl_dx), *[P(out.get(g)) for g in GRADS], P(out["relax_iters"]),
                                 P(out["status"]))
        return out

    def _check_dl(self, t):
        if tuple(t.shape) != (self.B, self.n) or t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError("dl_dx must be contiguous float32 [B, n]")


class QPFunction(torch.autograd.Function):
    """x* = QPFunction.apply(solver, Q, q, A, b, G, h); backward = Alg. 2 + 3."""

    @staticmethod
    def forward(ctx, solver: QPSolver, Q, q, A, b, G, h):
        data = [t.contiguous() for t in (Q, q, A, b, G, h)]
        out = solver.solve(*data)
        ctx.solver = solver
        ctx.generation = solver.generation
        ctx.save_for_backward(*data)
        return out["x"]

    @staticmethod
    def backward(ctx, gx):
        solver = ctx.solver
        if solver.generation != ctx.generation:
            # the solver was applied again since this forward (a layer used
            # twice, an evaluation solve in between): the C ctx holds the later
            # solve, so solve this graph's problems again (deterministic: the
            # same x*) before differentiating
            solver.solve(*ctx.saved_tensors)
        g = solver.backward(gx.contiguous())
        return (None, g["dQ"], g["dq"], g["dA"], g["db"], g["dG"], g["dh"])


def solve(Q, q, A, b, G, h, shared=(), **cfg):
    """One-shot convenience: returns dict(x, s, z, y, iters, status)."""
    B = q.shape[0] if "q" not in shared else Q.shape[0]
    n = q.shape[-1]
    m = b.shape[-1]
    p = h.shape[-1]
    s = QPSolver(B, n, m, p, shared=shared, device=q.device.index or 0, **cfg)
    return s.solve(Q, q, A, b, G, h)
