"""Shared helpers for the parity tests: run the CUDA path through the C ABI
and compare it with the oracle using the north-star tolerances
(BASELINE.json north_star):
  * primal/dual residuals and gap <= 1e-5 relative, evaluated in f64 from the
    f32 outputs (the relative form of reading Q4);
  * x within 1e-4 relative of the f64 oracle;
  * gradients within 1e-3 relative of the f64 oracle, per field:
    ||g - g_ref||_2 / max(||g_ref||_2, 1e-2 ||bundle_ref||_2), where the
    bundle is all six fields of that problem (a field below 1% of the bundle —
    e.g. grad_q of a 1-D QP pinned by an active constraint, ~kappa_relax in
    size — is measured against 1% of the bundle: its f32 value is computed
    through a cancellation of O(1) terms);
  * iteration counts equal to the f32 oracle (M-form) or within +-1."""
from __future__ import annotations

import numpy as np

GRADS = ("dQ", "dq", "dA", "db", "dG", "dh")
FIELDS = ("Q", "q", "A", "b", "G", "h")

TOL_RES = 1e-5
TOL_X = 1e-4
TOL_GRAD = 1e-3


def run_gpu(batch, mem="device", need_backward=True, dl=None, formulation="implicit", **cfg):
    import torch
    from paper_2605_17913_b200.solver import QPSolver
    shared = [k for k, v in batch.shared.items() if v]
    S = QPSolver(batch.batch, batch.n, batch.m, batch.p, shared=shared, mem=mem, formulation=formulation, **cfg)
    dev = "cuda:0"

    def T(name):
        a = getattr(batch, name)
        a = a[0] if name in shared else a
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
        return t.to(dev) if mem == "device" else t.pin_memory()

    data = [T(f) for f in FIELDS]
    out = S.solve(*data)
    res = {k: v.cpu().numpy() if hasattr(v, "cpu") else v for k, v in out.items()}
    if need_backward:
        d = torch.from_numpy(np.ascontiguousarray(batch.dl_dx if dl is None else dl, dtype=np.float32))
        d = d.to(dev) if mem == "device" else d.pin_memory()
        g = S.backward(d)
        torch.cuda.synchronize()
        res.update({k: v.cpu().numpy() for k, v in g.items()})
        res["grad_status"] = res.pop("status") if "status" in g else None
        res["status"] = out["status"].cpu().numpy()
    torch.cuda.synchronize()
    res["info"] = S.info()
    S.close()
    return res


def rel_residuals(batch, x, y, z, s):
    """f64 relative KKT residuals of f32 outputs (Eq. 4; scales of reading Q4)."""
    out = []
    for i in range(batch.batch):
        P = {k: v.astype(np.float64) for k, v in batch.problem(i).items()}
        xi, yi, zi, si = (t[i].astype(np.float64) for t in (x, y, z, s))
        Qx, Gz, Ay = P["Q"] @ xi, P["G"].T @ zi, P["A"].T @ yi
        rt = Qx + P["q"] + Gz + Ay
        st = max(1.0, *(np.abs(t).max(initial=0) for t in (Qx, P["q"], Gz, Ay)))
        Ax, Gx = P["A"] @ xi, P["G"] @ xi
        re = Ax - P["b"]
        se = max(1.0, np.abs(Ax).max(initial=0), np.abs(P["b"]).max(initial=0))
        ri = Gx + si - P["h"]
        si_ = max(1.0, np.abs(Gx).max(initial=0), np.abs(si).max(initial=0), np.abs(P["h"]).max(initial=0))
        obj = 0.5 * xi @ Qx + P["q"] @ xi
        gap = si @ zi
        out.append((np.abs(rt).max(initial=0) / st, np.abs(re).max(initial=0) / se,
                    np.abs(ri).max(initial=0) / si_, gap / max(1.0, abs(obj))))
    return np.array(out)


def rel_err_rows(a, r, floor=None):
    a = a.reshape(a.shape[0], -1).astype(np.float64)
    r = r.reshape(r.shape[0], -1).astype(np.float64)
    num = np.linalg.norm(a - r, axis=1)
    den = np.linalg.norm(r, axis=1)
    if floor is not None:
        den = np.maximum(den, floor)
    return np.where(den > 0, num / np.maximum(den, 1e-300), num)


def bundle_norm(grads, idx=None):
    """Per-problem 2-norm of the whole gradient bundle (per-problem fields only)."""
    tot = None
    for k in GRADS:
        g = grads[k]
        if g.ndim < 2 or g.size == 0:
            continue
        v = (g.reshape(g.shape[0], -1).astype(np.float64) ** 2).sum(1)
        tot = v if tot is None else tot + v
    out = np.sqrt(tot)
    return out if idx is None else out[idx]


def x_rel(a, r):
    return np.abs(a - r).max(axis=1) / np.maximum(1.0, np.abs(r).max(axis=1))


def shared_sum(batch, grads):
    """Batch-sum per-problem oracle gradients for the fields the batch shares."""
    out = {}
    for g, f in zip(GRADS, FIELDS):
        out[g] = grads[g].sum(axis=0) if batch.shared.get(f, False) else grads[g]
    return out
