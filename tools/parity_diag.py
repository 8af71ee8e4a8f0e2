"""Parity diagnostics (builder tool, GPU box): for each case print, per
gradient field, the UNFLOORED relative error ||g - g64|| / ||g64|| of the GPU
path and of the f32 oracle (M_PART, the same algorithm class) against the
f64 oracle, plus the f64-evaluated relative residuals and x errors.

usage: python tools/parity_diag.py [case ...]   (cases: cfg1 cfg2 cfg3 cfg4s)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle as O  # noqa: E402
from paper_2605_17913_b200 import generators as gen  # noqa: E402
from tests.helpers import GRADS, rel_residuals, run_gpu, x_rel  # noqa: E402

CASES = {"cfg1": lambda: gen.make_config(1), "cfg2": lambda: gen.make_config(2, batch=96),
         "cfg3": lambda: gen.make_config(3, batch=48),
         "cfg4s": lambda: gen.make_config(4, batch=16)}


def errs(g, ref, ok):
    out = {}
    for k in GRADS:
        a, r = g[k], ref[k]
        if r.size == 0 or a.shape != r.shape:
            continue
        a = a[ok].reshape(ok.sum(), -1).astype(np.float64)
        r = r[ok].reshape(ok.sum(), -1).astype(np.float64)
        num = np.linalg.norm(a - r, axis=1)
        den = np.linalg.norm(r, axis=1)
        e = num / np.maximum(den, 1e-300)
        out[k] = (e.max(), int(np.argmax(e)), den[np.argmax(e)])
    return out


def main(names):
    for name in names:
        b = CASES[name]()
        if any(b.shared.values()):  # per-problem gradients: every field replicated
            rep = {k: (np.repeat(getattr(b, k), b.batch, 0) if b.shared.get(k) else getattr(b, k))
                   for k in ("Q", "q", "A", "b", "G", "h")}
            b = gen.QPBatch(b.n, b.m, b.p, **rep, dl_dx=b.dl_dx, batch=b.batch, shared={}, meta=dict(b.meta))
        g = run_gpu(b)
        r64 = O.solve(b, O.Cfg.f64(), "f64")
        r32 = O.solve(b, O.Cfg.f32(), "f32")
        ok = (r32["status"] == 0) & (g["status"] == 0)
        g64 = O.backward(b, r64, O.Cfg.f64(), "f64")
        g32 = O.backward(b, r32, O.Cfg.f32(), "f32")
        res = rel_residuals(b, g["x"], g["y"], g["z"], g["s"])
        res32 = rel_residuals(b, r32["x"], r32["y"], r32["z"], r32["s"])
        print(f"== {name}: B={b.batch} ok={ok.sum()} info={g['info'].get('path')}")
        print(f"   residuals GPU max per kind (t,e,i,gap): {res[ok].max(0)}  f32-oracle: {res32[ok].max(0)}")
        print(f"   x rel GPU {x_rel(g['x'], r64['x'])[ok].max():.3e}  f32-oracle {x_rel(r32['x'], r64['x'])[ok].max():.3e}")
        d_it = np.abs(g["iters"].astype(int) - r32["iters"].astype(int))[ok]
        print(f"   iters |GPU - f32 oracle| max {d_it.max()} mean-equal {np.mean(d_it == 0):.2f}")
        eg, eo = errs(g, g64, ok), errs(g32, g64, ok)
        for k in eg:
            print(f"   {k}: GPU {eg[k][0]:.3e} (prob {eg[k][1]}, |ref| {eg[k][2]:.2e})   "
                  f"f32-oracle {eo[k][0]:.3e} (prob {eo[k][1]}, |ref| {eo[k][2]:.2e})")
        sys.stdout.flush()


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
