"""Memory-safety and race checks of every kernel instantiation — the
substitute for compute-sanitizer, which is closed on the GPU pool (runs
under it have left GPUs needing a reset).  For each case, with QPB200_GUARD
set (include/qpb200.h qp_debug_check_guards):

* every ctx workspace carries 64 KB guard bands of 0xFF on both sides, and
  the caller's buffers are views into larger allocations with 4 KB sentinel
  bands: after solve + backward no guard or sentinel word may have changed
  (an out-of-bounds write by any kernel, into the ctx's memory or the
  caller's, fails the test);
* every output element is written (outputs are pre-filled with a NaN
  sentinel — the initcheck analogue for outputs) and no input is modified;
* the same calls repeated give bitwise identical results (a data race
  between threads or CTAs would show as run-to-run differences; the
  reductions have a fixed order)."""
import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen

pytestmark = pytest.mark.gpu

SENT = np.int32(0x7FC0DEAD)  # a NaN payload no kernel produces
GB = 1024                     # sentinel floats on each side of a caller buffer
FIELDS = ("Q", "q", "A", "b", "G", "h")

CASES = {
    "path1_128": (lambda: gen.make_config(2, batch=40), {}, {}, dict(path=1, threads=128)),
    "path1_256x2": (lambda: gen.make_config(3, batch=8), {}, {}, dict(path=1, threads=256)),
    "path1_1cta": (lambda: gen.g_rand(7, 6, 80, 8, 160), {}, {}, dict(path=1)),
    "small_n_64": (lambda: gen.make_config(1, batch=600), {}, {}, dict(threads=64)),
    "batched_shared_G": (lambda: gen.make_config(4, batch=12), {"QPB200_BCHUNK": "5"}, {}, dict(path=4)),
    "batched_per_problem_G": (lambda: gen.g_rand(13, 5, 130, 4, 200), {}, {}, dict(path=4)),
    "persistent_large_n": (lambda: gen.g_rand(13, 5, 130, 4, 200), {"QPB200_PERSISTENT_BIG": "1"}, {},
                           dict(path=3)),
    "standard_arm": (lambda: gen.make_config(1), {}, dict(formulation="explicit"), dict(path=1)),
    "host_async_pipeline": (lambda: gen.make_config(2, batch=200), {}, dict(mem="host_async"), dict(path=1)),
    "q12c_fallback": (lambda: gen.g_dup_active(41, 16, 50, 10, 100, 45), {}, {}, dict(path=1)),
}


def _guarded(shape, dtype, fill, host):
    import torch
    n = int(np.prod(shape)) if len(shape) else 1
    base = torch.empty(n + 2 * GB, dtype=torch.int32, pin_memory=host, device=None if host else "cuda:0")
    base.fill_(int(SENT))
    body = base[GB:GB + n]
    if fill is not None:
        body.copy_(torch.from_numpy(np.ascontiguousarray(fill).view(np.int32).reshape(-1)).to(body.device))
    t = body.view(torch.float32 if dtype == "f" else torch.int32).view(*shape)
    return base, t


def _bands_ok(base):
    b = base.cpu().numpy()
    return bool(np.all(b[:GB] == SENT) and np.all(b[-GB:] == SENT))


@pytest.mark.parametrize("case", sorted(CASES))
def test_guards_outputs_and_repeatability(monkeypatch, case):
    import torch
    from paper_2605_17913_b200 import capi
    from paper_2605_17913_b200.solver import GRADS, QPSolver
    make, env, kw, want = CASES[case]
    monkeypatch.setenv("QPB200_GUARD", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    b = make()
    host = kw.get("mem", "device") != "device"
    shared = [k for k, v in b.shared.items() if v]
    S = QPSolver(b.batch, b.n, b.m, b.p, shared=shared, **kw)
    B, n, m, p = b.batch, b.n, b.m, b.p
    ins = {}
    for f in FIELDS:
        a = getattr(b, f)
        a = a[0] if f in shared else a
        ins[f] = _guarded(a.shape, "f", a.astype(np.float32), host)
    dl = _guarded(b.dl_dx.shape, "f", b.dl_dx, host)
    shp = {"Q": (n, n), "q": (n,), "A": (m, n), "b": (m,), "G": (p, n), "h": (p,)}
    results = []
    for rep in range(2):
        outs = {k: _guarded(s, "f", None, host) for k, s in (("x", (B, n)), ("s", (B, p)), ("z", (B, p)),
                                                              ("y", (B, m)))}
        outs["iters"] = _guarded((B,), "i", None, host)
        outs["status"] = _guarded((B,), "i", None, host)
        gout = {g: _guarded(shp[f] if f in shared else (B, *shp[f]), "f", None, host)
                for g, f in zip(GRADS, FIELDS)}
        gout["relax_iters"] = _guarded((B,), "i", None, host)
        gout["status"] = _guarded((B,), "i", None, host)
        S.solve(*[ins[f][1] for f in FIELDS], out={k: v[1] for k, v in outs.items()})
        S.backward(dl[1], out={k: v[1] for k, v in gout.items()})
        torch.cuda.synchronize()
        info = S.info()
        for k, v in want.items():
            assert info[k] == v, (k, info)
        assert capi.qp_debug_check_guards(S.h) == 0, "a kernel wrote outside a ctx workspace"
        res = {}
        for name, (base, t) in list(outs.items()) + [("g" + k, v) for k, v in gout.items()]:
            assert _bands_ok(base), f"write outside the caller's {name}"
            arr = t.cpu().numpy()
            assert not np.any(arr.view(np.int32) == SENT), f"{name}: elements never written"
            res[name] = arr.copy()
        for f in FIELDS:
            base, t = ins[f]
            assert _bands_ok(base), f"write outside input {f}"
            a = getattr(b, f)
            assert np.array_equal(t.cpu().numpy(), (a[0] if f in shared else a).astype(np.float32)), f"{f} modified"
        assert _bands_ok(dl[0]) and np.array_equal(dl[1].cpu().numpy(), b.dl_dx)
        results.append(res)
    S.close()
    for k in results[0]:
        assert np.array_equal(results[0][k], results[1][k], equal_nan=True), f"{k} differs between runs"
