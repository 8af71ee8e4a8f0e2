"""Stream-ordering and call-sequence contracts of the C ABI and the binding
(round-1 advisor findings): the programmatic launch of the backward must not
read a cotangent or overwrite a buffer the previous kernel on the stream
still uses; a second backward after one solve in QP_MEM_HOST_ASYNC mode must
recompute; a QPSolver applied twice before autograd's backward must
differentiate the right solve."""
import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen

from .helpers import FIELDS, run_gpu

pytestmark = pytest.mark.gpu


def _dev(b, shared=()):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(getattr(b, f)[0] if f in shared else getattr(b, f))).cuda()
            for f in FIELDS]


@pytest.mark.parametrize("B", [16, 300])
def test_backward_reads_cotangent_written_by_previous_kernel(B):
    """Two solvers on one stream; ctx A's ∇q is ctx B's cotangent, with no
    synchronisation: B's backward (launched programmatically behind A's)
    must see A's finished output.  Reference: the same chain with a device
    synchronisation between every call."""
    import torch
    from paper_2605_17913_b200.solver import QPSolver
    ba = gen.g_rand(21, B, 50, 10, 100)
    bb = gen.g_rand(22, B, 50, 10, 100)
    SA = QPSolver(B, 50, 10, 100)
    SB = QPSolver(B, 50, 10, 100)
    da, db = _dev(ba), _dev(bb)
    dla = torch.from_numpy(ba.dl_dx).cuda()
    res = []
    for sync in (True, False, False):
        step = torch.cuda.synchronize if sync else (lambda: None)
        SA.solve(*da); step()
        SB.solve(*db); step()
        ga = SA.backward(dla); step()
        gb = SB.backward(ga["dq"])
        torch.cuda.synchronize()
        res.append({k: v.cpu().numpy().copy() for k, v in gb.items()})
    SA.close(); SB.close()
    assert np.all(res[0]["status"] == 0)
    assert np.abs(res[0]["dq"]).max() > 0
    for r in res[1:]:
        for k in res[0]:
            assert np.array_equal(res[0][k], r[k]), k


@pytest.mark.parametrize("cfg,B", [(2, 301), (1, 16)])
def test_host_async_second_backward_recomputes(cfg, B):
    """QP_MEM_HOST_ASYNC: one solve, then two backward calls with different
    cotangents enqueued back to back; each must equal the device-mode
    gradients for its own cotangent (the chunk counters are reset on the
    chunk streams)."""
    import torch
    from paper_2605_17913_b200.solver import QPSolver
    b = gen.make_config(cfg, batch=B)
    dl2 = np.random.default_rng(7).standard_normal(b.dl_dx.shape).astype(np.float32)
    want1, want2 = run_gpu(b), run_gpu(b, dl=dl2)
    S = QPSolver(b.batch, b.n, b.m, b.p, mem="host_async")
    data = [torch.from_numpy(np.ascontiguousarray(getattr(b, f))).pin_memory() for f in FIELDS]
    S.solve(*data)
    # host inputs must stay alive and unmodified until the stream is
    # synchronised (QP_MEM_HOST_ASYNC contract): keep both cotangents
    h1, h2 = torch.from_numpy(b.dl_dx).pin_memory(), torch.from_numpy(dl2).pin_memory()
    g1 = S.backward(h1)
    g2 = S.backward(h2)
    torch.cuda.synchronize()
    S.close()
    for k in ("dQ", "dq", "dA", "db", "dG", "dh", "relax_iters"):
        assert np.array_equal(g1[k].numpy(), want1[k]), k
        assert np.array_equal(g2[k].numpy(), want2[k]), k


def test_qpfunction_solver_applied_twice():
    """The same QPSolver used for two forwards before backward (a layer
    applied twice): the first graph's gradients must be those of its own
    inputs, as with a separate solver."""
    import torch
    from paper_2605_17913_b200.solver import QPFunction, QPSolver
    b1, b2 = gen.g_rand(31, 8, 20, 3, 30), gen.g_rand(32, 8, 20, 3, 30)
    S = QPSolver(8, 20, 3, 30)
    t1 = [t.requires_grad_() for t in _dev(b1)]
    t2 = [t.requires_grad_() for t in _dev(b2)]
    x1 = QPFunction.apply(S, *t1)
    x2 = QPFunction.apply(S, *t2)
    w = torch.from_numpy(b1.dl_dx).cuda()
    (x1 * w).sum().backward()
    (x2 * w).sum().backward()
    ref = run_gpu(b1)
    ref2 = run_gpu(b2, dl=b1.dl_dx)
    for t, k in zip(t1, ("dQ", "dq", "dA", "db", "dG", "dh")):
        assert np.array_equal(t.grad.cpu().numpy(), ref[k]), k
    for t, k in zip(t2, ("dQ", "dq", "dA", "db", "dG", "dh")):
        assert np.array_equal(t.grad.cpu().numpy(), ref2[k]), k
    S.close()
