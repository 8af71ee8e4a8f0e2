"""One small run of every kernel instantiation, for compute-sanitizer
(tools/sanitize.sh).  usage: python tools/sanitize_cases.py CASE
Cases: p1_128 (path 1, 128 threads, 4 CTAs/SM), p1_256x2 (256 threads,
2 CTAs/SM), p1_256x1 (256 threads, 1 CTA/SM), small64 (64-thread small-n
path), bigN (large-N kernels: tcgen05 assembly + factorisation), explicit
(standard arm), shared (batch-sum kernels), host_async (8-chunk host
pipeline, two backward calls), pdl (backward launched behind the solve
with programmatic serialisation, no host sync)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_17913_b200 import generators as gen  # noqa: E402
from paper_2605_17913_b200.solver import QPSolver  # noqa: E402

F = ("Q", "q", "A", "b", "G", "h")


def run(b, mem="device", formulation="implicit", backwards=1, sync=True, expect=None, **cfg):
    shared = [k for k, v in b.shared.items() if v]
    S = QPSolver(b.batch, b.n, b.m, b.p, shared=shared, mem=mem, formulation=formulation, **cfg)
    info = S.info()
    if expect:
        for k, v in expect.items():
            assert info[k] == v, (k, info)

    def T(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.cuda() if mem == "device" else t.pin_memory()

    data = [T(getattr(b, f)[0] if f in shared else getattr(b, f)) for f in F]
    out = S.solve(*data)
    if sync:
        torch.cuda.synchronize()
    for i in range(backwards):
        g = S.backward(T(b.dl_dx * (1.0 + i)))
    torch.cuda.synchronize()
    st = out["status"].cpu().numpy()
    print(case, info, "status", np.bincount(st & 0xFF), "grad", np.bincount(g["status"].cpu().numpy() & 0xFF))
    S.close()


case = sys.argv[1]
if case == "p1_128":
    run(gen.make_config(2, batch=8), expect=dict(path=1, threads=128))
elif case == "p1_256x2":
    run(gen.make_config(3, batch=4), expect=dict(path=1, threads=256))
elif case == "p1_256x1":
    run(gen.make_workload("cbf9", batch=4) if False else gen.g_rand(7, 3, 80, 8, 160), expect=dict(path=1))
elif case == "small64":
    run(gen.make_config(1, batch=600), expect=dict(threads=64))
elif case == "bigN":
    run(gen.g_rand(2, 2, 130, 0, 200), expect=dict(threads=256))
elif case == "explicit":
    run(gen.make_config(1, batch=4), formulation="explicit")
elif case == "shared":
    run(gen.g_rand_shared(4, 6, 20, 2, 30))
elif case == "host_async":
    run(gen.make_config(2, batch=130), mem="host_async", backwards=2, sync=False)
elif case == "pdl":
    run(gen.make_config(2, batch=40), sync=False, backwards=2)
else:
    raise SystemExit(f"unknown case {case}")
