"""Time one solve+backward of config C at batch B (device events), print status summary.
usage: run_cfg.py C B"""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # noqa: E401,E702
import sys
import time

import numpy as np
import torch

from paper_2605_17913_b200 import generators as gen
from paper_2605_17913_b200.solver import QPSolver

cfg, B = int(sys.argv[1]), int(sys.argv[2])
t0 = time.time()
pb = gen.make_config(cfg, batch=B)
print(f"generated in {time.time() - t0:.1f}s", flush=True)
dev = torch.device("cuda:0")
sh = [k for k, v in pb.shared.items() if v]
t = {k: torch.from_numpy(getattr(pb, k)[0] if k in sh else getattr(pb, k)).to(dev)
     for k in ("Q", "q", "A", "b", "G", "h")}
S = QPSolver(B, pb.n, pb.m, pb.p, shared=sh, device=0)
print(S.info(), flush=True)
dl = torch.from_numpy(pb.dl_dx).to(dev)
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
out = S.solve(**t)
e[1].record()
g = S.backward(dl)
e[2].record()
torch.cuda.synchronize()
print(f"solve {e[0].elapsed_time(e[1]):.1f} ms  backward {e[1].elapsed_time(e[2]):.1f} ms")
print("status", np.bincount(out["status"].cpu().numpy() & 0xff), "iters", out["iters"].cpu().numpy()[:16])
