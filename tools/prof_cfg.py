"""Run solve+backward of config C at batch B twice (profiling target for ncu:
-s <launches of the first pass> -c ...).  usage: prof_cfg.py C B"""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # noqa: E401,E702
import sys

import torch

from paper_2605_17913_b200 import generators as gen
from paper_2605_17913_b200.solver import QPSolver

cfg, B = int(sys.argv[1]), int(sys.argv[2])
pb = gen.make_config(cfg, batch=B)
dev = torch.device("cuda:0")
sh = [k for k, v in pb.shared.items() if v]
t = {k: torch.from_numpy(getattr(pb, k)[0] if k in sh else getattr(pb, k)).to(dev)
     for k in ("Q", "q", "A", "b", "G", "h")}
S = QPSolver(B, pb.n, pb.m, pb.p, shared=sh, device=0)
dl = torch.ones(B, pb.n, device=dev)
for _ in range(2):
    out = S.solve(**t)
    S.backward(dl)
torch.cuda.synchronize()
print(S.info())
