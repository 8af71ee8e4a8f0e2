"""Write tests/golden/cfg5_oracle.npz: the CPU oracle's results for the first
two problems of BASELINE config 5 (n = 1024, p = 2048, m = 0), which the
oracle needs tens of minutes per problem to produce — too slow to recompute
inside a GPU test.  Calls ONLY oracle/ (and the seeded generators); nothing
here comes from the CUDA path.

Stored per problem (f64 oracle with the M_PART solver — reading Q12b, the
congruent sign(v)-partitioned form of Eq. 14, pinned equal to the
paper-literal K14 solve to 1e-9 in tests/test_oracle_linalg.py — because the
K14 Gaussian elimination on N = 3072 would take hours here):
  x, s, z (Alg. 1's solution), iters;
  the relaxed point xr, zr (Alg. 2) and the Alg. 3 vectors dx = ∇q,
  dz = −∇h; relax_iters.  The matrix gradients ∇Q = ½(dx xrᵀ + xr dxᵀ) and
  ∇G = dz xrᵀ + zr dxᵀ are the oracle's outer products of these vectors
  (Alg. 3) and are expanded from them in the test.
Plus the f32 oracle (M_PART) iteration counts of problem 0 (the
iteration-count reference) and its x.

usage: python tools/make_cfg5_golden.py   (≈1 h on 2 host threads)"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2605_17913_b200 import generators as gen  # noqa: E402


def main():
    b = gen.make_config(5, batch=2)
    t0 = time.time()
    c64 = O.Cfg.f64(kkt_solver=O.SOLVER_M_PART)
    r = O.solve(b, c64, "f64", nthreads=2)
    print(f"f64 solve {time.time() - t0:.0f} s iters {r['iters']} status {r['status']}", flush=True)
    g = O.backward(b, r, c64, "f64", nthreads=2)
    print(f"f64 backward {time.time() - t0:.0f} s relax {g['relax_iters']} status {g['status']}", flush=True)
    b0 = b.subset([0])
    r32 = O.solve(b0, O.Cfg.f32(), "f32", nthreads=1)
    print(f"f32 solve {time.time() - t0:.0f} s iters {r32['iters']}", flush=True)
    np.savez_compressed(
        os.path.join(ROOT, "tests", "golden", "cfg5_oracle.npz"),
        x=r["x"], s=r["s"], z=r["z"], iters=r["iters"], status=r["status"],
        xr=g["relaxed"]["x"], zr=g["relaxed"]["z"], dx=g["dq"], dz=-g["dh"], relax_iters=g["relax_iters"],
        gstatus=g["status"], iters32=r32["iters"], x32=r32["x"], s32=r32["s"], z32=r32["z"],
        note=np.array("config 5 problems 0,1 (generators.make_config(5)); f64 oracle M_PART; "
                      "written by tools/make_cfg5_golden.py"))


if __name__ == "__main__":
    main()
