"""Config 5 (n = 1024, p = 2048, one CTA per problem, KKT in the global
workspace, tensor-core assembly) at its full problem size on a small batch.
The oracle needs minutes per problem at this size, so parity is checked
through properties that hold at any size:

* forward: the f64 KKT residuals and gap of the f32 outputs (Eq. 4, the
  relative form of reading Q4) are within the north-star 1e-5;
* backward: the q-gradient is J d with J = -(M^-1)_xx of the symmetric,
  quasi-definite relaxed KKT matrix M (App. A.2, Alg. 3, reading Q7), so the
  map d -> dq is linear, symmetric (<d1, J d2> = <d2, J d1>) and negative
  semi-definite (<d, J d> <= 0); dQ is symmetric and dh = -dz is
  consistent with dG's rank-2 structure."""
import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen

from .helpers import FIELDS, TOL_RES, rel_residuals

pytestmark = pytest.mark.gpu


def test_cfg5_full_size_properties():
    import torch
    from paper_2605_17913_b200.solver import QPSolver
    B = 2
    pb = gen.make_config(5, batch=B)
    dev = "cuda:0"
    S = QPSolver(B, pb.n, pb.m, pb.p)
    assert S.info()["path"] == 4  # batched phase engine
    data = [torch.from_numpy(np.ascontiguousarray(getattr(pb, f))).to(dev) for f in FIELDS]
    out = S.solve(*data)
    torch.cuda.synchronize()
    st = out["status"].cpu().numpy()
    assert np.all(st == 0), st
    x, y, z, s = (out[k].cpu().numpy() for k in ("x", "y", "z", "s"))
    res = rel_residuals(pb, x, y, z, s)
    assert res.max() <= TOL_RES, res
    rng = np.random.default_rng(5)
    d1 = rng.standard_normal((B, pb.n)).astype(np.float32)
    d2 = rng.standard_normal((B, pb.n)).astype(np.float32)
    g = {}
    for name, d in (("1", d1), ("2", d2), ("12", d1 + d2)):
        gg = S.backward(torch.from_numpy(d).to(dev))
        torch.cuda.synchronize()
        g[name] = {k: v.cpu().numpy().astype(np.float64) for k, v in gg.items()}
        assert np.all(g[name]["status"] == 0)
        for k in ("dQ", "dq", "dG", "dh"):
            assert np.all(np.isfinite(g[name][k])), k
    S.close()
    J1, J2, J12 = g["1"]["dq"], g["2"]["dq"], g["12"]["dq"]
    nrm = np.linalg.norm(J12, axis=1)
    assert (np.linalg.norm(J12 - J1 - J2, axis=1) / nrm).max() < 1e-4   # linear in d
    a = np.einsum("bi,bi->b", d1.astype(np.float64), J2)
    b = np.einsum("bi,bi->b", d2.astype(np.float64), J1)
    scale = np.linalg.norm(d1, axis=1) * np.linalg.norm(J2, axis=1)
    assert (np.abs(a - b) / scale).max() < 1e-4                           # symmetric
    q1 = np.einsum("bi,bi->b", d1.astype(np.float64), J1)
    assert np.all(q1 <= 1e-5 * np.linalg.norm(d1, axis=1) * np.linalg.norm(J1, axis=1))  # NSD
    dQ = g["1"]["dQ"]
    assert np.abs(dQ - np.swapaxes(dQ, 1, 2)).max() <= 1e-6 * np.abs(dQ).max()
    # dG = dz x_r^T + z_r dx^T with dz = -dh, dx = dq: rows of dG - (-dh) x_r^T lie along dq
    dG, dh = g["1"]["dG"], g["1"]["dh"]
    for i in range(B):
        # least-squares x_r from dG ≈ -dh x_r^T + z_r dq^T: project out the dq direction
        R = dG[i] - np.outer(-dh[i], x[i])                      # ≈ z_r dq^T + O(x_r - x*)
        u = J1[i] / np.linalg.norm(J1[i])
        resid = R - np.outer(R @ u, u)                          # remove the rank-1 dq part
        assert np.linalg.norm(resid) <= 1e-2 * np.linalg.norm(dG[i]), np.linalg.norm(resid) / np.linalg.norm(dG[i])


def test_cfg5_against_oracle_golden():
    """Config 5 at full size (n = 1024, p = 2048) against the CPU oracle.  The
    oracle needs tens of minutes per problem here, so its results for
    problems 0 and 1 were written once by tools/make_cfg5_golden.py (which
    calls only oracle/ — f64 with the M_PART solver, reading Q12b, pinned
    equal to the paper-literal Eq. 14 solve) into tests/golden/cfg5_oracle.npz.
    North-star bar, unfloored: x within 1e-4 of f64, residuals ≤ 1e-5, every
    gradient field within 1e-3 (∇Q, ∇G expanded from the oracle's Alg. 3
    vectors by P:559-575's outer products), iterations within ±1 of the f32
    oracle (problem 0); precision-limit exception of tests/helpers.py where
    the f32 oracle result exists (problem 0)."""
    import os
    from .helpers import TOL_GRAD, TOL_X, run_gpu, within_bar, x_rel
    gold = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_oracle.npz")))
    pb = gen.make_config(5, batch=2)
    g = run_gpu(pb)
    assert np.all(g["status"] == 0) and np.all(g["grad_status"] == 0)
    assert np.all(gold["status"] == 0) and np.all(gold["gstatus"] == 0)
    inf = np.array([np.inf])
    ex32 = np.concatenate([x_rel(gold["x32"], gold["x"][:1]), inf])      # f32 oracle only for problem 0
    within_bar(x_rel(g["x"], gold["x"]), ex32, TOL_X, "x")
    res = rel_residuals(pb, g["x"], g["y"], g["z"], g["s"])
    sub = pb.subset([0])
    res32 = rel_residuals(sub, gold["x32"], np.zeros((1, 0), np.float32), gold["z32"], gold["s32"])
    for j in range(4):
        within_bar(res[:, j], np.concatenate([res32[:, j], [0.0]]), TOL_RES, f"residual {j}")
    assert abs(int(g["iters"][0]) - int(gold["iters32"][0])) <= 1, (g["iters"], gold["iters32"])
    dx, dz, xr, zr = (gold[k].astype(np.float64) for k in ("dx", "dz", "xr", "zr"))
    ref = {"dq": dx, "dh": -dz,
           "dQ": 0.5 * (np.einsum("bi,bj->bij", dx, xr) + np.einsum("bi,bj->bij", xr, dx)),
           "dG": np.einsum("bi,bj->bij", dz, xr) + np.einsum("bi,bj->bij", zr, dx)}
    for k, r in ref.items():
        a = g[k].reshape(2, -1).astype(np.float64)
        r = r.reshape(2, -1)
        err = np.linalg.norm(a - r, axis=1) / np.linalg.norm(r, axis=1)
        assert err.max() <= TOL_GRAD, (k, err)
