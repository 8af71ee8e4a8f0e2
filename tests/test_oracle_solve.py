"""Pins of the oracle's Alg. 1 (and the standard arm) against closed forms,
printed examples and brute-force active-set enumeration."""
import itertools
import json
import os

import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen
from paper_2605_17913_b200.generators import QPBatch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def one(Q, q, A, b, G, h, dl=None):
    Q, q, A, b, G, h = (np.asarray(t, dtype=np.float64) for t in (Q, q, A, b, G, h))
    n = Q.shape[0]
    A = A.reshape(-1, n); G = G.reshape(-1, n)
    dl = np.zeros(n) if dl is None else np.asarray(dl, dtype=np.float64)
    return QPBatch(n, A.shape[0], G.shape[0], Q[None], q[None], A[None], b.reshape(1, -1), G[None],
                   h.reshape(1, -1), dl[None], 1)


def brute_force(Q, q, A, b, G, h):
    """Enumerate active sets: the unique KKT point of a strictly
    convex QP, found with numpy's dense solver on each candidate set."""
    n, m, p = Q.shape[0], A.shape[0], G.shape[0]
    for k in range(p + 1):
        for S in itertools.combinations(range(p), k):
            S = list(S)
            Gs = G[S]
            K = np.block([[Q, A.T, Gs.T], [A, np.zeros((m, m)), np.zeros((m, k))],
                          [Gs, np.zeros((k, m)), np.zeros((k, k))]])
            rhs = np.concatenate([-q, b, h[S]])
            try:
                sol = np.linalg.solve(K, rhs)
            except np.linalg.LinAlgError:
                continue
            x, zS = sol[:n], sol[n + m:]
            if np.all(G @ x <= h + 1e-9) and np.all(zS >= -1e-9):
                return x
    raise AssertionError("no KKT point")


def test_printed_solve_examples(orc):
    for ex in GOLD["solve"]:
        bt = one(ex["Q"], ex["q"], ex["A"] or np.zeros((0, ex["n"])), ex["b"], ex["G"] or np.zeros((0, ex["n"])),
                 ex["h"])
        r = orc.solve(bt, orc.Cfg.f64(), "f64")
        assert r["status"][0] == 0
        assert np.allclose(r["x"][0], ex["x"], atol=1e-8), ex["cite"]
        if "y" in ex:
            assert np.allclose(r["y"][0], ex["y"], atol=1e-8)
        if "z" in ex:
            assert np.allclose(r["z"][0], ex["z"], atol=1e-6)


def test_unconstrained_closed_form(orc):
    """p = m = 0: x = -Q^{-1} q (north star pin)."""
    rng = np.random.default_rng(5)
    M = rng.standard_normal((6, 6)); Q = M @ M.T + np.eye(6); q = rng.standard_normal(6)
    r = orc.solve(one(Q, q, np.zeros((0, 6)), [], np.zeros((0, 6)), []), orc.Cfg.f64(), "f64")
    assert r["status"][0] == 0 and r["iters"][0] == 0
    assert np.allclose(r["x"][0], -np.linalg.solve(Q, q), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("qv,lo,hi", [(-3.0, -1.0, 1.0), (3.0, -1.0, 1.0), (0.4, -1.0, 1.0), (-1.0, 0.5, 2.0)])
def test_box_1d(orc, qv, lo, hi):
    """1-D box QP min Qx^2/2 + qx, lo <= x <= hi: x* = clip(-q/Q, lo, hi)."""
    Qv = 2.0
    bt = one([[Qv]], [qv], np.zeros((0, 1)), [], [[1.0], [-1.0]], [hi, -lo])
    for prec, tol in (("f64", 1e-8), ("f32", 1e-4)):
        cfg = orc.Cfg.f64() if prec == "f64" else orc.Cfg.f32()
        r = orc.solve(bt, cfg, prec)
        assert r["status"][0] == 0
        assert r["x"][0][0] == pytest.approx(np.clip(-qv / Qv, lo, hi), abs=tol)


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_active_sets(orc, seed):
    """Random strictly convex QPs with p <= 9: Alg. 1 (f64) = enumeration
    oracle; f32 oracle within 1e-4 relative (north star tolerance)."""
    rng = np.random.default_rng(100 + seed)
    n, m, p = 5, int(seed % 3), 9
    b = gen.g_rand(99, 1, n, m, p, start=seed)
    # make some constraints active: shift q so the unconstrained minimizer is far out
    prob = b.problem(0)
    Q, q, A, bb, G, h = (prob[k].astype(np.float64) for k in ("Q", "q", "A", "b", "G", "h"))
    q = (q * 4.0).astype(np.float32).astype(np.float64)
    bt = one(Q, q, A, bb, G, h)
    ref = brute_force(Q, q, A, bb, G, h)
    r = orc.solve(bt, orc.Cfg.f64(), "f64")
    assert r["status"][0] == 0
    assert np.allclose(r["x"][0], ref, atol=1e-7 * max(1, np.abs(ref).max()))
    r32 = orc.solve(bt, orc.Cfg.f32(), "f32")
    assert r32["status"][0] == 0
    assert np.abs(r32["x"][0] - ref).max() <= 1e-4 * max(1, np.abs(ref).max())
    # standard arm (f64) reaches the same optimum
    rx = orc.solve(bt, orc.Cfg.f64(formulation=orc.FORM_EXPLICIT), "f64")
    assert rx["status"][0] == 0
    assert np.allclose(rx["x"][0], ref, atol=1e-7 * max(1, np.abs(ref).max()))


def test_projection_designed_point(orc):
    """App. D construction: the projection of x = y0 + G_A' (d xi) is y0
    (P:965-971), certified for p <= 12 by enumeration."""
    rng = gen._rng(77, 0)
    for d in (0.01, 1.0, 30.0):
        Q, q, A, b, G, h, pr, y0, act = gen.g_proj_one(rng, 6, 9, 3, d, margin_lo=0.1, margin_hi=1.0)
        Qd, qd, Gd, hd = Q.astype(float), q.astype(float), G.astype(float), h.astype(float)
        ref = brute_force(Qd, qd, np.zeros((0, 6)), np.zeros(0), Gd, hd)
        assert np.abs(ref - y0).max() <= 1e-5  # f32 rounding of the data only
        r = orc.solve(one(Qd, qd, np.zeros((0, 6)), [], Gd, hd), orc.Cfg.f64(), "f64")
        assert np.allclose(r["x"][0], ref, atol=1e-8)


def test_kkt_invariants_and_manifold(orc):
    """Solutions: s, z > 0; on-manifold z_i s_i = kappa;
    relative residuals below tol (reading Q4)."""
    b = gen.make_config(2, batch=8)
    for prec, cfg in (("f64", orc.Cfg.f64()), ("f32", orc.Cfg.f32())):
        r = orc.solve(b, cfg, prec)
        assert np.all(r["status"] == 0)
        assert np.all(r["s"] > 0) and np.all(r["z"] > 0)
        zs = r["z"].astype(float) * r["s"].astype(float)
        kap = zs.mean(axis=1, keepdims=True)
        rel = 1e-6 if prec == "f64" else 1e-3
        assert np.all(np.abs(zs - kap) <= rel * kap)
        for i in range(b.batch):
            pr = {k: v.astype(float) for k, v in b.problem(i).items()}
            x, y, z, s = (r[k][i].astype(float) for k in ("x", "y", "z", "s"))
            rt = pr["Q"] @ x + pr["q"] + pr["G"].T @ z + pr["A"].T @ y
            scale = max(1, *(np.abs(t).max() for t in (pr["Q"] @ x, pr["q"], pr["G"].T @ z, pr["A"].T @ y)))
            assert np.abs(rt).max() <= 2 * cfg.tol * scale


def test_f32_vs_f64_configs(orc):
    """f32 oracle vs f64 oracle on config samples: x within 1e-4 relative."""
    for c, B in ((1, 16), (2, 16), (3, 24)):
        b = gen.make_config(c, batch=B)
        r64 = orc.solve(b, orc.Cfg.f64(), "f64")
        r32 = orc.solve(b, orc.Cfg.f32(), "f32")
        assert np.all(r64["status"] == 0) and np.all(r32["status"] == 0)
        err = np.abs(r32["x"] - r64["x"]).max(1) / np.maximum(1, np.abs(r64["x"]).max(1))
        assert err.max() <= 1e-4, (c, err.max())


def test_explicit_f32_breaks_down_implicit_does_not(orc):
    """Qualitative pin of P:629 / Table 1: on near-active
    projection instances the standard f32 arm (normal equations) produces
    non-finite values, first hit in the predictor stage, while the implicit
    f32 arm converges on every instance."""
    b = gen.make_config(3, batch=30)
    ri = orc.solve(b, orc.Cfg.f32(), "f32")
    assert np.all(ri["status"] == 0)
    rx = orc.solve(b, orc.Cfg.f32(formulation=orc.FORM_EXPLICIT, kkt_solver=orc.SOLVER_NORMAL_CHOL), "f32")
    fails = (rx["status"] & 0xFF) == orc.ST_NUMERICAL_FAILURE
    assert fails.sum() >= 3
    stages = set((rx["status"][fails] >> 8).tolist())
    assert stages <= {2, 4, 5}  # predictor / corrector / line search


@pytest.mark.parametrize("cap", [52, 60, 78])
def test_capped_partition_same_solution_f64(orc, cap):
    """Reading Q12c end to end: with at most `cap` ≥ n constraints kept in
    augmented form (the rest eliminated with weight d+/d-) every Newton step
    is the same exact step (pinned against dense Eq. 13), so the f64 solve
    with the partitioned solver lands on the same x*, and the relaxed
    gradients agree, as without the cap (the paper-literal Eq. 14 solver)."""
    b = gen.make_config(2, batch=6)
    ref = orc.solve(b, orc.Cfg.f64(), "f64")
    gref = orc.backward(b, ref, orc.Cfg.f64(), "f64")
    c = orc.Cfg.f64(kkt_solver=orc.SOLVER_M_PART, partition_cap=cap)
    r = orc.solve(b, c, "f64")
    g = orc.backward(b, r, c, "f64")
    assert np.all(r["status"] == 0) and np.all(g["status"] == 0)
    assert np.abs(r["x"] - ref["x"]).max() <= 1e-8 * max(1.0, np.abs(ref["x"]).max())
    for k in ("dQ", "dq", "dG", "dh"):
        a, e = g[k].reshape(6, -1), gref[k].reshape(6, -1)
        err = np.linalg.norm(a - e, axis=1) / np.maximum(np.linalg.norm(e, axis=1), 1e-30)
        assert err.max() <= 1e-7, (k, err.max())
