"""Pins of the oracle's Newton step: the Eq. 14 condensation and the M-form
congruence against a dense Eq. 13 assembled here from P:274-290, plus the
line search (Eq. 6), initialization and residual (Eq. 4/10) pins."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rand_qp(rng, n, m, p):
    M = rng.standard_normal((n, n))
    Q = M @ M.T / n + 0.1 * np.eye(n)
    Q = 0.5 * (Q + Q.T)
    return dict(Q=Q, q=rng.standard_normal(n), A=rng.standard_normal((m, n)), b=rng.standard_normal(m),
                G=rng.standard_normal((p, n)), h=rng.standard_normal(p))


def dense_eq13(prob, n, m, p, v, kappa, r, r_kappa, d_plus, d_minus, c):
    """Eq. 13 assembled block by block; unknown order
    (dx, dy, dz, ds, dv, dkappa)."""
    N = n + m + 3 * p + 1
    K = np.zeros((N, N))
    ix, iy, iz, is_, iv, ik = 0, n, n + m, n + m + p, n + m + 2 * p, n + m + 3 * p
    K[ix:ix + n, ix:ix + n] = prob["Q"]
    K[ix:ix + n, iy:iy + m] = prob["A"].T
    K[ix:ix + n, iz:iz + p] = prob["G"].T
    K[iy:iy + m, ix:ix + n] = prob["A"]
    K[iz:iz + p, ix:ix + n] = prob["G"]          # row block 3 (r_i)
    K[iz:iz + p, is_:is_ + p] = np.eye(p)
    K[is_:is_ + p, iz:iz + p] = np.eye(p)        # row block 4 (r_z)
    K[is_:is_ + p, iv:iv + p] = -np.diag(d_plus)
    K[is_:is_ + p, ik] = -c
    K[iv:iv + p, is_:is_ + p] = np.eye(p)        # row block 5 (r_s)
    K[iv:iv + p, iv:iv + p] = np.diag(d_minus)
    K[iv:iv + p, ik] = -c
    K[ik, ik] = 1.0                              # row 6 (r_kappa)
    rhs = -np.concatenate([r["rt"], r["re"], r["ri"], r["rz"], r["rs"], [r_kappa]])
    return K, rhs


@pytest.mark.parametrize("seed", range(50))
def test_condensation_matches_dense_eq13(orc, seed):
    """Eq. 14 solve + Eq. 13 rows 4-6 back-substitution satisfies the dense
    Eq. 13 with residual <= 1e-10 ||rhs|| in f64; the
    M-form (congruent, reading Q12) gives the same step."""
    rng = np.random.default_rng(seed)
    n, m, p = rng.integers(1, 7), rng.integers(0, 4), rng.integers(1, 7)
    m = min(m, n)
    prob = rand_qp(rng, n, m, p)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    z, s = rng.uniform(0.05, 2.0, p), rng.uniform(0.05, 2.0, p)
    kappa = float(s @ z / p)
    kt = 0.1 * kappa
    st = orc.newton_step(prob, n, m, p, x, y, z, s, kt, solver=orc.SOLVER_K14_GEPP)
    assert st["kappa"] == pytest.approx(kappa, rel=1e-14)
    r = orc.residuals(prob, n, m, p, x, y, z, s)
    ret = orc.retract(z - s, kappa)
    K, rhs = dense_eq13(prob, n, m, p, z - s, kappa, r, kappa - kt, ret["dp"], ret["dm"], ret["c"])
    sol = np.concatenate([st["dx"], st["dy"], st["dz"], st["ds"], st["dv"], [st["dk"]]])
    assert np.linalg.norm(K @ sol - rhs, np.inf) <= 1e-10 * max(1.0, np.linalg.norm(rhs, np.inf))
    # independent dense solve of Eq. 13 (library primitive) agrees
    ref = np.linalg.solve(K, rhs)
    assert np.allclose(sol, ref, rtol=1e-8, atol=1e-8 * np.abs(ref).max())
    for solver in (orc.SOLVER_M_LDL, orc.SOLVER_M_PART):
        stm = orc.newton_step(prob, n, m, p, x, y, z, s, kt, solver=solver, floor_rel=1e-14)
        assert stm["nfloor"] == 0
        for k in ("dx", "dy", "dz", "ds", "dv"):
            assert np.allclose(stm[k], st[k], rtol=1e-9, atol=1e-9 * max([1.0, *np.abs(st[k])])), (solver, k)


@pytest.mark.parametrize("seed", range(20))
def test_capped_partition_matches_dense_eq13(orc, seed):
    """Reading Q12c: keeping only the pcap constraints with the largest v_i > 0
    in augmented form (the rest eliminated with weight d+/d-) is still an
    exact block elimination, so the step equals the dense Eq. 13 solve
     for every cap, including 0 (every w_i eliminated)."""
    rng = np.random.default_rng(1000 + seed)
    n, m, p = int(rng.integers(2, 7)), int(rng.integers(0, 3)), int(rng.integers(4, 10))
    prob = rand_qp(rng, n, m, p)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    z, s = rng.uniform(0.05, 2.0, p), rng.uniform(0.05, 2.0, p)
    v = z - s
    kappa = float(s @ z / p)
    kt = 0.1 * kappa
    r = orc.residuals(prob, n, m, p, x, y, z, s)
    ret = orc.retract(v, kappa)
    K, rhs = dense_eq13(prob, n, m, p, v, kappa, r, kappa - kt, ret["dp"], ret["dm"], ret["c"])
    ref = np.linalg.solve(K, rhs)
    for cap in range(0, int((v > 0).sum()) + 1):
        st = orc.newton_step(prob, n, m, p, x, y, z, s, kt, solver=orc.SOLVER_M_PART, floor_rel=1e-14,
                             partition_cap=cap)
        sol = np.concatenate([st["dx"], st["dy"], st["dz"], st["ds"], st["dv"], [st["dk"]]])
        assert np.allclose(sol, ref, rtol=1e-8, atol=1e-8 * np.abs(ref).max()), cap


def test_zero_residual_zero_step(orc):
    """All residuals zero and kappa_target = kappa -> zero step."""
    n, p = 3, 2
    Q = np.eye(n); G = np.array([[1.0, 0, 0], [0, 1.0, 0]])
    kappa = 0.04
    z = s = np.full(p, np.sqrt(kappa))  # on-manifold with v = 0
    x = np.array([0.2, -0.1, 0.5])
    h = G @ x + s
    q = -(Q @ x + G.T @ z)
    prob = dict(Q=Q, q=q, A=np.zeros((0, n)), b=np.zeros(0), G=G, h=h)
    st = orc.newton_step(prob, n, 0, p, x, np.zeros(0), z, s, kappa)
    for k in ("dx", "dz", "ds", "dv"):
        assert np.abs(st[k]).max() <= 1e-15
    r = orc.residuals(prob, n, 0, p, x, np.zeros(0), z, s)
    assert max(np.abs(v).max() for v in r.values() if v.size) <= 1e-15


def test_residual_pins(orc):
    """S:121 unconstrained minimizer -> r_t = 0; S:122 on-manifold -> r_z = r_s = 0."""
    prob = dict(Q=np.eye(2), q=np.array([-1.0, -1.0]), A=np.zeros((0, 2)), b=np.zeros(0),
                G=np.zeros((0, 2)), h=np.zeros(0))
    r = orc.residuals(prob, 2, 0, 0, np.ones(2), np.zeros(0), np.zeros(0), np.zeros(0))
    assert np.abs(r["rt"]).max() == 0.0
    rng = np.random.default_rng(0)
    v = rng.standard_normal(5)
    ret = orc.retract(v, 1e-3)
    z, s = ret["z"], ret["s"]
    prob = dict(Q=np.eye(2), q=np.zeros(2), A=np.zeros((0, 2)), b=np.zeros(0),
                G=rng.standard_normal((5, 2)), h=rng.standard_normal(5))
    r = orc.residuals(prob, 2, 0, 5, np.zeros(2), np.zeros(0), z, s)
    scale = np.maximum(np.abs(z), np.abs(s))
    assert np.all(np.abs(r["rz"]) <= 8 * np.finfo(float).eps * scale)
    assert np.all(np.abs(r["rs"]) <= 8 * np.finfo(float).eps * scale)


def test_linesearch_printed_examples(orc):
    for ex in GOLD["linesearch"]:
        for prec in ("f64", "f32"):
            a = orc.linesearch(ex["s"], ex["z"], ex["ds"], ex["dz"], ex["tau"], prec)
            assert a == pytest.approx(ex["alpha"], rel=1e-6), ex["cite"]


def test_linesearch_keeps_interior(orc):
    """alpha = min(1, tau*alpha_max) keeps s + alpha ds >= (1-tau) s (Q3)."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        p = 7
        s, z = rng.uniform(0.1, 2, p), rng.uniform(0.1, 2, p)
        ds, dz = rng.standard_normal(p) * 3, rng.standard_normal(p) * 3
        a = orc.linesearch(s, z, ds, dz, 0.99)
        assert 0 < a <= 1
        assert np.all(s + a * ds >= 0.01 * s - 1e-15) and np.all(z + a * dz >= 0.01 * z - 1e-15)


def test_initialization(orc):
    """S:149 CVXOPT initialization: s, z > 0; with p = 0 it solves the
    equality KKT exactly; random n=5, m=2, p=4 -> r_e ~ 0."""
    rng = np.random.default_rng(1)
    prob = rand_qp(rng, 5, 2, 4)
    it = orc.initialize(prob, 5, 2, 4)
    assert it["ok"] and np.all(it["s"] > 0) and np.all(it["z"] > 0)
    assert np.abs(prob["A"] @ it["x"] - prob["b"]).max() <= 1e-10
    # (x, y) solve [[Q + ... ]]: the init system's first block row holds exactly
    # with z^ = G x - h: Q x + A'y + G'(G x - h) = -q.
    zh = prob["G"] @ it["x"] - prob["h"]
    assert np.abs(prob["Q"] @ it["x"] + prob["A"].T @ it["y"] + prob["G"].T @ zh + prob["q"]).max() <= 1e-10
    # p = 0, A=[1]: x solves the equality-constrained QP exactly
    pr = dict(Q=np.array([[2.0]]), q=np.array([1.0]), A=np.array([[1.0]]), b=np.array([2.0]),
              G=np.zeros((0, 1)), h=np.zeros(0))
    it = orc.initialize(pr, 1, 1, 0)
    assert it["x"][0] == pytest.approx(2.0) and it["y"][0] == pytest.approx(-5.0)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_initialization_shift_constructed(orc, prec):
    """S:149 (reading Q11) on constructed QPs whose init solve is known in
    closed form.  n = 1, Q = [1], G = [[1], [-1]], m = 0: the init system
    [[Q, Gᵀ], [G, -I]] (x, ẑ) = (-q, h) gives x = (h1 - h2 - q)/3,
    ẑ = (x - h1, -x - h2); s~ = -ẑ, z~ = ẑ; α_p = -min s~, α_d = -min z~;
    s = s~ + (1 + α_p) iff α_p >= 0 (else s = s~), z likewise.
    Case A (α_p = -3 < 0 -> no shift: "always shift" would give s = (1, 3);
    α_d = 5 -> z = ẑ + 6); case B (α_p = 0 -> shift by exactly 1, where a
    shift of 2 + α would give 2; α_d = 2 -> z = ẑ + 3)."""
    G = np.array([[1.0], [-1.0]])
    cases = [  # (q, h1, h2) -> (x, s, z)
        (-2.0, 3.0, 5.0, 0.0, (3.0, 5.0), (3.0, 1.0)),
        (0.0, 4.0, -2.0, 2.0, (3.0, 1.0), (1.0, 3.0)),
    ]
    for q, h1, h2, x, s, z in cases:
        pr = dict(Q=np.array([[1.0]]), q=np.array([q]), A=np.zeros((0, 1)), b=np.zeros(0), G=G,
                  h=np.array([h1, h2]))
        it = orc.initialize(pr, 1, 0, 2, prec=prec)
        assert it["ok"]
        tol = 1e-12 if prec == "f64" else 1e-6
        assert abs(it["x"][0] - x) <= tol
        assert np.abs(it["s"] - np.array(s)).max() <= tol, it["s"]
        assert np.abs(it["z"] - np.array(z)).max() <= tol, it["z"]


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_ldl_pivot_floor_branch(orc, prec):
    """Reading Q12: a pivot on the wrong side of ±θ (θ = floor_rel·max|diag|)
    is replaced by ±θ and counted; the factor and the solve then follow the
    floored pivot exactly.  Hand-computed 2×2 and 3×3 cases:
      M = [[1, 1], [1, 1]], npos = 1: d0 = 1, l10 = 1, d1 = 0 is not <= -θ
        -> d1 = -θ (1 floor); M x = (1, 3) solved as L D Lᵀ x = b:
        u = (1, 2), w = (1, -2/θ), x = (1 + 2/θ, -2/θ).
      M = [[1, 2], [2, 1]], npos = 2: d1 = 1 - 4 = -3 < θ -> d1 = +θ.
      M = diag(4, -1, -2) with npos = 3: d1 = -1 -> θ, d2 = -2 -> θ (2 floors);
        no floor when npos = 1 (quasi-definite signs respected)."""
    fr = 0.25
    r = orc.ldl([[1.0, 1.0], [1.0, 1.0]], 1, fr, [1.0, 3.0], prec=prec)
    th = fr * 1.0
    assert r["nfloor"] == 1
    assert np.allclose(r["D"], [1.0, -th]) and np.allclose(r["L"], [[1, 0], [1, 1]])
    assert np.allclose(r["x"], [1 + 2 / th, -2 / th], rtol=1e-6)
    r = orc.ldl([[1.0, 2.0], [2.0, 1.0]], 2, fr, [1.0, 0.0], prec=prec)
    assert r["nfloor"] == 1 and np.allclose(r["D"], [1.0, th]) and np.allclose(r["L"][1, 0], 2.0)
    # (L D Lᵀ) x = b with the floored D
    LDL = r["L"] @ np.diag(r["D"]) @ r["L"].T
    assert np.allclose(LDL @ r["x"], [1.0, 0.0], atol=1e-5)
    M3 = np.diag([4.0, -1.0, -2.0])
    r = orc.ldl(M3, 3, fr, [1.0, 1.0, 1.0], prec=prec)
    assert r["nfloor"] == 2 and np.allclose(r["D"], [4.0, fr * 4.0, fr * 4.0])
    r = orc.ldl(M3, 1, fr, [1.0, 1.0, 1.0], prec=prec)
    assert r["nfloor"] == 0 and np.allclose(r["D"], [4.0, -1.0, -2.0])
    assert np.allclose(r["x"], [0.25, -1.0, -0.5])
