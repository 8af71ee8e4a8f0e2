"""Seeded synthetic QP generators shared by the oracle tests, the CUDA parity
tests and bench.py.

This module holds NONE of the method's arithmetic (no residuals, no
retraction, no KKT algebra): it only draws problem data.  Both the oracle
(`oracle/`) and the CUDA path (`paper_2605_17913_b200`) receive the arrays it
returns.  Every problem i of config c is drawn from its own stream
``np.random.SeedSequence([c, i])`` (PCG64), so any subset of a batch can be
regenerated bit-identically on its own (SURVEY.md §8(d) "Synthetic inputs").

All data is drawn in float64 and then rounded ONCE to float32; the float32
values are the problem.  The f64 oracle runs on those same (exactly
representable) values, so GPU-vs-oracle differences are solver differences,
never input differences.

Workload recipes (DESIGN.md §3 restates them with citations):

* ``g_rand(n, m, p)`` — "random feasible dense QP" (BASELINE.json configs 1,
  2, 5; shared data of config 4): M~N(0,1)^{n×n}, Q = M Mᵀ/n + 0.1·I
  (strictly convex), q~N(0,1); A~N(0,1)/√n, x0~N(0,1), b = A x0;
  G~N(0,1)/√n, s0~U(0,1), h = G x0 + s0 (x0 strictly feasible);
  ∇ₓℓ~N(0,1).
* ``g_proj(n, p, m_act, d)`` — polytope projection of PAPER.md App. D
  (P:887-921): unit-norm rows of G, boundary point y0, m_act
  active rows h_A = G_A y0, inactive rows h = G y0 + margin with margin
  log-uniform in [1e-3, 1] ("near-active", BASELINE config 3), query
  x = y0 + G_Aᵀ(d·ξ), ξ~U(0.5,1.5); Q = I, q = −x;
  ∇ₓℓ = probe v~N(0,I).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

F32 = np.float32


def _rng(cfg: int, i: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(cfg), int(i)])))


@dataclass
class QPBatch:
    """A batch of dense QPs in the C-ABI layout: batch-major, row-major f32.

    A field whose batch dimension is 1 and whose ``shared_*`` flag is set is
    shared across the batch (C-ABI batch stride 0)."""

    n: int
    m: int
    p: int
    Q: np.ndarray  # [B|1, n, n]
    q: np.ndarray  # [B|1, n]
    A: np.ndarray  # [B|1, m, n]
    b: np.ndarray  # [B|1, m]
    G: np.ndarray  # [B|1, p, n]
    h: np.ndarray  # [B|1, p]
    dl_dx: np.ndarray  # [B, n]
    batch: int
    shared: dict = field(default_factory=dict)  # name -> True if stride 0
    meta: dict = field(default_factory=dict)

    def problem(self, i: int) -> dict:
        """Dense f32 arrays of problem i (shared fields broadcast)."""
        def pick(name):
            arr = getattr(self, name)
            return arr[0] if self.shared.get(name, False) else arr[i]
        return {k: pick(k) for k in ("Q", "q", "A", "b", "G", "h")} | {"dl_dx": self.dl_dx[i]}

    def subset(self, idx) -> "QPBatch":
        idx = np.asarray(idx, dtype=np.int64)
        def sel(name):
            arr = getattr(self, name)
            return arr if self.shared.get(name, False) else np.ascontiguousarray(arr[idx])
        return QPBatch(self.n, self.m, self.p, sel("Q"), sel("q"), sel("A"), sel("b"),
                       sel("G"), sel("h"), np.ascontiguousarray(self.dl_dx[idx]), len(idx),
                       dict(self.shared), dict(self.meta))


def _sym(Q: np.ndarray) -> np.ndarray:
    return 0.5 * (Q + Q.T)


def g_rand_one(rng: np.random.Generator, n: int, m: int, p: int):
    M = rng.standard_normal((n, n))
    Q = _sym(M @ M.T / n + 0.1 * np.eye(n))
    q = rng.standard_normal(n)
    A = rng.standard_normal((m, n)) / np.sqrt(n)
    x0 = rng.standard_normal(n)
    G = rng.standard_normal((p, n)) / np.sqrt(n)
    s0 = rng.uniform(0.0, 1.0, p)
    # Round the matrices first so that b and h are computed from the f32 data
    # the solver actually sees (x0 stays strictly feasible up to f32 rounding
    # of b, h themselves).
    A32, G32 = A.astype(F32), G.astype(F32)
    b = A32.astype(np.float64) @ x0
    h = G32.astype(np.float64) @ x0 + s0
    dl = rng.standard_normal(n)
    return Q.astype(F32), q.astype(F32), A32, b.astype(F32), G32, h.astype(F32), dl.astype(F32)


def g_rand(cfg: int, batch: int, n: int, m: int, p: int, start: int = 0) -> QPBatch:
    """Config-`cfg` batch of random feasible strictly convex QPs."""
    Qs = np.empty((batch, n, n), F32); qs = np.empty((batch, n), F32)
    As = np.empty((batch, m, n), F32); bs = np.empty((batch, m), F32)
    Gs = np.empty((batch, p, n), F32); hs = np.empty((batch, p), F32)
    dls = np.empty((batch, n), F32)
    for j in range(batch):
        Q, q, A, b, G, h, dl = g_rand_one(_rng(cfg, start + j), n, m, p)
        Qs[j], qs[j], As[j], bs[j], Gs[j], hs[j], dls[j] = Q, q, A, b, G, h, dl
    return QPBatch(n, m, p, Qs, qs, As, bs, Gs, hs, dls, batch,
                   meta={"recipe": "g_rand", "cfg": cfg, "start": start})


def g_dup_active(cfg: int, batch: int, n: int, m: int, p: int, n_act: int, start: int = 0) -> QPBatch:
    """Degenerate QPs that VIOLATE LICQ with many strongly active constraints
    (the situation reading Q12c's kept-set cap must survive):
    n_act distinct hyperplanes g_iᵀx = h_i, each appearing TWICE in G (2·n_act
    active rows whose normals are linearly dependent), through a chosen point
    x0; the other p − 2·n_act rows inactive with margins U(0.5, 1.5).  q is set
    so that x0 is optimal with positive multipliers on the active rows:
    q = −Q x0 − Σ_i λ_i g_i − Aᵀμ, λ_i ~ U(0.5, 1.5), b = A x0.  The solution
    is therefore x* = x0 exactly (the multiplier split between the duplicates
    is not unique).  Q, A as in g_rand; ∇ₓℓ ~ N(0, 1).  meta["x_star"] = x0."""
    assert 2 * n_act <= p
    Qs = np.empty((batch, n, n), F32); qs = np.empty((batch, n), F32)
    As = np.empty((batch, m, n), F32); bs = np.empty((batch, m), F32)
    Gs = np.empty((batch, p, n), F32); hs = np.empty((batch, p), F32)
    dls = np.empty((batch, n), F32); xs = np.empty((batch, n))
    for j in range(batch):
        rng = _rng(cfg, start + j)
        M = rng.standard_normal((n, n))
        Q = _sym(M @ M.T / n + 0.1 * np.eye(n)).astype(F32).astype(np.float64)
        A = (rng.standard_normal((m, n)) / np.sqrt(n)).astype(F32).astype(np.float64)
        Gd = (rng.standard_normal((n_act, n)) / np.sqrt(n)).astype(F32).astype(np.float64)
        Gi = (rng.standard_normal((p - 2 * n_act, n)) / np.sqrt(n)).astype(F32).astype(np.float64)
        x0 = rng.standard_normal(n).astype(F32).astype(np.float64)
        lam = rng.uniform(0.5, 1.5, n_act)
        mu = rng.standard_normal(m)
        G = np.concatenate([Gd, Gd, Gi])
        h = np.concatenate([Gd @ x0, Gd @ x0, Gi @ x0 + rng.uniform(0.5, 1.5, p - 2 * n_act)])
        q = -(Q @ x0) - Gd.T @ lam - A.T @ mu
        Qs[j], qs[j], As[j], bs[j] = Q, q, A, A @ x0
        Gs[j], hs[j], dls[j], xs[j] = G, h, rng.standard_normal(n), x0
    return QPBatch(n, m, p, Qs, qs, As, bs, Gs, hs, dls, batch,
                   meta={"recipe": "g_dup_active", "cfg": cfg, "start": start, "x_star": xs})


def g_rand_shared(cfg: int, batch: int, n: int, m: int, p: int, start: int = 0) -> QPBatch:
    """Config 4 ("end-to-end/bilevel"): Q, A, b, G, h shared across the batch
    (drawn once from stream [cfg, 0]); per-instance q_b~N(0,1) and ∇ₓℓ_b~N(0,1)
    from streams [cfg, 1+i]."""
    Q, _, A, b, G, h, _ = g_rand_one(_rng(cfg, 0), n, m, p)
    qs = np.empty((batch, n), F32); dls = np.empty((batch, n), F32)
    for j in range(batch):
        r = _rng(cfg, 1 + start + j)
        qs[j] = r.standard_normal(n).astype(F32)
        dls[j] = r.standard_normal(n).astype(F32)
    return QPBatch(n, m, p, Q[None], qs, A[None], b[None], G[None], h[None], dls, batch,
                   shared={"Q": True, "A": True, "b": True, "G": True, "h": True},
                   meta={"recipe": "g_rand_shared", "cfg": cfg, "start": start})


def g_proj_one(rng: np.random.Generator, n: int, p: int, m_act: int, d: float,
               margin_lo: float = 1e-3, margin_hi: float = 1.0):
    """One polytope-projection instance (App. D.1-D.3).

    Returns f32 (Q, q, A, b, G, h, probe) plus f64 (y0, active_idx) for the
    hard-Jacobian reference.  Active rows are redrawn until G_A has full row
    rank ("rank(G_A) = m")."""
    for _ in range(100):
        G = rng.standard_normal((p, n))
        G /= np.linalg.norm(G, axis=1, keepdims=True)
        active = np.sort(rng.choice(p, size=m_act, replace=False))
        if m_act == 0 or np.linalg.matrix_rank(G[active]) == m_act:
            break
    else:  # pragma: no cover
        raise RuntimeError("rank-deficient active set after 100 redraws")
    G32 = G.astype(F32)
    Gd = G32.astype(np.float64)
    y0 = rng.standard_normal(n)
    margin = np.exp(rng.uniform(np.log(margin_lo), np.log(margin_hi), p))
    h = Gd @ y0
    inactive = np.ones(p, bool); inactive[active] = False
    h[inactive] += margin[inactive]
    xi = rng.uniform(0.5, 1.5, m_act)
    xq = y0 + Gd[active].T @ (d * xi)
    probe = rng.standard_normal(n)
    Q = np.eye(n, dtype=F32)
    return (Q, (-xq).astype(F32), np.zeros((0, n), F32), np.zeros(0, F32), G32,
            h.astype(F32), probe.astype(F32), y0, active)


D_GRID = np.logspace(-2, 2, 21)
MR_GRID = (0.2, 0.6, 0.8)


def g_proj(cfg: int, batch: int, n: int, p: int, start: int = 0) -> QPBatch:
    """Config 3 batch: instance i cycles (m_r, d) over MR_GRID × D_GRID
     with its own seed stream [cfg, i]."""
    Qs = np.empty((batch, n, n), F32); qs = np.empty((batch, n), F32)
    Gs = np.empty((batch, p, n), F32); hs = np.empty((batch, p), F32)
    dls = np.empty((batch, n), F32)
    y0s = np.empty((batch, n)); actives = []
    mrs = np.empty(batch); ds = np.empty(batch)
    for j in range(batch):
        i = start + j
        mr = MR_GRID[i % 3]; d = D_GRID[(i // 3) % len(D_GRID)]
        m_act = int(round(mr * n))
        Q, q, _, _, G, h, pr, y0, act = g_proj_one(_rng(cfg, i), n, p, m_act, d)
        Qs[j], qs[j], Gs[j], hs[j], dls[j] = Q, q, G, h, pr
        y0s[j] = y0; actives.append(act); mrs[j] = mr; ds[j] = d
    return QPBatch(n, 0, p, Qs, qs, np.zeros((batch, 0, n), F32), np.zeros((batch, 0), F32),
                   Gs, hs, dls, batch,
                   meta={"recipe": "g_proj", "cfg": cfg, "start": start, "y0": y0s,
                         "active": actives, "m_r": mrs, "d": ds})


# BASELINE.json configs (m_eq/p readings for 4 and 5 are
# SURVEY's proposal, restated in DESIGN.md).
CONFIGS = {
    1: dict(name="cfg1_rand_n10_m2_p20_B16", n=10, m=2, p=20, batch=16, recipe="g_rand"),
    2: dict(name="cfg2_optnet_n50_m10_p100_B1024", n=50, m=10, p=100, batch=1024, recipe="g_rand"),
    3: dict(name="cfg3_proj_n100_p125_B4096", n=100, m=0, p=125, batch=4096, recipe="g_proj"),
    4: dict(name="cfg4_bilevel_shared_n200_p400_B8192", n=200, m=0, p=400, batch=8192,
            recipe="g_rand_shared"),
    5: dict(name="cfg5_large_n1024_p2048_B256", n=1024, m=0, p=2048, batch=256, recipe="g_rand"),
}


def make_config(cfg: int, batch: int | None = None, start: int = 0) -> QPBatch:
    c = CONFIGS[cfg]
    B = c["batch"] if batch is None else batch
    if c["recipe"] == "g_rand":
        return g_rand(cfg, B, c["n"], c["m"], c["p"], start)
    if c["recipe"] == "g_rand_shared":
        return g_rand_shared(cfg, B, c["n"], c["m"], c["p"], start)
    return g_proj(cfg, B, c["n"], c["p"], start)


# ---------------------------------------------------------------------------
# the paper's application shapes as synthetic batches.
# ---------------------------------------------------------------------------
def g_cbf_one(rng: np.random.Generator, agents: int, n_obs: int = 3, r_agent: float = 0.35,
              u_max: float = 2.0, kp: float = 1.5):
    """One centralised CBF safety-filter QP (App. F):
    min_u ½‖u − u_nom‖² s.t. the zeroing-CBF rows for every (agent, obstacle)
    and every agent pair, and the box |u_k| ≤ u_max; u ∈ R^{2·agents},
    p = 4n + n·obs + n(n−1)/2 rows (n = agents; 70 for 7 agents).

    Synthetic stand-ins for what the paper learns or rolls out: positions are
    rejection-sampled safe (every barrier h > 0, so u = 0 is strictly
    feasible), half of them close to an obstacle boundary and some close to an
    earlier agent (the paper's data concentrate "near regions where safety
    constraints become active"); u_nom is the goal-seeking PD proposal
     clipped to the box plus an N(0, 0.5²) "network" correction that
    may leave it; the learned gains α are U(0.5, 5)."""
    L = 2.0 + 1.5 * np.sqrt(agents)
    c = rng.uniform(0.2 * L, 0.8 * L, (n_obs, 2))
    r = rng.uniform(0.3, 0.8, n_obs)
    P = np.empty((agents, 2))
    for i in range(agents):
        for _ in range(10000):
            u = rng.random()
            if u < 0.5:
                o = rng.integers(n_obs)
                ang = rng.uniform(0.0, 2.0 * np.pi)
                dist = r[o] + 0.02 + rng.exponential(0.2)
                cand = c[o] + dist * np.array([np.cos(ang), np.sin(ang)])
            elif u < 0.7 and i > 0:
                j = rng.integers(i)
                ang = rng.uniform(0.0, 2.0 * np.pi)
                dist = 2 * r_agent + 0.02 + rng.exponential(0.1)
                cand = P[j] + dist * np.array([np.cos(ang), np.sin(ang)])
            else:
                cand = rng.uniform(0.0, L, 2)
            ok = np.all(np.linalg.norm(c - cand, axis=1) > r + 0.01)
            ok = ok and (i == 0 or np.all(np.linalg.norm(P[:i] - cand, axis=1) > 2 * r_agent + 0.01))
            if ok:
                break
        else:  # pragma: no cover
            raise RuntimeError("could not place a safe agent")
        P[i] = cand
    goals = rng.uniform(0.0, L, (agents, 2))
    dgo = goals - P
    u_pd = kp * dgo / np.maximum(np.linalg.norm(dgo, axis=1, keepdims=True), 1e-3)
    u_nom = np.clip(u_pd, -u_max, u_max) + 0.5 * rng.standard_normal((agents, 2))
    nv = 2 * agents
    rows, rhs = [], []
    for i in range(agents):            # obstacle barriers: −∇h·u_i ≤ α h
        for o in range(n_obs):
            g = np.zeros(nv)
            g[2 * i:2 * i + 2] = -2.0 * (P[i] - c[o])
            rows.append(g)
            rhs.append(rng.uniform(0.5, 5.0) * (np.sum((P[i] - c[o]) ** 2) - r[o] ** 2))
    for i in range(agents):            # pair barriers: −∇h·u ≤ α h
        for j in range(i + 1, agents):
            g = np.zeros(nv)
            dij = P[i] - P[j]
            g[2 * i:2 * i + 2] = -2.0 * dij
            g[2 * j:2 * j + 2] = 2.0 * dij
            rows.append(g)
            rhs.append(rng.uniform(0.5, 5.0) * (np.sum(dij ** 2) - (2 * r_agent) ** 2))
    for k in range(nv):                # box
        g = np.zeros(nv); g[k] = 1.0; rows.append(g); rhs.append(u_max)
        g = np.zeros(nv); g[k] = -1.0; rows.append(g); rhs.append(u_max)
    G = np.array(rows)
    h = np.array(rhs)
    dl = rng.standard_normal(nv)
    return (np.eye(nv, dtype=F32), (-u_nom.reshape(-1)).astype(F32), np.zeros((0, nv), F32), np.zeros(0, F32),
            G.astype(F32), h.astype(F32), dl.astype(F32))


def g_cbf(agents: int, batch: int, start: int = 0, stream: int = 100) -> QPBatch:
    """A batch of safety-filter QPs; problem i uses SeedSequence([stream + agents, i])."""
    nv = 2 * agents
    p = 4 * agents + 3 * agents + agents * (agents - 1) // 2
    Qs = np.empty((batch, nv, nv), F32); qs = np.empty((batch, nv), F32)
    Gs = np.empty((batch, p, nv), F32); hs = np.empty((batch, p), F32)
    dls = np.empty((batch, nv), F32)
    for j in range(batch):
        Q, q, _, _, G, h, dl = g_cbf_one(_rng(stream + agents, start + j), agents)
        Qs[j], qs[j], Gs[j], hs[j], dls[j] = Q, q, G, h, dl
    return QPBatch(nv, 0, p, Qs, qs, np.zeros((batch, 0, nv), F32), np.zeros((batch, 0), F32), Gs, hs, dls,
                   batch, meta={"recipe": "g_cbf", "agents": agents, "start": start})


# N4 workloads (not BASELINE.json configs): name -> (builder, default batch)
WORKLOADS = {
    "cbf7": dict(name="cbf7_safety_filter_n14_p70_B4096", build=lambda B, s: g_cbf(7, B, s), batch=4096),
    "cbf9": dict(name="cbf9_safety_filter_n18_p135_B4096", build=lambda B, s: g_cbf(9, B, s), batch=4096),
}


def make_workload(name: str, batch: int | None = None, start: int = 0) -> QPBatch:
    w = WORKLOADS[name]
    return w["build"](w["batch"] if batch is None else batch, start)


def _bernstein_gram(m: int) -> np.ndarray:
    """G[i][j] = ∫₀¹ b_i^m(u) b_j^m(u) du = C(m,i) C(m,j) / ((2m+1) C(2m,i+j))."""
    from math import comb
    return np.array([[comb(m, i) * comb(m, j) / ((2 * m + 1) * comb(2 * m, i + j)) for j in range(m + 1)]
                     for i in range(m + 1)])


def _bezier_diff(n: int, r: int) -> np.ndarray:
    """M_r: control points of the r-th u-derivative of a degree-n Bézier curve."""
    M = np.eye(n + 1)
    for k in range(r):
        m = n - k
        D = np.zeros((m, m + 1))
        for j in range(m):
            D[j, j], D[j, j + 1] = -m, m
        M = D @ M
    return M


def g_bezier_one(rng: np.random.Generator, K: int, deg: int = 4, weights=(0.1, 0.1, 1.0, 0.1),
                 vel=10.0, acc=2.0):
    """One inner QP of the bilevel trajectory optimisation (App. E,
    P:1045-1107): K Bézier segments of degree 4 in the plane, x = stacked
    control points (K·5·2); Q(T) = Σ_r w_r T_k^{1−2r} M_rᵀ Gram M_r per segment
    and axis (r = 1..4, w = (0.1, 0.1, 1, 0.1)), q = 0;
    equalities: start/goal points, C² continuity across segments
    (M_r P)/T^r matched for r = 0, 1, 2, rest at both ends (r = 1, 2);
    inequalities: every control point of segment k inside its safe cell
    (a rotated box, 4 facets) and |M_r P_k / T_k^r| ≤ (10, 2) for r = 1, 2
    (P:1090-1094).  Synthetic stand-ins for the maps (pydecomp) and the outer
    L-BFGS iterate: a corridor of K overlapping cells along a random walk
    toward the goal, durations T_k ~ U(1.5, 3)."""
    d, npt = 2, deg + 1
    nv = K * npt * d
    # corridor of overlapping rotated boxes
    centers = np.zeros((K, 2))
    heading = rng.uniform(0.0, 2.0 * np.pi)
    for k in range(1, K):
        heading += rng.uniform(-np.pi / 4, np.pi / 4)
        centers[k] = centers[k - 1] + 1.5 * np.array([np.cos(heading), np.sin(heading)])
    half = rng.uniform(0.9, 1.3, (K, 2))
    theta = rng.uniform(0.0, np.pi / 2, K)
    T = rng.uniform(1.5, 3.0, K)
    start, goal = centers[0], centers[-1]

    def idx(k, j, a):  # variable index of control point j of segment k, axis a
        return (k * npt + j) * d + a

    Q = np.zeros((nv, nv))
    for k in range(K):
        Qk = np.zeros((npt, npt))
        for r, w in enumerate(weights, start=1):
            Mr = _bezier_diff(deg, r)
            Qk += w * T[k] ** (1 - 2 * r) * Mr.T @ _bernstein_gram(deg - r) @ Mr
        for a in range(d):
            ids = [idx(k, j, a) for j in range(npt)]
            Q[np.ix_(ids, ids)] += Qk
    rows, rhs = [], []

    def eq(coeffs, val):
        g = np.zeros(nv)
        for (k, j, a), c in coeffs:
            g[idx(k, j, a)] += c
        rows.append(g); rhs.append(val)
    for a in range(d):
        eq([((0, 0, a), 1.0)], start[a])
        eq([((K - 1, deg, a), 1.0)], goal[a])
    for r in (0, 1, 2):
        Mr = _bezier_diff(deg, r)
        for a in range(d):
            for k in range(K - 1):      # (M_r P_k)_end / T_k^r = (M_r P_{k+1})_start / T_{k+1}^r
                co = [((k, j, a), Mr[-1, j] / T[k] ** r) for j in range(npt)]
                co += [((k + 1, j, a), -Mr[0, j] / T[k + 1] ** r) for j in range(npt)]
                eq(co, 0.0)
            if r > 0:                   # rest at both ends
                eq([((0, j, a), Mr[0, j] / T[0] ** r) for j in range(npt)], 0.0)
                eq([((K - 1, j, a), Mr[-1, j] / T[K - 1] ** r) for j in range(npt)], 0.0)
    A = np.array(rows); b = np.array(rhs)
    rows, rhs = [], []
    for k in range(K):                  # cell membership of every control point
        R = np.array([[np.cos(theta[k]), -np.sin(theta[k])], [np.sin(theta[k]), np.cos(theta[k])]])
        for j in range(npt):
            for ax in range(2):
                for sgn in (1.0, -1.0):
                    nrm = sgn * R[:, ax]
                    g = np.zeros(nv)
                    g[idx(k, j, 0)], g[idx(k, j, 1)] = nrm
                    rows.append(g); rhs.append(nrm @ centers[k] + half[k, ax])
    for r, bound in ((1, vel), (2, acc)):  # derivative control polygons
        Mr = _bezier_diff(deg, r)
        for k in range(K):
            for i in range(Mr.shape[0]):
                for a in range(d):
                    for sgn in (1.0, -1.0):
                        g = np.zeros(nv)
                        for j in range(npt):
                            g[idx(k, j, a)] = sgn * Mr[i, j] / T[k] ** r
                        rows.append(g); rhs.append(bound)
    G = np.array(rows); h = np.array(rhs)
    dl = rng.standard_normal(nv)
    return (Q.astype(F32), np.zeros(nv, F32), A.astype(F32), b.astype(F32), G.astype(F32), h.astype(F32),
            dl.astype(F32))


def g_bezier(K: int, batch: int, start: int = 0, stream: int = 200) -> QPBatch:
    """A batch of Bézier trajectory QPs; problem i uses SeedSequence([stream + K, i])."""
    Q0, _, A0, _, G0, _, _ = g_bezier_one(_rng(stream + K, start), K)
    nv, m, p = Q0.shape[0], A0.shape[0], G0.shape[0]
    Qs = np.empty((batch, nv, nv), F32); qs = np.zeros((batch, nv), F32)
    As = np.empty((batch, m, nv), F32); bs = np.empty((batch, m), F32)
    Gs = np.empty((batch, p, nv), F32); hs = np.empty((batch, p), F32)
    dls = np.empty((batch, nv), F32)
    for j in range(batch):
        Q, _, A, b, G, h, dl = g_bezier_one(_rng(stream + K, start + j), K)
        Qs[j], As[j], bs[j], Gs[j], hs[j], dls[j] = Q, A, b, G, h, dl
    return QPBatch(nv, m, p, Qs, qs, As, bs, Gs, hs, dls, batch,
                   meta={"recipe": "g_bezier", "segments": K, "start": start})


# solver settings of the paper's bilevel sweep: solver_tol = 1e-4
WORKLOADS.update({
    "bezier4": dict(name="bezier4_trajectory_n40_m30_p192_B2048", build=lambda B, s: g_bezier(4, B, s), batch=2048,
                    solver=dict(tol=1e-4)),
    "bezier8": dict(name="bezier8_trajectory_n80_m54_p384_B1024", build=lambda B, s: g_bezier(8, B, s), batch=1024,
                    solver=dict(tol=1e-4)),
})
