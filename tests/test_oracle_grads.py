"""Pins of the oracle's Alg. 2 (relax) and Alg. 3 (gradients): closed forms,
the printed example, central finite differences of the relaxed map, the
kappa_relax -> 0 hard-Jacobian limit (App. D.2) and explicit/implicit
agreement."""
import json
import os

import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen
from paper_2605_17913_b200.generators import QPBatch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
FIELDS = ("dQ", "dq", "dA", "db", "dG", "dh")


def one(prob, dl):
    n = prob["Q"].shape[0]
    A = np.asarray(prob["A"], float).reshape(-1, n); G = np.asarray(prob["G"], float).reshape(-1, n)
    return QPBatch(n, A.shape[0], G.shape[0], np.asarray(prob["Q"], float)[None],
                   np.asarray(prob["q"], float)[None], A[None], np.asarray(prob["b"], float).reshape(1, -1),
                   G[None], np.asarray(prob["h"], float).reshape(1, -1), np.asarray(dl, float)[None], 1)


def relaxed_x(orc, bt, cfg):
    r = orc.solve(bt, cfg, "f64")
    g = orc.backward(bt, r, cfg, "f64")
    assert g["status"][0] == 0
    return g["relaxed"]["x"][0], g


def test_printed_unconstrained_gradient(orc):
    ex = GOLD["gradient"][0]
    bt = one(dict(Q=np.array(ex["Q"]), q=np.array(ex["q"]), A=np.zeros((0, 2)), b=np.zeros(0),
                  G=np.zeros((0, 2)), h=np.zeros(0)), ex["dl_dx"])
    _, g = relaxed_x(orc, bt, orc.Cfg.f64())
    assert np.allclose(g["dq"][0], ex["dq"], atol=1e-14), ex["cite"]


@pytest.mark.parametrize("qv,hv", [(-3.0, 1.0), (0.5, 1.0), (-1.05, 1.0)])
def test_box_1d_central_path_closed_form(orc, qv, hv):
    """min x^2/2 + qx s.t. x <= h.  The central path at kappa has the closed
    form s = ((h+q) + sqrt((h+q)^2 + 4 kappa))/2, z = kappa/s, x = h - s, and
    its derivatives are dx/dh = z/(z+s), dx/dq = -s/(z+s) (DESIGN.md App. A.1)."""
    kr = 1e-2
    cfg = orc.Cfg.f64(kappa_relax=kr)
    bt = one(dict(Q=np.array([[1.0]]), q=np.array([qv]), A=np.zeros((0, 1)), b=np.zeros(0),
                  G=np.array([[1.0]]), h=np.array([hv])), [1.0])
    x, g = relaxed_x(orc, bt, cfg)
    s = ((hv + qv) + np.sqrt((hv + qv) ** 2 + 4 * kr)) / 2
    z = kr / s
    assert x[0] == pytest.approx(hv - s, abs=1e-10)
    assert g["relaxed"]["z"][0][0] == pytest.approx(z, rel=1e-8)
    assert g["dh"][0][0] == pytest.approx(z / (z + s), rel=1e-8)
    assert g["dq"][0][0] == pytest.approx(-s / (z + s), rel=1e-8)
    assert g["dQ"][0][0, 0] == pytest.approx(g["dq"][0][0] * x[0], rel=1e-8)     # sym(dx x')
    assert g["dG"][0][0, 0] == pytest.approx(-g["dh"][0][0] * x[0] + z * g["dq"][0][0], rel=1e-8)


@pytest.mark.parametrize("seed", range(6))
def test_finite_differences_all_fields(orc, seed):
    """Central FD of l(theta) = grad_x l . x_relax(theta) in f64, h = 1e-6,
    full re-solve + re-relax per perturbation, relative 1e-4.
    Q is perturbed symmetrically (reading Q19)."""
    n, m, p = 5, 1, 4
    kr = 1e-2
    cfg = orc.Cfg.f64(kappa_relax=kr, relax_ktol=1e-12, tol=1e-12)
    b = gen.g_rand(98, 1, n, m, p, start=seed)
    prob = {k: v.astype(float) for k, v in b.problem(0).items()}
    prob["q"] = prob["q"] * 3  # push some constraints toward activity
    dl = prob.pop("dl_dx")
    _, g = relaxed_x(orc, one(prob, dl), cfg)
    eps = 1e-6

    def loss(pr):
        xr, _ = relaxed_x(orc, one(pr, dl), cfg)
        return float(dl @ xr)

    for field, gf in (("q", "dq"), ("b", "db"), ("h", "dh"), ("A", "dA"), ("G", "dG"), ("Q", "dQ")):
        base = prob[field]
        fd = np.zeros_like(base)
        for idx in np.ndindex(base.shape):
            if field == "Q" and idx[0] > idx[1]:
                continue
            pp = {k: v.copy() for k, v in prob.items()}; pm = {k: v.copy() for k, v in prob.items()}
            pp[field][idx] += eps; pm[field][idx] -= eps
            if field == "Q" and idx[0] != idx[1]:
                pp[field][idx[::-1]] += eps; pm[field][idx[::-1]] -= eps
            fd[idx] = (loss(pp) - loss(pm)) / (2 * eps)
        an = g[gf][0].copy()
        if field == "Q":  # compare the symmetric-pair derivative dQ_ij + dQ_ji
            an = np.where(np.eye(n, dtype=bool), an, an + an.T)
            mask = np.tril(np.ones((n, n), bool))
            an, fd = an[mask], fd.T[mask]
        err = np.linalg.norm(an - fd) / max(np.linalg.norm(fd), 1e-12)
        assert err <= 1e-4, (field, err)


def test_hard_jacobian_limit(orc):
    """As kappa_relax -> 0 the gradient w.r.t. the query point, -grad_q,
    tends to J_hard v = (I - G_A'(G_A G_A')^{-1} G_A) v (App. D.2),
    with an error that shrinks with kappa_relax (the relaxation floor)."""
    rng = gen._rng(55, 1)
    Q, q, A, b, G, h, probe, y0, act = gen.g_proj_one(rng, 8, 10, 4, 1.0, margin_lo=0.2)
    prob = dict(Q=Q.astype(float), q=q.astype(float), A=np.zeros((0, 8)), b=np.zeros(0), G=G.astype(float),
                h=h.astype(float))
    GA = prob["G"][act]
    Jh = np.eye(8) - GA.T @ np.linalg.solve(GA @ GA.T, GA)
    assert np.allclose(Jh @ Jh, Jh, atol=1e-10) and np.allclose(Jh, Jh.T, atol=1e-12)
    gh = Jh @ probe.astype(float)
    errs = []
    for kr in (1e-2, 1e-4, 1e-6, 1e-8):
        _, g = relaxed_x(orc, one(prob, probe), orc.Cfg.f64(kappa_relax=kr))
        gx = -g["dq"][0]
        errs.append(np.linalg.norm(gx - gh) / np.linalg.norm(gh))
    assert errs[-1] <= 1e-5
    assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:]))


def test_explicit_and_implicit_gradients_agree_f64(orc):
    """Both paradigms differentiate the same relaxed central-path map:
    gradients agree to 1e-6 relative in f64."""
    b = gen.make_config(2, batch=4)
    ci, ce = orc.Cfg.f64(), orc.Cfg.f64(formulation=orc.FORM_EXPLICIT)
    gi = orc.backward(b, orc.solve(b, ci, "f64"), ci, "f64")
    ge = orc.backward(b, orc.solve(b, ce, "f64"), ce, "f64")
    assert np.all(gi["status"] == 0) and np.all(ge["status"] == 0)
    for k in FIELDS:
        a, r = ge[k].reshape(4, -1), gi[k].reshape(4, -1)
        err = np.linalg.norm(a - r, axis=1) / np.maximum(np.linalg.norm(r, axis=1), 1e-30)
        assert err.max() <= 1e-6, (k, err.max())


def test_zero_cotangent_zero_gradients(orc):
    b = gen.make_config(1, batch=2)
    r = orc.solve(b, orc.Cfg.f64(), "f64")
    g = orc.backward(b, r, orc.Cfg.f64(), "f64", dl_dx=np.zeros_like(b.dl_dx))
    assert all(np.abs(g[k]).max() == 0 for k in FIELDS if g[k].size)


def test_relax_reaches_kappa_relax(orc):
    """Alg. 2 ends on the central path at kappa_relax: z_i s_i = kappa_relax
     and the feasibility residuals are below tol."""
    b = gen.make_config(2, batch=4)
    for prec, cfg, rel in (("f64", orc.Cfg.f64(), 1e-8), ("f32", orc.Cfg.f32(), 1e-3)):
        r = orc.solve(b, cfg, prec)
        g = orc.backward(b, r, cfg, prec)
        assert np.all(g["status"] == 0)
        zs = g["relaxed"]["z"].astype(float) * g["relaxed"]["s"].astype(float)
        assert np.all(np.abs(zs / cfg.kappa_relax - 1) <= rel)
        assert np.all(g["relax_iters"] >= 1)


def test_chord_relax_same_relaxed_map_f64(orc):
    """N2(i) evaluation harness (relax_mode=1: Alg. 2 steps with the Alg. 1
    factorisation nearest kappa_relax, final factorisation at the
    relaxed point for Alg. 3): the relaxed point is the unique central-path
    point at kappa_relax, so the gradients equal the exact-Newton relax's to
    1e-7 in f64 wherever the chord iteration converges."""
    b = gen.make_config(2, batch=8)
    c0, c1 = orc.Cfg.f64(), orc.Cfg.f64(relax_mode=1)
    r = orc.solve(b, c0, "f64")
    g0, g1 = orc.backward(b, r, c0, "f64"), orc.backward(b, r, c1, "f64")
    ok = g1["status"] == 0
    assert np.all(g0["status"] == 0) and ok.sum() >= 6
    for k in FIELDS:
        a, ref = g1[k].reshape(8, -1)[ok], g0[k].reshape(8, -1)[ok]
        err = np.linalg.norm(a - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
        assert err.max() <= 1e-7, (k, err.max())
