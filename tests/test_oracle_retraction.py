"""Pins of the oracle's retraction map (Eq. 9, 11, 12; App. C) against the
paper's identities, printed examples and an extended-precision evaluation."""
import json
import os
from decimal import Decimal, getcontext

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))

V = np.concatenate([-np.logspace(-8, 8, 41), np.logspace(-8, 8, 41), [0.0]])
KAPPAS = [1e-9, 1e-6, 1e-4, 1e-2, 1.0]


@pytest.mark.parametrize("kappa", KAPPAS)
def test_product_identity_eq9(orc, kappa):
    """b(v) b(-v) = kappa (Eq. 9); S:528 tolerances."""
    for prec, tol in (("f64", 1e-12), ("f32", 1e-5)):
        r = orc.retract(V, kappa, prec)
        prod = r["z"].astype(np.float64) * r["s"].astype(np.float64)
        kap = float(np.float32(kappa)) if prec == "f32" else kappa
        assert np.max(np.abs(prod - kap) / kap) <= tol, prec


@pytest.mark.parametrize("kappa", KAPPAS)
def test_derivative_properties_eq11(orc, kappa):
    """d+ + d- = 1 (Eq. 11a) within 4 ulp; 0 < d <= 1 (Eq. 11b)."""
    for prec in ("f64", "f32"):
        r = orc.retract(V, kappa, prec)
        eps = np.finfo(np.float64 if prec == "f64" else np.float32).eps
        s = r["dp"].astype(np.float64) + r["dm"].astype(np.float64)
        assert np.max(np.abs(s - 1.0)) <= 4 * eps
        assert np.all(r["dp"] > 0) and np.all(r["dp"] <= 1)
        assert np.all(r["dm"] > 0) and np.all(r["dm"] <= 1)


def test_coordinate_identity(orc):
    """b(v) - b(-v) = v: the algebraic consequence of Eq. 12 behind Alg. 1's
    v <- z - s."""
    for kappa in KAPPAS:
        r = orc.retract(V, kappa, "f64")
        d = r["z"] - r["s"]
        assert np.all(np.abs(d - V) <= 4 * np.finfo(float).eps * np.maximum(np.abs(V), np.sqrt(kappa)))


def test_printed_examples(orc):
    for ex in GOLD["retraction"]:
        r = orc.retract([ex["v"]], ex["kappa"], "f64")
        for k in ("z", "s", "dp", "dm", "c"):
            if k in ex:
                assert r[k][0] == pytest.approx(ex[k], rel=1e-15), (ex["cite"], k)


def _b_decimal(v, kappa):
    getcontext().prec = 60
    v, kappa = Decimal(v), Decimal(kappa)
    return (v + (v * v + 4 * kappa).sqrt()) / 2


def test_cancellation_witness_app_c(orc):
    """v = -1e6, kappa = 1: App. C branch matches a 60-digit evaluation of
    Eq. 12; the naive one-branch formula fails in f32."""
    exact = float(_b_decimal(-1e6, 1.0))
    for prec, tol in (("f64", 1e-12), ("f32", 1e-5)):
        z = float(orc.retract([-1e6], 1.0, prec)["z"][0])
        assert abs(z - exact) / exact <= tol, prec
    v = np.float32(-1e6)
    naive = (v + np.sqrt(v * v + np.float32(4))) / np.float32(2)
    assert abs(float(naive) - exact) / exact > 1e-2  # catastrophic cancellation


def test_derivatives_vs_finite_differences(orc):
    """App. C derivative and c = d b / d kappa (Q10) vs central differences
    of Eq. 12 in f64, away from the cancellation regime."""
    v = np.linspace(-3, 3, 25)
    for kappa in (1e-2, 1e-1, 1.0):
        h = 1e-6
        r = orc.retract(v, kappa, "f64")
        zp, zm = orc.retract(v + h, kappa, "f64")["z"], orc.retract(v - h, kappa, "f64")["z"]
        assert np.allclose(r["dp"], (zp - zm) / (2 * h), rtol=1e-6, atol=1e-9)
        kp, km = orc.retract(v, kappa + h, "f64")["z"], orc.retract(v, kappa - h, "f64")["z"]
        assert np.allclose(r["c"], (kp - km) / (2 * h), rtol=1e-6, atol=1e-9)


def test_on_manifold_closed_forms(orc):
    """On z = b(v), s = b(-v): d+ = z/(z+s), d- = s/(z+s), c = 1/(z+s)
    (DESIGN.md App. A.1 / SURVEY App. A.1)."""
    for kappa in KAPPAS:
        r = orc.retract(V, kappa, "f64")
        zs = r["z"] + r["s"]
        assert np.allclose(r["dp"], r["z"] / zs, rtol=1e-12, atol=0)
        assert np.allclose(r["dm"], r["s"] / zs, rtol=1e-12, atol=0)
        assert np.allclose(r["c"], 1.0 / zs, rtol=1e-12, atol=0)


def test_monotone(orc):
    r = orc.retract(np.sort(V), 1e-4, "f64")
    assert np.all(np.diff(r["z"]) >= 0)
