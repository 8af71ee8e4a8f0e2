"""Oracle pins of the guarded chord relax (relax_mode 2, reading Q26;
SURVEY §8(f) N2(i)).  The relaxed point is the unique
central-path point at κ_relax, so whichever linear solves reach
it, Alg. 3's gradients there are the same map; these tests pin that and the
guard's two limits against exact Newton (reading Q6)."""
import numpy as np
import pytest

import oracle as O
from paper_2605_17913_b200 import generators as gen

from .helpers import GRADS


@pytest.fixture(scope="module")
def cfg2():
    b = gen.make_config(2, batch=8)
    return b, O.solve(b, O.Cfg.f64(), "f64")


def test_guarded_chord_same_relaxed_map_f64(cfg2):
    b, r = cfg2
    g0 = O.backward(b, r, O.Cfg.f64(), "f64")
    g2 = O.backward(b, r, O.Cfg.f64(relax_mode=2), "f64")
    assert np.all(g0["status"] == 0) and np.all(g2["status"] == 0)
    for k in GRADS:
        a, ref = g2[k].reshape(8, -1), g0[k].reshape(8, -1)
        err = np.linalg.norm(a - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
        assert err.max() <= 1e-7, (k, err.max())
    for k in ("x", "y", "z", "s"):  # the relaxed point itself
        assert np.abs(g2["relaxed"][k] - g0["relaxed"][k]).max() <= 1e-7 * max(1.0, np.abs(g0["relaxed"][k]).max())


def test_chord_max_zero_is_exact_newton(cfg2):
    """chord_max = 0 leaves chord mode before any chord step: bitwise exact Newton."""
    b, r = cfg2
    g0 = O.backward(b, r, O.Cfg.f64(), "f64")
    g1 = O.backward(b, r, O.Cfg.f64(relax_mode=2, chord_max=0), "f64")
    for k in GRADS + ("relax_iters", "status"):
        assert np.array_equal(g0[k], g1[k]), k


def test_chord_needs_more_steps_but_fewer_factorisations_f32():
    """Linear (chord) instead of quadratic (Newton) convergence: at least as
    many relax steps, the same relaxed map at the f32 bar."""
    b = gen.make_config(2, batch=16)
    c0, c2 = O.Cfg.f32(), O.Cfg.f32(relax_mode=2)
    r = O.solve(b, c0, "f32")
    g0, g2 = O.backward(b, r, c0, "f32"), O.backward(b, r, c2, "f32")
    assert np.all(g2["status"] == 0)
    assert g2["relax_iters"].mean() >= g0["relax_iters"].mean()
    for k in GRADS:
        a, ref = g2[k].reshape(16, -1), g0[k].reshape(16, -1)
        err = np.linalg.norm(a - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
        assert err.max() <= 1e-3, (k, err.max())
