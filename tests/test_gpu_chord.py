"""Guarded chord relax (reading Q26: Alg. 2 reuses the
factorisation Alg. 1 computed nearest κ_relax — "the matrix factorizations K̃
computed during the forward solve ... can be heavily reused"; "if K̃
not cached", P:513 — while its steps contract, then exact Newton).  The
relaxed point is the unique central-path point at κ_relax, so the gradients
are held to the same north-star bar against the f64 oracle (exact-Newton
relax), with the f32 oracle in the same relax mode as the precision-limit
reference; the solve is untouched by the mode."""
import numpy as np
import pytest

import oracle as O
from paper_2605_17913_b200 import generators as gen

from .helpers import GRADS, rel_err_rows, run_gpu
from .test_gpu_parity import check_against_oracle

pytestmark = pytest.mark.gpu

CHORD = dict(relax_mode=2)


def _relax_stats(g, r32_chord):
    d = np.abs(g["relax_iters"].astype(int) - r32_chord["relax_iters"].astype(int))
    return d


@pytest.mark.parametrize("chunk", [None, 5])
def test_chord_cfg4_subset(monkeypatch, chunk):
    """Config-4 shapes (shared Q, G, h: the kr_gemm assembly) on the batched
    engine, one chunk and (QPB200_BCHUNK=5) ragged chunks whose caches must
    survive the later chunks of the solve."""
    if chunk:
        monkeypatch.setenv("QPB200_BCHUNK", str(chunk))
    b = gen.make_config(4, batch=16)
    g = run_gpu(b, **CHORD)
    assert g["info"]["path"] == 4 and g["info"]["relax_mode"] == 2
    assert g["info"]["chord_steps"] > 0
    c32 = O.Cfg.f32(relax_mode=2)
    check_against_oracle(b, g, cfg32=c32)
    gn = run_gpu(b, relax_mode=0)  # exact-Newton relax: the solve is bitwise the same, the gradients agree
    for k in ("x", "s", "z", "y", "iters", "status"):
        assert np.array_equal(g[k], gn[k]), k
    for k in GRADS:
        if gn[k].size:
            rows = 1 if b.shared.get(k[1:], False) else b.batch
            assert rel_err_rows(g[k].reshape(rows, -1), gn[k].reshape(rows, -1)).max() <= 1e-3, k
    r32 = O.solve(b, c32, "f32")
    b32 = O.backward(b, r32, c32, "f32")
    d = _relax_stats(g, b32)
    print("relax iters GPU", g["relax_iters"].tolist(), "f32 oracle (chord)", b32["relax_iters"].tolist())
    assert np.mean(d <= 1) >= 0.75


def test_chord_per_problem_data():
    """Per-problem G (the tcgen05 bnd_assemble tiles), n=130, m=4, p=200."""
    b = gen.g_rand(13, 8, 130, 4, 200)
    g = run_gpu(b, **CHORD)
    assert g["info"]["path"] == 4 and g["info"]["chord_steps"] > 0
    check_against_oracle(b, g, cfg32=O.Cfg.f32(relax_mode=2))


def test_chord_max_zero_is_newton():
    """chord_max = 0: the guard leaves chord mode before the first step, so
    the backward is exact Newton — bitwise the relax_mode = 0 result."""
    b = gen.make_config(4, batch=8)
    g0 = run_gpu(b, relax_mode=0)
    g1 = run_gpu(b, relax_mode=2, chord_max=0)
    assert g1["info"]["chord_steps"] == 0
    for k in GRADS + ("relax_iters", "grad_status"):
        assert np.array_equal(g0[k], g1[k]), k


def test_chord_strict_guard_falls_back():
    """chord_rho tiny: every chord step after the first fails the contraction
    test, so each problem takes at most 1-2 chord steps and finishes with
    exact Newton — still at the oracle bar."""
    b = gen.make_config(4, batch=8)
    g = run_gpu(b, relax_mode=2, chord_rho=1e-6)
    assert 0 < g["info"]["chord_steps"] <= 2 * 8
    check_against_oracle(b, g, cfg32=O.Cfg.f32(relax_mode=2, chord_rho=1e-6))


# ---------------------------------------------------------------------------
# path 1 (one persistent CTA per QP, KKT in shared memory): the solve copies
# its factor to the cache, a chord step copies it back into the KKT buffer
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,batch", [(1, 16), (2, 96), (3, 48)])
def test_chord_path1(cfg, batch):
    b = gen.make_config(cfg, batch=batch)
    g = run_gpu(b, **CHORD)
    assert g["info"]["path"] == 1 and g["info"]["relax_mode"] == 2
    assert g["info"]["chord_steps"] > 0
    check_against_oracle(b, g, cfg32=O.Cfg.f32(relax_mode=2))
    gn = run_gpu(b, relax_mode=0)
    for k in ("x", "s", "z", "y", "iters", "status"):
        assert np.array_equal(g[k], gn[k]), k
    assert gn["info"]["relax_mode"] == 0 and gn["info"]["chord_steps"] == 0


def test_chord_path1_max_zero_is_newton():
    b = gen.make_config(2, batch=64)
    g0 = run_gpu(b, relax_mode=0)
    g1 = run_gpu(b, relax_mode=2, chord_max=0)
    assert g1["info"]["chord_steps"] == 0
    for k in GRADS + ("relax_iters", "grad_status"):
        assert np.array_equal(g0[k], g1[k]), k


@pytest.mark.parametrize("mem", ["host", "host_async"])
def test_chord_path1_host_modes(mem):
    """Host-buffer modes (8 chunk streams; host_async: each backward chunk
    follows its solve chunk on its stream, with the programmatic backward
    launch): the same results as device mode."""
    b = gen.make_config(2, batch=301)
    gd = run_gpu(b, **CHORD)
    gh = run_gpu(b, mem=mem, **CHORD)
    for k in ("x", "iters") + GRADS + ("relax_iters",):
        assert np.array_equal(gd[k], gh[k]), k
