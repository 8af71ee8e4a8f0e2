"""The TMA-fed Schur update of the batched engine (bnd_tc_update_tma, opt-in
with QPB200_TC_TMA: persistent, warp-specialised, operands staged by
cp.async.bulk.tensor into 128-byte-swizzled tiles through per-16-row-block
tensor maps, split for 3×TF32 in shared memory, MMAs on SWIZZLE_128B
descriptors): the same Newton arithmetic as the register-staged kernel, so
the oracle bar and ±1 iteration agreement with it."""
import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen

from .helpers import GRADS, rel_err_rows, run_gpu
from .test_gpu_parity import check_against_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", ["42", "22"])
@pytest.mark.parametrize("case", ["cfg4", "per_problem"])
def test_tma_schur_update(monkeypatch, variant, case):
    b = gen.make_config(4, batch=16) if case == "cfg4" else gen.g_rand(13, 8, 130, 4, 200)
    g0 = run_gpu(b)
    monkeypatch.setenv("QPB200_TC_TMA", variant)
    g = run_gpu(b)
    assert g["info"]["path"] == 4
    check_against_oracle(b, g)
    assert np.abs(g["iters"].astype(int) - g0["iters"].astype(int)).max() <= 1
    assert np.abs(g["x"] - g0["x"]).max() <= 1e-4 * max(1.0, np.abs(g0["x"]).max())
    for k in GRADS:
        if g0[k].size:
            rows = 1 if b.shared.get(k[1:], False) else b.batch
            assert rel_err_rows(g[k].reshape(rows, -1), g0[k].reshape(rows, -1)).max() <= 1e-3, k
