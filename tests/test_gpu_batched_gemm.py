"""Config-4 residual products as batched GEMMs (bnd_sgemm: Q and G shared by
the batch, so G x, Q x, Gᵀ z, Gᵀ t and G Δx of every problem are GEMMs over
the batch instead of per-problem GEMVs): the same FP32 FMA
arithmetic in another summation order — the oracle bar, and agreement with
the per-problem GEMV path (QPB200_NO_PRE) to ±1 iteration and 1e-4 in x."""
import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen

from .helpers import GRADS, rel_err_rows, run_gpu
from .test_gpu_parity import check_against_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("batch", [16, 130])
def test_batched_gemm_residuals(monkeypatch, batch):
    b = gen.make_config(4, batch=batch)
    g = run_gpu(b)
    assert g["info"]["path"] == 4
    if batch <= 16:
        check_against_oracle(b, g)
    monkeypatch.setenv("QPB200_NO_PRE", "1")
    g0 = run_gpu(b)
    assert np.abs(g["iters"].astype(int) - g0["iters"].astype(int)).max() <= 1
    assert np.abs(g["x"] - g0["x"]).max() <= 1e-4 * max(1.0, np.abs(g0["x"]).max())
    for k in GRADS:
        if g0[k].size:
            rows = 1 if b.shared.get(k[1:], False) else b.batch
            assert rel_err_rows(g[k].reshape(rows, -1), g0[k].reshape(rows, -1)).max() <= 1e-3, k
