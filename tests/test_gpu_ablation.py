"""two cells of the App. D.3 ablation harness
(tools/ablation.py) — the paper's claim on this hardware: the implicit f32
arm is NaN-free and tracks the f64 relaxation floor, the standard
f32 arm breaks down with first hits in the predictor / relaxation
(Table 1)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import ablation  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p,m,kappa", [(10, 12, 6, 1e-4), (20, 25, 12, 1e-7)])
def test_ablation_cell(n, p, m, kappa):
    b, gh = ablation.cell_batch(n, p, m)
    tol = min(kappa, 1e-4)
    imp32 = ablation.summarise(ablation.run_gpu_arm(b, "implicit", max(tol, 1e-6), kappa), gh)
    exp32 = ablation.summarise(ablation.run_gpu_arm(b, "explicit", max(tol, 1e-6), kappa), gh)
    imp64 = ablation.summarise(ablation.run_oracle_arm(b, "implicit", tol, kappa), gh)
    assert imp32["failures"] == 0 and imp32["nan_rate"] == 0.0
    assert imp64["failures"] == 0
    # f32 implicit sits on the f64 relaxation floor
    assert abs(imp32["median_grad_err"] / imp64["median_grad_err"] - 1) < 0.05
    # the standard arm breaks down in f32 on these near-active instances
    assert exp32["nan_rate"] > 0.1
    assert set(exp32["stages"]) <= {"predictor", "relax", "corrector", "linesearch", "centering", "scaling"}
