"""the paper's application shapes as synthetic batches —
the centralised CBF safety-filter QP (App. F) for 7
agents (14 variables, 70 constraints, the paper's nominal setting) and 9
agents (18 variables, 99 constraints by P:1214's formula) — against the oracle
with the same bar as the BASELINE configs (tests/helpers.py)."""
import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen

from .helpers import run_gpu
from .test_gpu_parity import check_against_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,B", [("cbf7", 128), ("cbf9", 96)])
def test_safety_filter_shapes(name, B):
    b = gen.make_workload(name, batch=B)
    g = run_gpu(b)
    st = check_against_oracle(b, g)
    assert st["iters_equal"] >= 0.5


@pytest.mark.parametrize("mem", ["device", "host"])
def test_safety_filter_full_batch_sampled(mem):
    """cbf7 at its default batch (4096; host mode runs the 4-chunk pipeline):
    24 sampled problems checked one by one against the oracle."""
    b = gen.make_workload("cbf7")
    g = run_gpu(b, mem=mem)
    assert np.all(g["status"] == 0)
    idx = np.linspace(0, b.batch - 1, 24).astype(int)
    sub = b.subset(idx)
    gs = {k: (v[idx] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == b.batch else v)
          for k, v in g.items()}
    check_against_oracle(sub, gs)
