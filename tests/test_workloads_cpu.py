"""Generator checks for the N4 workloads (no GPU): shapes and row counts of
P:1212-1216, strict feasibility of u = 0 (every barrier h > 0, the box), and
the structure of the CBF rows (obstacle rows touch one agent, pair rows two,
with opposite gradients)."""
import numpy as np
import pytest

from paper_2605_17913_b200 import generators as gen


@pytest.mark.parametrize("agents,p", [(7, 70), (9, 99)])
def test_cbf_shapes_and_feasibility(agents, p):
    b = gen.g_cbf(agents, 16)
    assert (b.n, b.m, b.p) == (2 * agents, 0, p)
    assert np.all(b.h > 0)                              # u = 0 strictly feasible
    assert np.array_equal(b.Q[0], np.eye(2 * agents, dtype=np.float32))
    G = b.G[0]
    no = 3 * agents
    npair = agents * (agents - 1) // 2
    nz = (G != 0).sum(1)
    assert np.all(nz[:no] <= 2) and np.all(nz[no:no + npair] <= 4) and np.all(nz[no + npair:] == 1)
    for r in range(no, no + npair):                     # ∇_{p_i} h = −∇_{p_j} h
        cols = np.flatnonzero(G[r])
        v = G[r, cols].reshape(2, 2) if cols.size == 4 else None
        if v is not None:
            assert np.allclose(v[0], -v[1])
    assert np.allclose(b.h[:, no + npair:], 2.0)       # u_max


def test_cbf_deterministic_and_sliced():
    a = gen.make_workload("cbf7", batch=6)
    b = gen.make_workload("cbf7", batch=3, start=3)
    assert np.array_equal(a.G[3:], b.G) and np.array_equal(a.q[3:], b.q)
