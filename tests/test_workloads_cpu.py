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


@pytest.mark.parametrize("K", [4, 8])
def test_bezier_shapes_structure_feasibility(K):
    """App. E inner QP: x = K·5·2 control points; m = 4 + 6(K−1) + 8
    equalities (endpoints, C² continuity, rest at both ends); p = K(4·5 + 28)
    inequalities (4-facet cells × 5 points, velocity/acceleration polygons);
    Q ⪰ 0 with the translations of each segment in its null space; the
    constraint set is strictly feasible (LP, scipy)."""
    from scipy.optimize import linprog
    b = gen.g_bezier(K, 2)
    assert (b.n, b.m, b.p) == (10 * K, 6 * K + 6, 48 * K)
    Q = b.Q[0].astype(np.float64)
    assert np.allclose(Q, Q.T, atol=1e-6 * np.abs(Q).max())
    assert np.linalg.eigvalsh(Q).min() > -1e-5 * np.abs(Q).max()
    t = np.zeros(b.n); t[0::2] = 1.0                    # translate every control point along x
    assert np.abs(Q @ t).max() < 1e-4 * np.abs(Q).max()
    assert np.linalg.matrix_rank(b.A[0].astype(np.float64)) == b.m
    # strict feasibility: max margin eps s.t. A x = b, G x + eps ≤ h
    A, bb, G, h = (v[0].astype(np.float64) for v in (b.A, b.b, b.G, b.h))
    c = np.zeros(b.n + 1); c[-1] = -1.0
    res = linprog(c, A_ub=np.hstack([G, np.ones((b.p, 1))]), b_ub=h, A_eq=np.hstack([A, np.zeros((b.m, 1))]),
                  b_eq=bb, bounds=[(None, None)] * b.n + [(None, 1.0)], method="highs")
    assert res.status == 0 and -res.fun > 1e-3, res.message


def test_k14_backward_counts_no_factorisation_for_chord_steps():
    """flops.k14_backward (SURVEY §8(d) work model): a chord step of the
    guarded chord relax (reading Q26) reuses the solve's factorisation, so
    each removes exactly N³/3 from the K14-literal count."""
    from paper_2605_17913_b200 import flops as FL
    n, m, p = 50, 10, 100
    N = n + m + p
    base = FL.k14_backward(n, m, p, 4)
    assert abs(FL.k14_backward(n, m, p, 4, chord=3) - (base - 3 * N ** 3 / 3)) <= 1e-6 * base
    assert FL.k14_backward(n, m, p, 4, chord=0) == base
