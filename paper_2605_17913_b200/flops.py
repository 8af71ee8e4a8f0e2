"""Algorithmic work model of the hot path.

Counts are ALGORITHMIC: they use the unpadded KKT dimension N = n + p + m of
the bounded system (Eq. 14) and standard dense-kernel counts,
independent of how the kernels block or pad.  2 flops per multiply-add.

Per Newton iteration / factorisation (one problem):
  factorisation   N³/3                     (Cholesky-class LDLᵀ of Eq. 14)
  assembly        p·n·(n+1)                (Gᵀ D G, symmetric half)
  solve           2·N²                     (forward + backward substitution)
  residuals       2n² + 6pn + 4mn          (Qx, Gx, Gᵀz, Gᵀ(r_z+c r_κ), Ax, Aᵀy; Eq. 4, Eq. 10)
  step            2pn                      (Δv = GΔx + w)
The CVXOPT initialisation is one factorisation + assembly + solve.  The
backward adds, per relax iteration, the same iteration cost (factor-then-check
runs one more factorisation than steps) plus the adjoint solve 2N² + 2pn.

Algorithmic HBM bytes per problem (one solve + backward, each input read
once, each output written once): 4·(|Q|+|q|+|A|+|b|+|G|+|h|)·2 (read by both
kernels) + 4·(outputs: x,s,z,y + gradients of the same size as the data + ∇ₓℓ).
"""
from __future__ import annotations


def per_iteration(n: int, m: int, p: int) -> float:
    N = n + p + m
    return N ** 3 / 3 + p * n * (n + 1) + 2 * N ** 2 + (2 * n * n + 6 * p * n + 4 * m * n) + 2 * p * n


def init_flops(n: int, m: int, p: int) -> float:
    N = n + p + m
    return N ** 3 / 3 + p * n * (n + 1) + 2 * N ** 2 + 2 * p * n


def solve_flops(n, m, p, iters) -> float:
    """Flops of qp_solve_batched for one problem that took `iters` Newton steps
    (the last residual check does not factor)."""
    N = n + p + m
    resid = 2 * n * n + 6 * p * n + 4 * m * n
    return init_flops(n, m, p) + iters * per_iteration(n, m, p) + resid


def backward_flops(n, m, p, relax_iters) -> float:
    """Flops of qp_backward_batched for one problem: (relax_iters + 1)
    factorisations (factor-then-check), relax_iters solves/steps, adjoint solve."""
    N = n + p + m
    fac = N ** 3 / 3 + p * n * (n + 1) + (2 * n * n + 6 * p * n + 4 * m * n)
    step = 2 * N ** 2 + 2 * p * n
    return (relax_iters + 1) * fac + relax_iters * step + 2 * N ** 2 + 2 * p * n + 2 * (n * n + m * n + p * n)


# ---------------------------------------------------------------------------
# SURVEY.md §8(d) work model ("K14-literal"): the paper's own system, Eq. 14
# (P:292-307), of dimension N = n + p + m factored every iteration, its
# constant (1,1) block Q − GᵀG formed once per problem, so per Newton
# iteration N³/3 (factorisation) + 2N² (two triangular solves) + 2n² + 6pn +
# 4mn (the residual GEMVs of Eq. 4 / Eq. 10), and once per unit p·n².  These
# are the flops `roofline.frac` is quoted on; what the kernels execute (the
# smaller sign(v)-partitioned system of reading Q12b plus its assembly) is
# reported beside it as `frac_exec`.
# ---------------------------------------------------------------------------
def k14_iteration(n: int, m: int, p: int) -> float:
    N = n + p + m
    return N ** 3 / 3 + 2 * N ** 2 + (2 * n * n + 6 * p * n + 4 * m * n)


def k14_solve(n: int, m: int, p: int, iters) -> float:
    """qp_solve_batched, one problem with `iters` Newton steps: the CVXOPT
    initialisation (one factorisation + solve of an N-dimensional system,
    P:394), p·n² for Q − GᵀG, `iters` iterations, and the final residual
    evaluation that certifies convergence."""
    N = n + p + m
    return (N ** 3 / 3 + 2 * N ** 2) + p * n * n + iters * k14_iteration(n, m, p) + \
        (2 * n * n + 6 * p * n + 4 * m * n)


def k14_backward(n: int, m: int, p: int, relax_iters, chord: float = 0) -> float:
    """qp_backward_batched, one problem: Alg. 2 with `relax_iters` steps
    (relax_iters + 1 residual evaluations; factor-then-check, reading Q6: one
    factorisation per evaluation except for the `chord` steps of the guarded
    chord relax, reading Q26, which reuse the solve's), the Alg. 3 adjoint
    solve 2N², and the outer products of the gradients 2(n² + mn + pn)."""
    N = n + p + m
    resid = 2 * n * n + 6 * p * n + 4 * m * n
    return (relax_iters + 1) * resid + (relax_iters + 1 - chord) * N ** 3 / 3 + relax_iters * 2 * N ** 2 + \
        2 * N ** 2 + 2 * (n * n + m * n + p * n)


def data_bytes(n, m, p, shared=()) -> tuple[int, int]:
    """(per-problem bytes, shared bytes) of the six data fields."""
    sizes = {"Q": n * n, "q": n, "A": m * n, "b": m, "G": p * n, "h": p}
    per = sum(4 * v for k, v in sizes.items() if k not in shared)
    sh = sum(4 * v for k, v in sizes.items() if k in shared)
    return per, sh


def fp32_peak_tflops(sm_count: int = 148, sm_mhz: float = 1965.0) -> float:
    """FP32 FMA peak: SMs × 128 FP32 lanes × 2 flops × clock (B200_PROFILING.md
    / B300_MICROARCH.md unit counts; 148 SMs, 1965 MHz max clock)."""
    return sm_count * 128 * 2 * sm_mhz * 1e6 / 1e12
