"""paper_2605_17913_b200 — B200-native (sm_100a) batched f32 interior-point QP
solver with implicit, spectrally bounded complementarity and its
relaxation-based implicit-differentiation backward pass (arxiv 2605.17913).

Layout:
  csrc/         CUDA kernels (persistent CTA-per-QP IPM) and the C-ABI host library
  capi.py       ctypes binding of include/qpb200.h (same names)
  solver.py     torch-facing QPSolver / QPFunction
  dist.py       batch sharding + shared-gradient all-reduce (torch.distributed)
  generators.py seeded synthetic workloads (no solver arithmetic)

Importing the package does not load the CUDA library; the first solver call
does, and raises if it is missing (there is no CPU fallback)."""

__all__ = ["QPSolver", "QPFunction", "solve"]


def __getattr__(name):
    if name in __all__:
        from . import solver
        return getattr(solver, name)
    raise AttributeError(name)
