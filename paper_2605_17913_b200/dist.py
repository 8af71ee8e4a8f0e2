"""Multi-GPU plumbing: one process per GPU (torchrun), the batch sharded by
rank with no data-path collective, and ONE all-reduce (sum) for gradients of
parameters shared across the batch (end-to-end learning, BASELINE config 4;
SURVEY.md §8(e)).  Problems are independent, so per-problem outputs do not
depend on the sharding."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

SHARED_GRADS = {"Q": "dQ", "q": "dq", "A": "dA", "b": "db", "G": "dG", "h": "dh"}


def env_rank() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str | None = None) -> tuple[int, int, int]:
    rank, world, local = env_rank()
    if world > 1 and not dist.is_initialized():
        # QPB200_DIST_BACKEND=gloo: plumbing checks with several ranks on one GPU
        # (the ranks' kernels never wait on each other; NCCL refuses shared devices)
        be = backend or os.environ.get("QPB200_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if be == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(be, init_method="env://")
    return rank, world, local


def shard(batch_size: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [start, stop) of a global batch for `rank`."""
    base, rem = divmod(batch_size, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def allreduce_shared_grads(grads: dict, shared) -> None:
    """Sum the batch-summed gradients of shared fields over ranks, in place,
    with a single flat all-reduce."""
    names = [SHARED_GRADS[f] for f in ("Q", "q", "A", "b", "G", "h") if f in shared and SHARED_GRADS[f] in grads]
    if not names or not dist.is_initialized() or dist.get_world_size() == 1:
        return
    flat = torch.cat([grads[k].reshape(-1) for k in names])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    off = 0
    for k in names:
        nel = grads[k].numel()
        grads[k].copy_(flat[off:off + nel].view_as(grads[k]))
        off += nel


def max_over_ranks(x: float, device=None) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_initialized():
        dist.barrier()
