"""Multi-process (world_size 2, gloo on 127.0.0.1) checks of the host-side
multi-GPU logic in paper_2605_17913_b200/dist.py: batch sharding, the single
flat all-reduce of shared-parameter gradients (config 4), max-over-ranks
timing.  The data-path kernels are single-GPU; this covers the plumbing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_17913_b200 import dist as D
from paper_2605_17913_b200 import generators as gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        r, w, _ = D.init(backend="gloo")
        assert (r, w) == (rank, world)
        # shared gradients of config-4 shape, rank-dependent values
        g = {"dQ": torch.full((3, 3), float(rank + 1)), "dG": torch.arange(6.0).reshape(2, 3) * (rank + 1),
             "dh": torch.ones(2) * (rank + 1), "dq": torch.ones(4) * 7.0}
        D.allreduce_shared_grads(g, shared={"Q", "G", "h"})
        tmax = D.max_over_ranks(float(rank) * 10.0 + 1.0)
        # each rank regenerates its own slice of the global batch
        start, stop = D.shard(10, rank, world)
        b = gen.make_config(4, batch=stop - start, start=start)
        q.put((rank, g["dQ"].numpy().copy(), g["dG"].numpy().copy(), g["dh"].numpy().copy(), g["dq"].numpy().copy(),
               tmax, (start, stop), b.q.copy()))
        D.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(("error", repr(e)))


def test_two_rank_allreduce_and_sharding():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    assert all(r[0] != "error" for r in res), res
    res.sort(key=lambda r: r[0])
    for rank, dQ, dG, dh, dq, tmax, sl, qb in res:
        assert np.allclose(dQ, 3.0)                       # 1 + 2
        assert np.allclose(dG, np.arange(6.0).reshape(2, 3) * 3)
        assert np.allclose(dh, 3.0)
        assert np.allclose(dq, 7.0)                       # not shared: untouched
        assert tmax == 11.0
    assert res[0][6] == (0, 5) and res[1][6] == (5, 10)
    # the ranks' problems are the global batch's problems (seed streams [c, 1+i])
    full = gen.make_config(4, batch=10)
    assert np.array_equal(np.concatenate([res[0][7], res[1][7]]), full.q)


@pytest.mark.parametrize("B,world", [(10, 3), (1024, 8), (7, 8)])
def test_shard_partitions(B, world):
    sl = [D.shard(B, r, world) for r in range(world)]
    assert sl[0][0] == 0 and sl[-1][1] == B
    assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
    sizes = [b - a for a, b in sl]
    assert max(sizes) - min(sizes) <= 1
