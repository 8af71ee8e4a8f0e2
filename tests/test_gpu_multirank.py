"""The N > 1 launch path of bench.py (torchrun, one process per GPU, batch
sharded by rank, max-over-ranks timing, the config-4 shared-gradient
all-reduce) exercised with two ranks.  A 1-GPU box cannot host two NCCL ranks
on one device, so the ranks use gloo (QPB200_DIST_BACKEND) and share cuda:0;
their kernels never wait on each other."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg,batch", [(1, None), (4, 48)])
def test_two_rank_bench_line(cfg, batch):
    env = dict(os.environ, QPB200_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", str(cfg), "--steps", "2", "--warmup", "3", "--no-cpu"]
    if batch:
        cmd += ["--batch", str(batch)]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]          # rank 0 prints exactly one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    assert d["config"]["global_batch"] == 2 * d["config"]["batch_per_gpu"]
    assert d["solver"]["converged"] == d["config"]["batch_per_gpu"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
