"""The N > 1 launch path of bench.py (one process per GPU, the FIXED global
batch sharded by rank — strong scaling, SURVEY §8(e) — max-over-ranks timing,
the config-4 shared-gradient all-reduce) exercised with two ranks.  A 1-GPU
box cannot host two NCCL ranks on one device, so the ranks use gloo
(QPB200_DIST_BACKEND) and share cuda:0; their kernels never wait on each
other.  Per-problem outputs must be bitwise identical at world size 1 and 2
(problems are independent; the shared sums differ only by summation order)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, cfg, batch, dump, torchrun):
    env = dict(os.environ, QPB200_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    args = [os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--config", str(cfg), "--steps", "2",
            "--warmup", "3", "--no-cpu", "--dump", dump]
    if batch:
        args += ["--batch", str(batch)]
    if torchrun and world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
               "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    else:  # bench.py re-executes itself under torch.distributed.run for --gpus > 1
        cmd = [sys.executable] + args
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]          # rank 0 prints exactly one line
    return json.loads(lines[0]), out.stderr


@pytest.mark.parametrize("cfg,batch,torchrun", [(1, None, True), (4, 48, False)])
def test_two_rank_bench_line_strong_scaling(tmp_path, cfg, batch, torchrun):
    d1, _ = _run(1, cfg, batch, str(tmp_path / "w1"), True)
    d2, err = _run(2, cfg, batch, str(tmp_path / "w2"), torchrun)
    B = d1["config"]["global_batch"]
    assert d2["n_gpus"] == 2 and d2["steps"] == 2 and d2["value"] > 0 and d2["scaling"] == "strong"
    assert d2["config"]["global_batch"] == B                      # fixed global batch
    assert d2["config"]["batch_per_gpu"] == (B + 1) // 2
    assert d2["solver"]["converged"] == d2["config"]["batch_per_gpu"]
    assert d2["e2e"]["value"] > 0 and d2["gpu_launches"] > 0
    assert "nranks=2" in err
    r1 = dict(np.load(tmp_path / "w1" / "rank0.npz"))
    parts = [dict(np.load(tmp_path / "w2" / f"rank{r}.npz")) for r in range(2)]
    assert int(parts[0]["start"]) == 0 and int(parts[0]["stop"]) == int(parts[1]["start"])
    assert int(parts[1]["stop"]) == B
    shared = set(d1["config"]["shared"])
    for k in r1:
        if k in ("start", "stop"):
            continue
        if k.startswith("g_d") and k[3:] in shared:   # batch-summed then all-reduced
            tot = parts[0][k].astype(np.float64)       # (already the global sum on every rank)
            ref = r1[k].astype(np.float64)
            assert np.linalg.norm(tot - ref) <= 1e-5 * np.linalg.norm(ref), k
            continue
        both = np.concatenate([parts[0][k], parts[1][k]])
        assert np.array_equal(both, r1[k]), k          # per-problem outputs: bitwise
