"""bench.py contract on CPU: the reference arm (the oracle)
prints one JSON line with the keys the driver reads, and its metric, unit and
workload match the GPU arm's defaults."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    r = json.loads(lines[0])
    assert r["impl"] == "reference" and r["unit"] == "QP/s" and r["higher_is_better"] is True
    assert r["value"] > 0 and r["steps"] == 1 and r["warmup"] == 0 and r["n_gpus"] == 1
    assert r["config"]["workload"] == "cfg4_bilevel_shared_n200_p400_B8192"  # the default (metric) config
    assert r["cpu_baseline"]["kind"] == "oracle" and r["cpu_baseline"]["value"] == r["value"]
    assert r["cpu_baseline"]["cores"] >= 1 and r["scaling"] == "strong"
    assert r["e2e"] == {"value": r["value"], "unit": "QP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_gpus_without_torchrun_relaunches_and_reference_ranks_exit():
    """`--gpus 2` without torchrun re-executes bench.py under
    torch.distributed.run (one process per GPU); in the reference arm rank 0
    alone runs the oracle and prints the line, rank 1 exits 0."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "1",
                          "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    r = json.loads(lines[0])
    assert r["impl"] == "reference" and r["n_gpus"] == 2 and r["config"]["workload"].startswith("cfg1")
