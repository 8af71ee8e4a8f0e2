#!/usr/bin/env python
"""Benchmark: batched f32 QP solve + backward (Alg. 1 + Alg. 2 + Alg. 3 of
arxiv 2605.17913) through the C ABI on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Default workload: BASELINE.json config 4, the end-to-end / bilevel training
step (8192 QPs, n = 200, p = 400, Q, G, h shared by the batch, gradients
all-reduced) — the configuration the metric's "1/2/4/8 B200" is defined on.
One step = qp_solve_batched + qp_backward_batched over this rank's slice of
the FIXED global batch (strong scaling: rank r of N takes the contiguous
slice dist.shard(B, r, N)), plus the NCCL all-reduce of the shared-parameter
gradients.  `--gpus N` without torchrun re-executes itself under
`torch.distributed.run --nproc-per-node N` (one process per GPU).
Metric (BASELINE.json): QP solve+backward/sec, f32, device-timed, whole job
(global batch ÷ max-over-ranks time).  Rank 0 prints ONE JSON line.  See
DESIGN.md §7 for every field."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2605_17913_b200 import flops as FL  # noqa: E402
from paper_2605_17913_b200 import generators as gen  # noqa: E402

METRIC = "QP solve+backward/sec (f32, device-timed)"
UNIT = "QP/s"
FIELDS = ("Q", "q", "A", "b", "G", "h")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, help="BASELINE.json config index (1-based)")
    ap.add_argument("--batch", type=int, default=None,
                    help="override the GLOBAL batch (plumbing tests only; bench lines use the config's batch)")
    ap.add_argument("--workload", default=None, choices=sorted(gen.WORKLOADS),
                    help="an N4 application shape instead of a BASELINE.json config")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--relax-mode", type=int, default=None, choices=(0, 2),
                    help="Alg. 2 linear solves: 0 exact Newton, 2 guarded chord (reading Q26); default: the library's")
    ap.add_argument("--dump", default=None,
                    help="write this rank's outputs of the last timed step to DIR/rank<r>.npz (tests)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled DURING the timed region (B200_PROFILING.md "clocks" line)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid: str | None):
        self.uuid = uuid
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        rows = [r for r in self.rows if self.uuid is None or self.uuid in r[0]] or self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({nm for r in rows for nm, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# the oracle (CPU) legs
# ---------------------------------------------------------------------------
def workload_of(a) -> dict:
    """The workload bench.py runs: BASELINE.json config `--config`, or an N4
    application shape `--workload` (generators.WORKLOADS)."""
    w = _workload_of(a)
    if getattr(a, "relax_mode", None) is not None:
        w["solver"]["relax_mode"] = a.relax_mode
    return w


def _workload_of(a) -> dict:
    if getattr(a, "workload", None):
        w = gen.WORKLOADS[a.workload]
        b1 = gen.make_workload(a.workload, batch=1)
        return dict(name=w["name"], n=b1.n, m=b1.m, p=b1.p, batch=w["batch"], key=a.workload,
                    make=lambda B, start=0: gen.make_workload(a.workload, batch=B, start=start),
                    solver=dict(w.get("solver", {})))
    c = gen.CONFIGS[a.config]
    return dict(name=c["name"], n=c["n"], m=c["m"], p=c["p"], batch=c["batch"], key=f"cfg{a.config}",
                make=lambda B, start=0: gen.make_config(a.config, batch=B, start=start), solver={})


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate(W: dict, target_s: float, batch_cap: int, start: int = 0, prec: str = "f64",
                single_pass: bool = False):
    """Time the oracle on a bounded sample of the workload, all host cores:
    prec "f64" = the parity reference (paper-literal Eq. 14 + GEPP), "f32" =
    the iteration-count reference (M_PART, the CUDA path's algorithm class).
    Returns (QP/s, cores, n_problems, seconds)."""
    import oracle
    nt = oracle.hardware_threads()
    cfg = oracle.Cfg.f64() if prec == "f64" else oracle.Cfg.f32()
    pilot = W["make"](min(nt, batch_cap), start)
    t0 = time.perf_counter()
    r = oracle.solve(pilot, cfg, prec, nthreads=nt)
    oracle.backward(pilot, r, cfg, prec, nthreads=nt)
    dt = time.perf_counter() - t0
    rate = pilot.batch / max(dt, 1e-6)
    if single_pass:  # (very large problems: the pilot is the sample)
        return rate, nt, pilot.batch, dt
    ns = int(min(batch_cap, max(pilot.batch, round(rate * target_s))))
    ns = max(nt, (ns // nt) * nt) if ns >= nt else ns
    samp = W["make"](ns, start)
    t0 = time.perf_counter()
    r = oracle.solve(samp, cfg, prec, nthreads=nt)
    oracle.backward(samp, r, cfg, prec, nthreads=nt)
    dt = time.perf_counter() - t0
    return ns / dt, nt, ns, dt


def run_reference(a):
    """The reference arm: the oracle as it stands (f64, paper-literal Eq. 14 +
    GEPP) on the host cores, same workload, metric and unit; under torchrun
    only rank 0 runs it."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    c = workload_of(a)
    import oracle
    nt = oracle.hardware_threads()
    # calibrate one step to ~4 s of CPU work so K+W steps finish in minutes
    _, _, ns, _ = oracle_rate(c, 4.0, a.batch or c["batch"])
    samp = c["make"](ns)
    times = []
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        r = oracle.solve(samp, oracle.Cfg.f64(), "f64", nthreads=nt)
        oracle.backward(samp, r, oracle.Cfg.f64(), "f64", nthreads=nt)
        if i >= a.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = ns * a.steps / tot
    sample = (f"first {ns} problems of {c['name']} per step; f64 oracle "
              f"(Eq. 14 + GEPP), init + Alg. 1 + Alg. 2 + Alg. 3, std::thread over problems; CPU {cpu_model()}")
    out = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
           "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": c["name"], "batch_per_step": ns, "n": c["n"], "m_eq": c["m"], "p": c["p"]},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": nt, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------
# N > 1 without torchrun: one process per GPU via torch.distributed.run
# ---------------------------------------------------------------------------
def relaunch(a) -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    # NCCL communicator set-up on stderr (ranks, transport); stdout keeps the one JSON line
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(a)
    if a.impl == "reference":
        return run_reference(a)
    import torch
    from paper_2605_17913_b200 import dist as D
    from paper_2605_17913_b200.solver import QPSolver

    rank, world, local = D.init()
    if world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    ndev = torch.cuda.device_count()
    if world > ndev and os.environ.get("QPB200_DIST_BACKEND") != "gloo":
        print(f"bench.py: {world} ranks need {world} GPUs, this node has {ndev}", file=sys.stderr)
        return 2
    local = local % max(1, ndev)  # = LOCAL_RANK on a node with ≥ world GPUs (gloo plumbing tests share one)
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    c = workload_of(a)
    n, m, p = c["n"], c["m"], c["p"]
    B_glob = a.batch or c["batch"]
    start, stop = D.shard(B_glob, rank, world)  # strong scaling: this rank's slice of the fixed global batch
    B = stop - start
    batch = c["make"](B, start)  # problem i of the global batch is the same problem at every world size
    shared = [k for k, v in batch.shared.items() if v]
    if world > 1:
        # communicator up before timing; its size goes to stderr next to NCCL's own INIT lines
        t = torch.ones(1, device=dev)
        torch.distributed.all_reduce(t)
        print(f"[bench rank {rank}] communicator: backend={torch.distributed.get_backend()} nranks={int(t.item())} "
              f"problems [{start}, {stop})", file=sys.stderr, flush=True)
    S = QPSolver(B, n, m, p, shared=shared, device=local, **c["solver"])
    info = S.info()

    def T(f):
        arr = getattr(batch, f)
        arr = arr[0] if f in shared else arr
        return torch.from_numpy(np.ascontiguousarray(arr)).to(dev)

    data = [T(f) for f in FIELDS]
    dl = torch.from_numpy(batch.dl_dx).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step():
        out = S.solve(*data)
        g = S.backward(dl)
        D.allreduce_shared_grads(g, shared)
        return out, g

    for _ in range(a.warmup):
        out, g = step()
    torch.cuda.synchronize(dev)
    D.barrier()
    torch.cuda.synchronize(dev)
    props = torch.cuda.get_device_properties(dev)
    uuid = (str(getattr(props, "uuid", "")) or None) if world == 1 else None  # N > 1: every GPU of the node
    clk = ClockSampler(uuid)
    if rank == 0:
        clk.start()
        time.sleep(0.3)
    t_solve = t_bwd = 0.0
    for _ in range(a.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (outside the events)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        out = S.solve(*data)
        e1.record(stream)
        g = S.backward(dl)
        D.allreduce_shared_grads(g, shared)
        e2.record(stream)
        e2.synchronize()
        t_solve += e0.elapsed_time(e1)
        t_bwd += e1.elapsed_time(e2)
    torch.cuda.synchronize(dev)
    if rank == 0:
        clk.stop()
    D.barrier()
    total_ms = D.max_over_ranks(t_solve + t_bwd, dev)
    value = B_glob * a.steps / (total_ms / 1e3)

    if a.dump:
        os.makedirs(a.dump, exist_ok=True)
        np.savez(os.path.join(a.dump, f"rank{rank}.npz"), start=start, stop=stop,
                 **{k: v.cpu().numpy() for k, v in out.items()},
                 **{"g_" + k: v.cpu().numpy() for k, v in g.items()})
    info = S.info()  # after the calls: the batched engine counts its launches per call
    path4 = info.get("path") == 4
    iters = out["iters"].cpu().numpy()
    riters = g["relax_iters"].cpu().numpy()
    status = out["status"].cpu().numpy()
    gstatus = g["status"].cpu().numpy()
    ms_solve, ms_bwd = t_solve / a.steps, t_bwd / a.steps
    peak = FL.fp32_peak_tflops(props.multi_processor_count)
    dom_solve = ms_solve >= ms_bwd
    # SURVEY §8(d) algorithmic flops (K14-literal) of this rank's launches,
    # from the measured per-problem iteration counts
    k14_s = float(sum(FL.k14_solve(n, m, p, int(i)) for i in iters))
    # chord steps (reading Q26) factor nothing: the batch total from qp_info
    k14_b = float(sum(FL.k14_backward(n, m, p, int(r)) for r in riters)) - \
        float(info.get("chord_steps", 0)) * (n + p + m) ** 3 / 3
    # executed flops of the reduced systems, counted inside the kernels
    x_s, x_b = S.last_flops()
    f_dom, x_dom, ms_dom = (k14_s, x_s, ms_solve) if dom_solve else (k14_b, x_b, ms_bwd)
    achieved = f_dom / (ms_dom / 1e3) / 1e12
    if path4:  # batched phase engine: one call = a sequence of phase kernels
        kname = (f"qp_solve_batched ({info['launches_solve']} launches of the batched engine)" if dom_solve else
                 f"qp_backward_batched ({info['launches_backward']} launches of the batched engine)")
    else:
        kname = "ipm_kernel (solve launch)" if dom_solve else "ipm_kernel (backward launch)"
    roofline = {"bound": "alu", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                "work_model": "SURVEY §8(d) K14-literal: per iteration N^3/3 + 2N^2 + 2n^2 + 6pn + 4mn "
                              "(N = n+p+m) at the measured iteration counts, + init, + p*n^2 once (flops.py)",
                "peak_note": "FP32 FMA: SMs x 128 lanes x 2 flop x 1965 MHz (derived, DESIGN.md §6)",
                "traffic_note": "DRAM bytes per launch from ncu --set full: profiles/r2/ (not measurable in this run)",
                "flops_per_launch": f_dom, "ms_per_launch": ms_dom,
                "frac_exec": x_dom / (ms_dom / 1e3) / 1e12 / peak, "exec_flops_per_launch": x_dom,
                "solve_ms": ms_solve, "backward_ms": ms_bwd,
                "solve_tflops": k14_s / (ms_solve / 1e3) / 1e12, "backward_tflops": k14_b / (ms_bwd / 1e3) / 1e12,
                "step_tflops": (k14_s + k14_b) / ((ms_solve + ms_bwd) / 1e3) / 1e12}

    # ---- e2e: host buffers through the C ABI, H2D/D2H inside the timed region
    e2e = None
    if not a.no_e2e:
        Sh = QPSolver(B, n, m, p, shared=shared, device=local, mem="host_async", **c["solver"])
        hdata = [torch.from_numpy(np.ascontiguousarray(getattr(batch, f)[0] if f in shared else getattr(batch, f)))
                 .pin_memory() for f in FIELDS]
        hdl = torch.from_numpy(batch.dl_dx).pin_memory()

        # output buffers (pinned) allocated once, as a training loop would
        o0 = Sh.solve(*hdata)
        g0 = Sh.backward(hdl)

        def hstep():
            o = Sh.solve(*hdata, out=o0)
            gg = Sh.backward(hdl, out=g0)
            if shared:
                dd = {k: v.to(dev) for k, v in gg.items() if k in ("dQ", "dq", "dA", "db", "dG", "dh")}
                D.allreduce_shared_grads(dd, shared)
            return o, gg

        for _ in range(max(3, a.warmup)):
            hstep()
        torch.cuda.synchronize(dev)
        D.barrier()
        h_ms = 0.0
        for _ in range(a.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.default_stream(dev))
            o, gg = hstep()
            e1.record(torch.cuda.default_stream(dev))
            e1.synchronize()
            h_ms += e0.elapsed_time(e1)
        h_ms = D.max_over_ranks(h_ms, dev)
        per, sh = FL.data_bytes(n, m, p, shared)
        h2d = B * per + sh + B * n * 4
        d2h = sum(int(v.numel() * v.element_size()) for v in o.values()) + \
            sum(int(v.numel() * v.element_size()) for v in gg.values())
        e2e = {"value": B_glob * a.steps / (h_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": h_ms / a.steps,
               "note": "QP_MEM_HOST_ASYNC: pinned host inputs and outputs, per-rank bytes"}
        Sh.close()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu and n + m + p > 2048:
        # config-5 size: the f64 paper-literal solve (Eq. 14 + GEPP, N = 3072)
        # takes ~10 min per problem on one core (reading Q25); one problem per
        # host core of the f32 oracle (M_PART) is the bounded sample
        r32, cores, ns32, dt32 = oracle_rate(c, a.cpu_seconds, B, prec="f32", single_pass=True)
        cpu = {"value": r32, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"first {ns32} problems of {c['name']} ({dt32:.1f} s), one per host thread: f32 oracle "
                         f"(M_PART, reading Q12b), init + Alg. 1 + Alg. 2 + Alg. 3; the f64 Eq. 14 + GEPP oracle "
                         f"is not timed at this size (~10 min per problem, DESIGN.md reading Q25)",
               "f32_value": r32}
    elif rank == 0 and world == 1 and not a.no_cpu:
        rate, cores, ns, dt = oracle_rate(c, a.cpu_seconds, B)
        r32, _, ns32, dt32 = oracle_rate(c, a.cpu_seconds / 3, B, prec="f32")
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"first {ns} problems of {c['name']} ({dt:.1f} s): f64 oracle (Eq. 14 + GEPP), "
                         f"init + Alg. 1 + Alg. 2 + Alg. 3, std::thread over problems",
               "f32_value": r32,
               "f32_sample": f"first {ns32} problems ({dt32:.1f} s): f32 oracle (M_PART, reading Q12b)"}

    clocks = clk.summary() if rank == 0 else None
    if rank == 0:
        launches = info["launches_solve"] + info["launches_backward"]
        res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f32", "data": "synthetic",
               "config": {"workload": c["name"], "global_batch": B_glob, "batch_per_gpu": B, "n": n, "m_eq": m,
                          "p": p, "shared": shared, "parallelism": f"dp{world} (fixed global batch sharded by rank"
                          + (", NCCL all-reduce of the shared-parameter gradients" if shared and world > 1 else "")
                          + ")",
                          "l2": "flushed between timed steps (256 MiB write outside the events)",
                          "tol": S.cfg.tol, "kappa_relax": S.cfg.kappa_relax, "sigma": S.cfg.sigma},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": a.steps * launches,
               "clocks": clocks,
               "solver": {"converged": int((status == 0).sum()), "grad_ok": int((gstatus == 0).sum()),
                          "iters_mean": float(iters.mean()), "iters_max": int(iters.max()),
                          "relax_iters_mean": float(riters.mean()), "kernel_info": info}}
        print(json.dumps(res), flush=True)
    S.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
