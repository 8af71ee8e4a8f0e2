#!/usr/bin/env python
"""Markdown table of the per-config bench lines (tools/perconfig.sh).
usage: perconfig_table.py IN.jsonl OUT.md"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
out = ["| workload | QP/s (device) | QP/s (e2e) | ms/step | solve ms | backward ms | alg. TFLOP/s (dominant launch) | "
       "frac of FP32 peak | iters mean / max | relax iters mean | path, threads, CTAs/SM, pcap | oracle QP/s (cores) |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for d in rows:
    r, s, k = d["roofline"], d["solver"], d["solver"]["kernel_info"]
    cpu = d.get("cpu_baseline") or {}
    e2e = d.get("e2e") or {}
    out.append(f"| {d['config']['workload']} | {d['value']:.4g} | {e2e.get('value', float('nan')):.4g} | "
               f"{d['ms_per_step']:.3f} | {r['solve_ms']:.3f} | {r['backward_ms']:.3f} | {r['achieved']:.3g} | "
               f"{r['frac']:.4f} | {s['iters_mean']:.2f} / {s['iters_max']} | {s['relax_iters_mean']:.2f} | "
               f"{k['path']}, {k['threads']}, {k['ctas_per_sm']}, {k.get('partition_cap', '')} | "
               f"{cpu.get('value', float('nan')):.4g} ({cpu.get('cores', '')}) |")
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out))
