#!/usr/bin/env python
"""Aggregate the per-line output of ncu_lines.py by enclosing device function.
usage: ncu_lines.py ... --top 2000 [--metric ...] | ncu_funcs.py"""
import bisect
import os
import re
import sys

CSRC = os.path.join(os.path.dirname(__file__), "..", "paper_2605_17913_b200", "csrc")


def starts(path):
    out = []
    for i, l in enumerate(open(path).read().splitlines(), 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?__(?:device|global)__[^(]*?(\w+)\s*\(", l)
        if m:
            out.append((i, m.group(1)))
    return out


F = {f: starts(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith(".cuh")}
agg = {}
for ln in sys.stdin:
    m = re.match(r"\s*([\d.]+)%\s+(\S+):(\d+)", ln)
    if not m:
        continue
    pct, f, l = float(m.group(1)), m.group(2), int(m.group(3))
    name = "?"
    if f in F:
        st = F[f]
        idx = bisect.bisect_right([s for s, _ in st], l) - 1
        if idx >= 0:
            name = st[idx][1]
    agg[f + ":" + name] = agg.get(f + ":" + name, 0) + pct
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:30]:
    print(f"{v:6.2f}% {k}")
