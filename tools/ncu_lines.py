#!/usr/bin/env python
"""Aggregate ncu per-SASS-instruction warp-stall samples by CUDA source line.

usage: tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--so path/to/lib.so] [--top 40]

Maps SASS addresses to source lines with `nvdisasm -g` on the same binary the
report was taken from (the in-tree .so travels to the GPU box unchanged)."""
import argparse
import csv
import glob
import io
import os
import re
import subprocess
import tempfile
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--so", default=os.path.join(os.path.dirname(__file__), "..", "paper_2605_17913_b200",
                                                 "libqpb200.so"))
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--fn", default=None, help="regex on the MANGLED name picking the function in the .so "
                    "(default: the kernel regex); needed when several instantiations match")
    ap.add_argument("--metric", default="Warp Stall Sampling (All Samples)",
                    help="per-instruction column to aggregate, e.g. 'Instructions Executed'")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--kernel-name", f"regex:{a.kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    kname = lines[0].split(",")[1].strip('"')
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
    samples = {}
    reasons = {}
    rcols = [c for c in (rows[0].keys() if rows else []) if c.startswith("stall_") and "Not Issued" not in c]
    for r in rows:
        try:
            ad = int(r["Address"], 16)
            samples[ad] = int(r[a.metric] or 0)
            reasons[ad] = {c[6:]: int(r[c] or 0) for c in rcols}
        except (ValueError, KeyError):
            pass
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(a.so)], cwd=tmp, capture_output=True)
    cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    sass = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
    # locate the function body
    mangled = None
    for m in re.finditer(r"^\.text\.(\S+):", sass, flags=re.M):
        if re.search(a.fn or a.kernel, m.group(1)):
            mangled = m.group(1)
            break
    body = sass.split(f".text.{mangled}:")[1]
    cur = None
    addr_line = {}
    for ln in body.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            addr_line[int(m.group(1), 16)] = cur
        if ln.startswith("\t.section") or ln.startswith(".section"):
            break
    agg = defaultdict(int)
    tot = 0
    base = min(samples) if samples else 0
    samples = {ad - base: s for ad, s in samples.items()}
    reasons = {ad - base: v for ad, v in reasons.items()}
    ragg = defaultdict(lambda: defaultdict(int))
    rtot = defaultdict(int)
    for ad, s in samples.items():
        key = addr_line.get(ad, ("?", 0))
        agg[key] += s
        tot += s
        for rn, rv in reasons.get(ad, {}).items():
            ragg[key][rn] += rv
            rtot[rn] += rv
    src_cache = {}
    print(f"{kname}: {tot} samples")
    for (f, l), s in sorted(agg.items(), key=lambda kv: -kv[1])[: a.top]:
        if f not in src_cache:
            p = os.path.join(os.path.dirname(a.so), "csrc", f)
            src_cache[f] = open(p).read().splitlines() if os.path.exists(p) else []
        txt = src_cache[f][l - 1].strip() if 0 < l <= len(src_cache[f]) else ""
        top = sorted(ragg[(f, l)].items(), key=lambda kv: -kv[1])[:2]
        rs = " ".join(f"{k}:{v}" for k, v in top if v)
        print(f"{100.0 * s / max(tot, 1):6.2f}%  {f}:{l:<5d} {txt[:90]:90s} [{rs}]")
    rt = sum(rtot.values()) or 1
    print("stall reasons:", ", ".join(f"{k} {100.0 * v / rt:.1f}%" for k, v in
                                      sorted(rtot.items(), key=lambda kv: -kv[1])[:10]))


if __name__ == "__main__":
    main()
