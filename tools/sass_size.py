#!/usr/bin/env python
"""SASS bytes per enclosing device function (by -lineinfo source lines) of one kernel.
usage: sass_size.py MANGLED_REGEX [--so lib]"""
import argparse
import bisect
import collections
import glob
import os
import re
import subprocess
import tempfile

ap = argparse.ArgumentParser()
ap.add_argument("fn")
ap.add_argument("--so", default=os.path.join(os.path.dirname(__file__), "..", "paper_2605_17913_b200", "libqpb200.so"))
a = ap.parse_args()
CSRC = os.path.join(os.path.dirname(__file__), "..", "paper_2605_17913_b200", "csrc")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(a.so)], cwd=tmp, capture_output=True)
cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
sass = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
mangled = next(m.group(1) for m in re.finditer(r"^\.text\.(\S+):", sass, flags=re.M) if re.search(a.fn, m.group(1)))
body = sass.split(f".text.{mangled}:")[1]
cur = None
cnt = collections.Counter()
for ln in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        cnt[cur] += 16
    if ln.startswith("\t.section") or ln.startswith(".section"):
        break


def starts(path):
    out = []
    for i, l in enumerate(open(path).read().splitlines(), 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?__(?:device|global)__[^(]*?(\w+)\s*\(", l)
        if m:
            out.append((i, m.group(1)))
    return out


F = {f: starts(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith(".cuh")}
agg = collections.Counter()
for key, b in cnt.items():
    name = "?"
    if key and key[0] in F:
        st = F[key[0]]
        i = bisect.bisect_right([s for s, _ in st], key[1]) - 1
        if i >= 0:
            name = st[i][1]
    agg[(key[0] if key else "?") + ":" + name] += b
print(mangled, sum(cnt.values()), "bytes")
for k, v in agg.most_common(25):
    print(f"{v:8d} {k}")
