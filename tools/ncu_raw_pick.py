"""Pick metrics from `ncu -i REP --page raw --csv` output (stdin or file):
one line per kernel launch, `metric = value unit` for columns matching the
given regexes.  usage: ncu_raw_pick.py RAW.csv REGEX..."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
rows = [r for r in rows if r and not r[0].startswith("==")]
hdr, units, data = rows[0], rows[1], rows[2:]
pats = [re.compile(p) for p in sys.argv[2:]]
for d in data:
    name = d[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"# {name[:80]}")
    for i, h in enumerate(hdr):
        if any(p.search(h) for p in pats):
            print(f"{h} = {d[i]} {units[i] if i < len(units) else ''}")
