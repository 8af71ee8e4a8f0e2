#!/bin/bash
# Turn the gpurun_out/ artifacts of tools/gpu_artifacts.sh TAG into the
# committed summaries under profiles/TAG (run here, after the gpurun call).
set -e
TAG=${1:-r1}
OUT=profiles/$TAG
mkdir -p $OUT
cp gpurun_out/launches_${TAG}.csv $OUT/launches.csv
tail -1 gpurun_out/bench_full_${TAG}.log > $OUT/bench_line.json
python - "$OUT" <<'PY'
import csv, collections, sys
out = sys.argv[1]
rows = [r for r in csv.reader(open(f"{out}/launches.csv")) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
nth = {}
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    name = r[ki].split("(")[0]
    if "ipm_kernel" in name:  # one kernel serves both calls: solve launches first, backward second
        nth[name] = nth.get(name, 0) + 1
        name += " [solve launch]" if nth[name] % 2 == 1 else " [backward launch]"
    tot[name] += v * scale.get(r[ui], 1.0)
    cnt[name] += 1
T = sum(tot.values())
with open(f"{out}/launches_summary.txt", "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold caches, serialised):\n")
    f.write("bench.py --no-cpu --no-e2e --steps 2 --warmup 1, config 2 (1024 QPs)\n")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{100 * v / T:6.2f}%  {v:9.3f} ms  {cnt[k]:3d} launches  {v / cnt[k]:8.3f} ms/launch  {k}\n")
PY
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep > $OUT/ncu_full_summary.txt
python tools/ncu_summary.py gpurun_out/prof_${TAG}_bwd.ncu-rep | sed 's/^void ipm_kernel/bwd  ipm_kernel/' >> $OUT/ncu_full_summary.txt
FN=$(python -c "import json; d=json.load(open('$OUT/bench_line.json')); i=d['solver']['kernel_info']; print('ILi%dELi%d' % (i['threads'], i['ctas_per_sm']))")
python tools/ncu_lines.py gpurun_out/prof_${TAG}.ncu-rep ipm_kernel --fn "ipm_kernel$FN" --top 60 > $OUT/source_lines_solve.txt 2>/dev/null
python tools/ncu_lines.py gpurun_out/prof_${TAG}_bwd.ncu-rep ipm_kernel --fn "ipm_kernel$FN" --top 60 > $OUT/source_lines_backward.txt 2>/dev/null
python tools/ncu_lines.py gpurun_out/prof_${TAG}.ncu-rep ipm_kernel --fn "ipm_kernel$FN" --top 3000 2>/dev/null | python tools/ncu_funcs.py > $OUT/functions_solve_stalls.txt
python tools/ncu_lines.py gpurun_out/prof_${TAG}.ncu-rep ipm_kernel --fn "ipm_kernel$FN" --top 3000 --metric "Instructions Executed" 2>/dev/null | python tools/ncu_funcs.py > $OUT/functions_solve_instructions.txt
python - "$TAG" <<'PY'
import csv, io, json, subprocess, sys
tag = sys.argv[1]
out = {}
for key, rep in (("solve", f"gpurun_out/prof_{tag}.ncu-rep"), ("backward", f"gpurun_out/prof_{tag}_bwd.ncu-rep")):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw))); h = rows[0]
    ix = [h.index(c) for c in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
    units = [rows[1][i] for i in ix]
    mb = lambda v, u: float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    r = rows[2]
    out[key] = mb(r[ix[0]], units[0]) + mb(r[ix[1]], units[1])
out["_doc"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes) of the solve and of the backward "
               "launch of ipm_kernel, ncu --set full captures summarised in profiles/" + tag + "/ncu_full_summary.txt "
               "(bench.py config 2, 1024 problems). Algorithmic minimum for the solve launch = problem data read "
               "once = 1024 x 32.8 KB = 33.6 MB.")
json.dump(out, open("profiles/traffic_cfg2.json", "w"), indent=1)
print(out)
PY
head -5 $OUT/launches_summary.txt; head -8 $OUT/ncu_full_summary.txt; head -6 $OUT/functions_solve_stalls.txt
