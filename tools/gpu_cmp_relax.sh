#!/bin/bash
# bench lines for Newton vs guarded-chord relax on the given configs
mkdir -p gpurun_out
TAG=${1:-cmp}; shift
for cfg in "$@"; do for rm in 0 2; do
timeout 900 python bench.py --no-cpu --config $cfg --relax-mode $rm > gpurun_out/bench_${TAG}_c${cfg}_rm$rm.log 2>&1
python - <<PY
import json
l=[x for x in open("gpurun_out/bench_${TAG}_c${cfg}_rm$rm.log") if x.startswith("{")][-1]; d=json.loads(l)
r=d["roofline"]; print("cfg $cfg rm $rm value %.1f solve_ms %.3f bwd_ms %.3f riters %.2f chord %s e2e %.1f" % (d["value"],r["solve_ms"],r["backward_ms"],d["solver"]["relax_iters_mean"],d["solver"]["kernel_info"].get("chord_steps"), d["e2e"]["value"]))
PY
done; done
