#!/bin/bash
# chord relax check: GPU chord tests, path-4 parity, cfg4 bench Newton vs chord
mkdir -p gpurun_out
TAG=${1:-chord}
timeout 1200 python -m pytest tests/test_gpu_chord.py tests/test_gpu_parity.py -k "chord or cfg4 or large_n or batched" -q -p no:cacheprovider --timeout 600 -rs -x > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest_rc=$?"; tail -5 gpurun_out/pytest_${TAG}.log
for rm in 0 2; do
timeout 600 python bench.py --no-cpu --relax-mode $rm > gpurun_out/bench_${TAG}_rm$rm.log 2>&1; echo "bench rm=$rm rc=$?"
python - <<PY
import json
l=[x for x in open("gpurun_out/bench_${TAG}_rm$rm.log") if x.startswith("{")][-1]; d=json.loads(l)
r=d["roofline"]; print("value",d["value"],"solve_ms",r["solve_ms"],"bwd_ms",r["backward_ms"],"riters",d["solver"]["relax_iters_mean"],"info",d["solver"]["kernel_info"].get("relax_mode"),d["solver"]["kernel_info"].get("chord_steps"), "e2e", d["e2e"]["value"])
PY
done
