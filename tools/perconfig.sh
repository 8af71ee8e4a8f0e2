#!/bin/bash
# Per-config bench lines (BASELINE.json configs 1-5 and the N4 application
# workloads): one `bench.py` JSON line each, collected under gpurun_out/.
# usage (on the GPU box): tools/perconfig.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
OUT=gpurun_out/perconfig_${TAG}.jsonl
: > $OUT
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 2>/dev/null | tail -1 >> $OUT
done
for w in cbf7 cbf9 bezier4 bezier8; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 2>/dev/null | tail -1 >> $OUT
done
wc -l $OUT
