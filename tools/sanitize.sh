#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every
# kernel instantiation (tools/sanitize_cases.py).  Run on the GPU box:
#   bash tools/sanitize.sh > gpurun_out/sanitize.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=${CASES:-"p1_128 p1_256x2 p1_256x1 small64 bigN explicit shared host_async pdl"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
for c in $CASES; do
  for t in $TOOLS; do
    echo "=== $c / $t"
    timeout 900 $CS --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py $c 2>&1 | \
      grep -v "^\s*$" | tail -12
    echo "rc=${PIPESTATUS[0]}"
  done
done
