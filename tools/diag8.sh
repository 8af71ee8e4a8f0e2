#!/bin/bash
mkdir -p gpurun_out
for c in 2 3 5; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d8_c$c.log 2>&1; echo "cfg$c rc=$?"; grep -o '"value": [0-9.]*' gpurun_out/d8_c$c.log | head -1
  QPB200_FORCE_GLOBAL=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d8_c${c}g.log 2>&1; echo "cfg$c forced-batched rc=$?"; grep -o '"value": [0-9.]*' gpurun_out/d8_c${c}g.log | head -1
done
