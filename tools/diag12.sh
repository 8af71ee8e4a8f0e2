#!/bin/bash
for f in 2 4; do for nl in 2 3; do
QPB200_KR_DIV=$f QPB200_BLANES=$nl timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d12.log 2>&1; echo "div $f lanes $nl rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/d12.log | head -1)"
done; done
