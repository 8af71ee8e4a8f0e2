#!/bin/bash
mkdir -p gpurun_out
for bc in 512 1024 2048 4096; do
for nl in 1 2; do
QPB200_BCHUNK=$bc QPB200_BLANES=$nl timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d10.log 2>&1; echo "bchunk $bc lanes $nl rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/d10.log | head -1)"
done; done
