#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d5_bench.log 2>&1; echo "bench rc=$?"; grep -o '"value": [0-9.]*' gpurun_out/d5_bench.log | head -1
bash tools/ncu_launches.sh 4 2048 c4d | head -9
