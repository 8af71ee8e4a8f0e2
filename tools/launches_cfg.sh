#!/bin/bash
# launch list (ncu gpu__time_duration, serialised, cold-cache) of one timed bench step of config $1
mkdir -p gpurun_out
C=${1:-4}
python bench.py --config $C --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/plain_$C.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$C.csv \
    python bench.py --config $C --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_launch_$C.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary_launches.py gpurun_out/launches_cfg$C.csv > gpurun_out/launches_cfg${C}_summary.txt
head -16 gpurun_out/launches_cfg${C}_summary.txt
