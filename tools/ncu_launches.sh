#!/bin/bash
# Per-kernel device time of one solve+backward (ncu launch list, cold-cache, serialised)
# usage: tools/ncu_launches.sh CFG B TAG
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$3.csv \
    python tools/run_cfg.py $1 $2 > gpurun_out/ncu_launch_$3.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary_launches.py gpurun_out/launches_$3.csv
