#!/bin/bash
# ncu --set full on one launch of a kernel: tools/ncu_kernel.sh REGEX SKIP CFG B TAG
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_$5 \
    python tools/run_cfg.py $3 $4 > gpurun_out/ncu_$5.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_$5.ncu-rep --page details --csv > gpurun_out/details_$5.csv 2>/dev/null
ncu -i gpurun_out/prof_$5.ncu-rep --page source --csv > gpurun_out/source_$5.csv 2>/dev/null
ls -la gpurun_out/prof_$5.ncu-rep
