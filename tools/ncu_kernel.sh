#!/bin/bash
# ncu --set full on one launch of a kernel: tools/ncu_kernel.sh REGEX SKIP CFG B TAG
# Writes text summaries (metrics + source-line stalls) next to the report;
# the .ncu-rep is removed unless KEEP=1 (gpurun_out/ is capped at 64 MiB).
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_$5 \
    python tools/run_cfg.py $3 $4 > gpurun_out/ncu_$5.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_$5.ncu-rep > gpurun_out/sum_$5.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_$5.ncu-rep $1 --top 25 > gpurun_out/lines_$5.txt 2>&1
[ "$KEEP" == "1" ] || rm -f gpurun_out/prof_$5.ncu-rep
