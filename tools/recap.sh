#!/bin/bash
# re-capture ncu --set full of chosen launches: tools/recap.sh NAME REGEX SKIP CFG B
O=gpurun_out/r2f; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $O/full_$1 \
    python tools/run_cfg.py $4 $5 > $O/ncu_full_$1.log 2>&1
python tools/ncu_summary.py $O/full_$1.ncu-rep > $O/full_$1_summary.txt 2>&1
ncu -i $O/full_$1.ncu-rep --page raw --csv > $O/full_$1_raw_all.csv 2>&1
python tools/ncu_raw_pick.py $O/full_$1_raw_all.csv 'dram__bytes_(read|write)\.sum$' 'sm__pipe_tensor.*cycles_active.*pct' 'sm__pipe_fma_cycles_active.*pct' '^gpu__time_duration\.sum$' 'sm__throughput\.avg\.pct' 'launch__(registers|occupancy_limit)' 'smsp__issue_active.avg.pct' > $O/full_$1_raw.txt 2>&1
rm -f $O/full_$1_raw_all.csv
python tools/ncu_lines.py $O/full_$1.ncu-rep $2 --top 20 > $O/full_$1_lines.txt 2>&1
rm -f $O/full_$1.ncu-rep
grep -E "Duration" $O/full_$1_summary.txt
