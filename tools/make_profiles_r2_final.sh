#!/bin/bash
# Round-2 final profile artifacts (run on the GPU box):  bash tools/make_profiles_r2_final.sh
# -> gpurun_out/r2f/: bench lines (configs 4, 2, 3, 5), ncu launch lists of one timed step
#    (configs 4 and 5), --set full summaries of the batched-engine kernels (config 4,
#    2048 problems) and of the path-1 kernel (config 2)
set -x
O=gpurun_out/r2f; mkdir -p $O
timeout 900 python bench.py > $O/bench_line.json 2> $O/bench_line.err
timeout 900 python bench.py --config 2 > $O/bench_line_cfg2.json 2> $O/bench_line_cfg2.err
timeout 900 python bench.py --config 3 --no-cpu > $O/bench_line_cfg3.json 2> $O/bench_line_cfg3.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > $O/bench_line_cfg5.json 2> $O/bench_line_cfg5.err
for C in 4 5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$C.csv \
      python bench.py --config $C --no-cpu --no-e2e --steps 1 --warmup 3 > $O/ncu_launch_$C.log 2>&1
  python tools/ncu_summary_launches.py $O/launches_cfg$C.csv > $O/launches_cfg${C}_summary.txt
  gzip -f $O/launches_cfg$C.csv
done
cap() {  # cap NAME REGEX SKIP CFG B
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $O/full_$1 \
      python tools/run_cfg.py $4 $5 > $O/ncu_full_$1.log 2>&1
  python tools/ncu_summary.py $O/full_$1.ncu-rep > $O/full_$1_summary.txt 2>&1
  ncu -i $O/full_$1.ncu-rep --page raw --csv > $O/full_$1_raw_all.csv 2>&1
  python tools/ncu_raw_pick.py $O/full_$1_raw_all.csv 'dram__bytes_(read|write)\.sum$' 'sm__pipe_tensor.*cycles_active.*pct' 'sm__pipe_fma_cycles_active.*pct' '^gpu__time_duration\.sum$' 'sm__throughput\.avg\.pct' 'launch__(registers|occupancy_limit)' 'smsp__issue_active.avg.pct' > $O/full_$1_raw.txt 2>&1
  rm -f $O/full_$1_raw_all.csv
  python tools/ncu_lines.py $O/full_$1.ncu-rep $2 --top 20 > $O/full_$1_lines.txt 2>&1
  rm -f $O/full_$1.ncu-rep
}
for k in bnd_tc_update kr_gemm bnd_pdiag bnd_prows bnd_solve bnd_resid bnd_update bnd_sgemm; do cap $k $k 12 4 2048; done
cap ipm_cfg2 ipm_kernel 0 2 1024
ls -la $O
