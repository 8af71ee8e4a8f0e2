#!/bin/bash
# Round-2 profile artifacts (run on the GPU box):  bash tools/make_profiles_r2.sh
# -> gpurun_out/r2/: bench lines, ncu launch list of one config-4 step, --set full
#    summaries (metrics, DRAM bytes, source-line stalls) of the batched-engine kernels
set -x
O=gpurun_out/r2; mkdir -p $O
timeout 900 python bench.py > $O/bench_line.json 2> $O/bench_line.err
timeout 900 python bench.py --config 2 > $O/bench_line_cfg2.json 2> $O/bench_line_cfg2.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu > $O/bench_line_cfg5.json 2> $O/bench_line_cfg5.err
# launch list of one timed config-4 step (cold-cache, serialised: shares, not absolutes)
python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > $O/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > $O/ncu_launch.log 2>&1
python tools/ncu_summary_launches.py $O/launches_cfg4.csv > $O/launches_cfg4_summary.txt
# one --set full capture per batched-engine kernel (a mid-solve launch of a 2048-problem run)
for k in kr_gemm bnd_tc_update bnd_pdiag bnd_prows bnd_solve bnd_resid bnd_update bnd_scatter; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o $O/full_$k \
      python tools/run_cfg.py 4 2048 > $O/ncu_full_$k.log 2>&1
  python tools/ncu_summary.py $O/full_$k.ncu-rep > $O/full_${k}_summary.txt 2>&1
  ncu -i $O/full_$k.ncu-rep --page raw --csv > $O/full_${k}_raw_all.csv 2>&1
  python tools/ncu_raw_pick.py $O/full_${k}_raw_all.csv 'dram__bytes_(read|write)\.sum$' 'sm__pipe_tensor.*cycles_active.*pct' 'sm__pipe_fma_cycles_active.*pct' '^gpu__time_duration\.sum$' 'sm__throughput\.avg\.pct' 'launch__(registers|occupancy_limit)' > $O/full_${k}_raw.txt 2>&1
  rm -f $O/full_${k}_raw_all.csv
  python tools/ncu_lines.py $O/full_$k.ncu-rep $k --top 20 > $O/full_${k}_lines.txt 2>&1
  rm -f $O/full_$k.ncu-rep
done
ls -la $O
