#!/bin/bash
# Round artifacts: full bench line, ncu launch list, one ncu --set full capture
# of the two hot kernels.  usage: tools/gpu_artifacts.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/gpu_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_full_${TAG}.log 2>&1; echo "bench_rc=$?"
tail -1 gpurun_out/bench_full_${TAG}.log | cut -c1-3000
python bench.py --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launch_rc=$?"
python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/plain2_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ipm_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG} \
    python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu_rc=$?"
# the same kernel serves both calls (solve launch first, backward launch second)
ncu --set full --clock-control none --import-source on -k regex:ipm_kernel -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd \
    python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_full_bwd_${TAG}.log 2>&1; echo "ncu_bwd_rc=$?"
