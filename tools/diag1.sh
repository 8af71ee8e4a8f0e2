#!/bin/bash
# round-2 first diagnostics: unfloored parity, cfg4 bench + phase profile
mkdir -p gpurun_out
timeout 900 python tools/parity_diag.py > gpurun_out/diag_parity.log 2>&1; echo "diag rc=$?"
timeout 300 python bench.py --config 4 --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/diag_bench4.log 2>&1; echo "b4 rc=$?"
QPB200_PHASE_PROFILE=1 timeout 300 python tools/run_cfg.py 4 1184 > gpurun_out/diag_prof4.log 2>&1; echo "p4 rc=$?"
QPB200_PHASE_PROFILE=1 timeout 300 python tools/run_cfg.py 2 1024 > gpurun_out/diag_prof2.log 2>&1; echo "p2 rc=$?"
