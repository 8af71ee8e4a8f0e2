#!/bin/bash
# ncu --set full of one mid-solve Schur-update launch (TMA warp-specialised kernel)
mkdir -p gpurun_out
QPB200_TMA_STAGES=${STAGES:-4} bash tools/ncu_kernel.sh bnd_tc_update 30 4 2048 tma_ws
python tools/ncu_raw_pick.py 2>/dev/null | head -1
head -30 gpurun_out/sum_tma_ws.txt; head -30 gpurun_out/lines_tma_ws.txt
