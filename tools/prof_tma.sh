#!/bin/bash
# ncu --set full of one mid-solve launch of the opt-in TMA Schur update (config 4, 2048 problems)
mkdir -p gpurun_out
QPB200_TC_TMA=${VARIANT:-42} bash tools/ncu_kernel.sh bnd_tc_update 30 4 2048 tma_ws
head -30 gpurun_out/sum_tma_ws.txt; head -30 gpurun_out/lines_tma_ws.txt
