#!/bin/bash
# TMA-fed Schur update (opt-in): path-4 parity tests, then config 4/5 bench lines of the
# register-staged kernel (default) and the TMA kernel variants (QPB200_TC_TMA=42|22)
mkdir -p gpurun_out
TAG=${1:-tma}
timeout 1200 python -m pytest tests/test_gpu_tma.py -q -p no:cacheprovider --timeout 900 -rs -x > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
for cfg in 4 5; do bash tools/exp_env.sh $cfg - QPB200_TC_TMA=42 QPB200_TC_TMA=22; done
