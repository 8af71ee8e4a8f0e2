#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_chord.py tests/test_gpu_parity.py tests/test_gpu_memcheck.py tests/test_gpu_batched_gemm.py tests/test_gpu_cfg5.py tests/test_gpu_tma.py -k "chord or cfg4 or batched or memcheck or large_n or cfg5 or tma or global or gemm" -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_fuse.log 2>&1
echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_fuse.log
bash tools/exp_env.sh 4 - QPB200_NO_FUSE=1
bash tools/exp_env.sh 5 - QPB200_NO_FUSE=1
