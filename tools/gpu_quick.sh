#!/bin/bash
# path-4 parity subset, then the given bench experiments: tools/gpu_quick.sh "CFG ENV..." ...
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_chord.py tests/test_gpu_parity.py tests/test_gpu_memcheck.py tests/test_gpu_batched_gemm.py tests/test_gpu_cfg5.py tests/test_gpu_tma.py -k "chord or cfg4 or batched or memcheck or large_n or cfg5 or tma or global or gemm" -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_quick.log 2>&1
echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_quick.log
for e in "$@"; do bash tools/exp_env.sh $e; done
