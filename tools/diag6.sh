#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_parity.py -k "batched_engine or cfg4_shared_subset or large_n_global or forced_matches" > gpurun_out/d6_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/d6_pytest.log
bash tools/diag5.sh
