#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_parity.py -k "batched_engine or cfg4_shared_subset or large_n_global or forced_matches or cfg4_full" > gpurun_out/d4_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/d4_pytest.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d4_bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/d4_bench.log
bash tools/ncu_launches.sh 4 2048 c4c
