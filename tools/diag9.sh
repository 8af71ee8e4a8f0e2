#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_parity.py -k "batched_engine or cfg4 or large_n_global or forced_matches" tests/test_gpu_memcheck.py > gpurun_out/d9_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/d9_pytest.log
for nl in 1 2 3; do
QPB200_BLANES=$nl timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d9_b$nl.log 2>&1; echo "lanes $nl rc=$?"; grep -o '"value": [0-9.]*' gpurun_out/d9_b$nl.log | head -1
done
