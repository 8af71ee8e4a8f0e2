#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_parity.py -k "batched_engine or cfg4 or large_n_global or forced_matches" > gpurun_out/d11_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/d11_pytest.log
timeout 900 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_memcheck.py tests/test_gpu_cfg5.py > gpurun_out/d11b_pytest.log 2>&1; echo "pytest2 rc=$?"; tail -2 gpurun_out/d11b_pytest.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d11.log 2>&1; echo "bench rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/d11.log | head -1)"
bash tools/ncu_launches.sh 4 2048 c4e 2>/dev/null | head -10
