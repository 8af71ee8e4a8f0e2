#!/bin/bash
timeout 900 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_cfg5.py tests/test_gpu_parity.py -k "cfg5 or batched_engine or cfg4_shared or large_n_global" > gpurun_out/d13_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/d13_pytest.log
for c in 5 4 2; do
timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d13.log 2>&1; echo "cfg$c rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/d13.log | head -1)"
done
