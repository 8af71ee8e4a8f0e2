#!/bin/bash
# full GPU check: pytest -m gpu, smoke, default bench line
mkdir -p gpurun_out
TAG=${1:-full}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest_rc=$?"; grep -E "passed|failed" gpurun_out/pytest_${TAG}.log | tail -3; grep -E "^FAILED" gpurun_out/pytest_${TAG}.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke_rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench_rc=$?"; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-400
