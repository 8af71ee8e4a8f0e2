#!/bin/bash
# One gpurun call: GPU parity tests, a short bench, optional ncu capture.
# usage: tools/gpu_check.sh TAG [ncu] [pytest-args...]
TAG=${1:-run}; shift
NCU=0; if [ "$1" == "ncu" ]; then NCU=1; shift; fi
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rs "$@" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest_rc=$?"; tail -15 gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1
echo "bench_rc=$?"; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-3000
if [ "$NCU" == "1" ]; then
  python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ipm_ -s 2 -c 2 -o gpurun_out/prof_${TAG} \
      python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}.log 2>&1
  echo "ncu_rc=$?"
fi
