#!/bin/bash
# TMA-fed Schur update: path-4 parity tests, then cfg4/cfg5 bench old vs TMA (stages x tiles per CTA)
mkdir -p gpurun_out
TAG=${1:-tma}
QPB200_TMA_STAGES=33 timeout 1200 python -m pytest tests/test_gpu_chord.py tests/test_gpu_parity.py tests/test_gpu_memcheck.py tests/test_gpu_cfg5.py -k "chord or cfg4 or large_n or batched or memcheck or guard or cfg5 or global" -q -p no:cacheprovider --timeout 900 -rs -x > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest_rc=$?"; tail -4 gpurun_out/pytest_${TAG}.log
for cfg in 4 5; do for v in old 22 42 23 33; do
  if [ $v == old ]; then export QPB200_TC_OLD=1; else unset QPB200_TC_OLD; export QPB200_TMA_STAGES=$v; fi
  timeout 600 python bench.py --no-cpu --no-e2e --config $cfg --steps 5 --warmup 3 > gpurun_out/tma_${cfg}_$v.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/tma_${cfg}_$v.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print('cfg $cfg tc $v value %.1f solve %.1f bwd %.1f' % (d['value'], r['solve_ms'], r['backward_ms']))" || tail -3 gpurun_out/tma_${cfg}_$v.log
done; done
