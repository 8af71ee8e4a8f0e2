#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_chord.py tests/test_gpu_parity.py tests/test_gpu_memcheck.py tests/test_gpu_multirank.py -k "chord or cfg4 or batched or memcheck or shared or multirank" -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_pre.log 2>&1
echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_pre.log
for v in 0 1; do
  if [ $v == 1 ]; then export QPB200_NO_PRE=1; fi
  timeout 600 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/pre_$v.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/pre_$v.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print('no_pre=$v value %.1f solve %.1f bwd %.1f iters %.3f riters %.3f' % (d['value'], r['solve_ms'], r['backward_ms'], d['solver']['iters_mean'], d['solver']['relax_iters_mean']))" || tail -3 gpurun_out/pre_$v.log
done
