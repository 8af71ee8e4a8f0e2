#!/bin/bash
# register-staged vs TMA Schur update at one lane / default lanes
for cfg in 4 5; do for ln in 1 d; do for v in old 22 42; do
  if [ $v == old ]; then export QPB200_TC_OLD=1; unset QPB200_TMA_STAGES; else unset QPB200_TC_OLD; export QPB200_TMA_STAGES=$v; fi
  if [ $ln == 1 ]; then export QPB200_BLANES=1; else unset QPB200_BLANES; fi
  timeout 600 python bench.py --no-cpu --no-e2e --config $cfg --steps 5 --warmup 3 > gpurun_out/tl_${cfg}_${ln}_$v.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/tl_${cfg}_${ln}_$v.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print('cfg $cfg lanes $ln tc $v value %.1f solve %.1f bwd %.1f' % (d['value'], r['solve_ms'], r['backward_ms']))" || tail -2 gpurun_out/tl_${cfg}_${ln}_$v.log
done; done; done
