#!/bin/bash
# lane-count experiment on configs 4 and 5 (QPB200_BLANES overrides the heuristic)
for cfg in 5 4; do for ln in 2 3 4; do
QPB200_BLANES=$ln timeout 600 python bench.py --no-cpu --no-e2e --config $cfg --steps 5 --warmup 3 > gpurun_out/lanes_${cfg}_${ln}.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/lanes_${cfg}_${ln}.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print('cfg $cfg lanes $ln value %.1f solve %.1f bwd %.1f' % (d['value'], r['solve_ms'], r['backward_ms']))"
done; done
