#!/bin/bash
# config-4 per-rank batch of an N-GPU strong-scaling run (8192/N), lanes 1/2/4
for B in 1024 2048 4096; do for ln in 1 2 4; do
  QPB200_BLANES=$ln timeout 600 python bench.py --no-cpu --no-e2e --config 4 --batch $B --steps 5 --warmup 3 > gpurun_out/sl.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/sl.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print('B $B lanes $ln value %.1f solve %.1f bwd %.1f' % (d['value'], r['solve_ms'], r['backward_ms']))" || tail -2 gpurun_out/sl.log
done; done
