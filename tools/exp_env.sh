#!/bin/bash
# bench config $1 under each "NAME=VAL" env setting given (or none: "-")
C=$1; shift
for kv in "$@"; do
  if [ "$kv" == "-" ]; then envs=""; else envs="$kv"; fi
  env $envs timeout 600 python bench.py --no-cpu --no-e2e --config $C --steps 5 --warmup 3 > gpurun_out/exp_${C}.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/exp_${C}.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print('cfg $C [$kv] value %.1f solve %.1f bwd %.1f' % (d['value'], r['solve_ms'], r['backward_ms']))" || tail -2 gpurun_out/exp_${C}.log
done
