# quick per-config device throughput (configs 2 and 3) and phase counters of config 2
bash tools/exp_quick.sh
for c in 3; do timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('cfg', $c, round(r['value']))"; done
