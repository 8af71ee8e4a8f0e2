QPB200_PHASE_PROFILE=1 PYTHONPATH=. timeout 200 python tools/prof_cfg.py 2 1024 2>&1 | grep -E "sub-phases|phase cycles" | tail -2
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(round(r['value']), r['roofline']['solve_ms'], r['roofline']['backward_ms'], r['e2e']['value'])"; done
