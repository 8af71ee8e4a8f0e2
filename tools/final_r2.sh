#!/bin/bash
# end-of-round check: pytest -m gpu, smoke, bench lines (configs 4, 2, 5) into gpurun_out/r2e/
O=gpurun_out/r2e; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs > $O/pytest.log 2>&1
echo "pytest_rc=$?"; grep -E "passed|failed" $O/pytest.log | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?"
timeout 900 python bench.py > $O/bench_line.json 2> $O/bench_line.err; echo "bench_rc=$?"
timeout 900 python bench.py --config 2 > $O/bench_line_cfg2.json 2> $O/bench_line_cfg2.err
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 > $O/bench_line_cfg5.json 2> $O/bench_line_cfg5.err; echo "cfg5_rc=$?"
for f in bench_line bench_line_cfg2 bench_line_cfg5; do
python -c "
import json
d=json.loads([l for l in open('$O/$f.json') if l.startswith('{')][-1]); r=d['roofline']
print('$f', d['config']['workload'], 'value %.1f e2e %.1f frac %.3f solve %.2f bwd %.2f cpu %s' % (d['value'], d['e2e']['value'], r['frac'], r['solve_ms'], r['backward_ms'], (d.get('cpu_baseline') or {}).get('value')))" 2>&1 | tail -1
done
