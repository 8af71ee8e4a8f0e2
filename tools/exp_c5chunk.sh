for ch in 256 64 32 16; do for ln in 1 2; do
QPB200_BCHUNK=$ch QPB200_BLANES=$ln timeout 600 python bench.py --no-cpu --no-e2e --config 5 --steps 3 --warmup 3 > gpurun_out/c5_${ch}_${ln}.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c5_${ch}_${ln}.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print('chunk $ch lanes $ln value %.1f solve %.1f bwd %.1f' % (d['value'], r['solve_ms'], r['backward_ms']))"
done; done
