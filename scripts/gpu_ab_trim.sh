#!/bin/bash
# A/B: grid trimming for small launches (DF11_TRIM_ROUNDS = 0 off, 4 default, 8) with the PDL kernel.
TAG=${1:-abtrim}
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 400 --warmup 10 --no-e2e --no-cpu-baseline --no-transfer "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=d.get('graph') or {}; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2), 'graph', round(g.get('value',0),1))" 2>&1 | tail -1; }
{
DF11_TRIM_ROUNDS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast" 2>&1 | tail -1
for round in 1 2; do
for c in matrix4096 flux_single_block llama8b_block; do
  for t in 0 4 8; do echo "$round trim=$t $c $(DF11_TRIM_ROUNDS=$t run --config $c)"; done
done
done
for t in 0 4; do echo "== size sweep trim=$t"; DF11_TRIM_ROUNDS=$t timeout 600 python scripts/bench_size_sweep.py --min-log2 20 --max-log2 26 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['log2'], round(d['decode_us'],2), round(d['decode_gbs'],1), d['bit_exact'])"; done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
