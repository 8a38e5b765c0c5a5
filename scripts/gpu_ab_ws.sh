#!/bin/bash
# A/B: warp-specialised kernel (DF11_WS=1) vs the product kernel; parity of the WS path first.
TAG=${1:-abws}
mkdir -p gpurun_out
run() { timeout 300 python bench.py --config $1 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer --no-graph 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2))" 2>&1 | tail -1; }
{
echo "== WS parity (no 1-bit-code cases)"
DF11_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "(parity_cases and fast and not notable and not constant_1bit and not two_symbol and not one_bit) or (full_size and fast)" 2>&1 | tail -3
for round in 1 2; do
for c in llama8b_block llama70b_block flux_double_block matrix4096; do
  echo "$round sp12 $c $(run $c)"
  echo "$round ws $c $(DF11_WS=1 run $c)"
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
