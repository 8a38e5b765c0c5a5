#!/bin/bash
# A/B: one REDUX.OR vote per checked decode step (redux.so) and kFirst 5 / 7 (first5.so, first7.so)
# vs the product kernel.
TAG=${1:-abredux}
V=paper_2504_11651_b200/lib/variants
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 400 --warmup 10 --no-e2e --no-cpu-baseline --no-transfer --no-graph "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2))" 2>&1 | tail -1; }
{
DF11_LIB=$V/redux.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k fast 2>&1 | tail -1
for round in 1 2; do
for c in llama8b_block flux_double_block; do
  echo "$round base $c $(run --config $c)"
  for v in redux first5 first7; do echo "$round $v $c $(DF11_LIB=$V/$v.so run --config $c)"; done
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
