#!/bin/bash
# A/B (closing round 2): PDL wait after the compaction (variant aftercompact.so) and the planner's
# tensor-switch cost (DF11_SWITCH_TILES_ENV 6 / 9 / 12) with the PDL product kernel.
TAG=${1:-abmisc}
V=paper_2504_11651_b200/lib/variants
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 400 --warmup 10 --no-e2e --no-cpu-baseline --no-transfer --no-graph "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2))" 2>&1 | tail -1; }
{
DF11_LIB=$V/aftercompact.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -q -x 2>&1 | tail -1
for round in 1 2; do
for c in llama8b_block flux_double_block matrix4096; do
  echo "$round base $c $(run --config $c)"
  echo "$round aftercompact $c $(DF11_LIB=$V/aftercompact.so run --config $c)"
  for sw in 6 12; do echo "$round switch=$sw $c $(DF11_SWITCH_TILES_ENV=$sw run --config $c)"; done
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
