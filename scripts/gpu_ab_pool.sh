#!/bin/bash
# A/B of the end-of-launch tile pool: prevtree (no pool code), this tree with the pool (DF11_POOL_PCT),
# and this tree with the pool disabled; parity tests first.
TAG=${1:-abpool}; CONFIGS=${2:-"llama8b_block llama70b_block flux_double_block matrix4096"}
mkdir -p gpurun_out
run() { timeout 600 python bench.py --config $1 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer --no-graph 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2))" 2>&1 | tail -1; }
{
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fuzz.py tests/test_gpu_runtime.py -x -q 2>&1 | tail -2
for round in 1 2; do
for c in $CONFIGS; do
  echo "$round prevtree $c $(cd prevtree && run $c)"
  echo "$round pool5 $c $(DF11_POOL_PCT=5 run $c)"
  echo "$round pool3 $c $(DF11_POOL_PCT=3 run $c)"
  echo "$round pool8 $c $(DF11_POOL_PCT=8 run $c)"
  echo "$round nopool $c $(DF11_POOL_PCT=0 run $c)"
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
