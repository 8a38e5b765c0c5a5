#!/bin/bash
# Quick perf check of a few configs (no tests).
mkdir -p gpurun_out
TAG=${1:-quick}
{
for c in ${CONFIGS:-llama8b_block flux_double_block flux_single_block matrix4096}; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],1), 'GB/s', round(d['ms_per_step'],4),'ms', 'frac', round(d['roofline']['frac'],3))"
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
