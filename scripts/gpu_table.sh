#!/bin/bash
# Load-time decode table: parity (with / without), A/B of with vs without on the configs.
TAG=${1:-tab}
mkdir -p gpurun_out
{
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for c in llama8b_block matrix4096 flux_double_block llama70b_block; do
  for r in 1 2; do
    for mode in table notable; do
      if [ $mode = notable ]; then E="--no-decode-table"; else E=""; fi
      timeout 600 python bench.py $E --config $c --steps 200 --warmup 5 --no-e2e --no-transfer --no-cpu-baseline 2>>gpurun_out/${TAG}_err.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c', '$mode', '$r', round(d['value'],1), round(r['frac'],4), round(d['ms_per_step']*1e3,2), round(r['launch_us']['mean'],2))"
    done
  done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
