#!/bin/bash
# A/B: prevtree (no load-time tables), this tree with and without load-time decode tables; two rounds.
TAG=${1:-abt}; CONFIGS=${2:-"llama8b_block matrix4096 flux_double_block"}
mkdir -p gpurun_out
run() { timeout 600 python bench.py --config $1 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(d['ms_per_step']*1e3,2), round(r['launch_us']['mean'],2))" 2>&1 | tail -1; }
{
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for round in 1 2; do
for c in $CONFIGS; do
  echo "$round prevtree $c $(cd prevtree && run $c)"
  echo "$round table $c $(run $c)"
  echo "$round notable $c $(run $c --no-decode-table)"
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
