#!/bin/bash
# A/B of prevtree/ (previous revision), the working tree and every lib/variants/*.so, two rounds.
# Prints value (GB/s), roofline frac, ms per step (us), mean launch (us).
# usage: bash scripts/gpu_ab_lib.sh TAG "configs" [extra bench args]
TAG=$1; CONFIGS=${2:-llama8b_block}; EXTRA=$3
mkdir -p gpurun_out
run() { timeout 600 python bench.py --config $1 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer $EXTRA 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(d['ms_per_step']*1e3,2), round(r['avg_launch_us'],2))" 2>&1 | tail -1; }
{
for round in 1 2; do
for c in $CONFIGS; do
  [ -d prevtree ] && echo "$round prevtree $c $(cd prevtree && run $c)"
  echo "$round tree $c $(run $c)"
  for v in paper_2504_11651_b200/lib/variants/*.so; do [ -f $v ] && echo "$round $(basename $v) $c $(DF11_LIB=$PWD/$v run $c)"; done
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
