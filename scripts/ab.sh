#!/bin/bash
# A/B: bench every lib/variants/*.so (plus the default lib) on CONFIGS, two rounds (noise check).
mkdir -p gpurun_out
TAG=${1:-ab}
{
for round in 1 2; do
for v in default paper_2504_11651_b200/lib/variants/*.so; do
  for c in ${CONFIGS:-llama8b_block llama70b_block flux_double_block}; do
    if [ "$v" = default ]; then L=""; else L="$v"; fi
    r=$(DF11_LIB=$L timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3))" 2>&1 | tail -1)
    echo "$round $(basename $v) $c $r"
  done
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
