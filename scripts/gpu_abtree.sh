#!/bin/bash
# A/B of the working tree against prevtree/ (scripts/mk_prevtree.sh), same box, two rounds.
# usage: bash scripts/gpu_abtree.sh TAG "config ..." ["ENV=..." ...]   (each extra ENV adds a variant of the working tree)
TAG=$1; CONFIGS=${2:-llama8b_block}; shift 2
mkdir -p gpurun_out
run() { (cd $1 && env $2 timeout 600 python bench.py --config $3 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4))" 2>&1 | tail -1); }
{
for round in 1 2; do
for c in $CONFIGS; do
  echo "$round prev $c $(run prevtree '' $c)"
  echo "$round new $c $(run . '' $c)"
  for e in "$@"; do echo "$round new:$e $c $(run . $e $c)"; done
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
