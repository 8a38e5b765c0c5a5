#!/bin/bash
# A/B of several built trees (directories with their own binding + library) on one box, two rounds.
# usage: bash scripts/gpu_abtrees.sh TAG "config ..." dir1 dir2 ...   ("." = the working tree)
TAG=$1; CONFIGS=$2; shift 2
mkdir -p gpurun_out
run() { (cd $1 && timeout 600 python bench.py --config $2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4))" 2>&1 | tail -1); }
{
for round in 1 2; do
for c in $CONFIGS; do
  for d in "$@"; do echo "$round $d $c $(run $d $c)"; done
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
