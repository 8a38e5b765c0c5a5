#!/bin/bash
# All BASELINE configs on one GPU (model sweeps at N=1; the 405B config decodes its 1/8 shard).
mkdir -p gpurun_out
TAG=${1:-configs}
{
nproc; free -g | head -2
for c in matrix4096 llama8b_block flux_double_block flux_single_block llama70b_block; do
  timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1
done
timeout 1500 python bench.py --config llama70b_model --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -2
timeout 1500 python bench.py --config llama405b_model --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -2
} > gpurun_out/${TAG}.log 2>&1
tail -3 gpurun_out/${TAG}.log
