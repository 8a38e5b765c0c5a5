#!/bin/bash
# ncu --set full capture of the product kernel (default lib) on the Llama-8B block.  usage: bash scripts/gpu_prof_default.sh TAG
TAG=$1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"(sp12|wt)_kernel" -s 2 -c 1 -o gpurun_out/${TAG}_prof \
  python bench.py --kernel fast --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-transfer > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
