#!/bin/bash
# One ncu --set full capture of fast_kernel on the Llama-8B block (no tests / bench).
TAG=${1:-prof}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"(fast|sp|sp12)_kernel" -s 2 -c 1 -o gpurun_out/${TAG}_prof \
  python bench.py --kernel fast --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-transfer > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
