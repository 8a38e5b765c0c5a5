#!/bin/bash
# ncu --set full capture of the product kernel from a variant lib.  usage: bash scripts/gpu_prof_var.sh TAG VARIANT
TAG=$1; V=$2
mkdir -p gpurun_out
DF11_LIB=paper_2504_11651_b200/lib/variants/$V.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:"(sp12|wt)_kernel" -s 2 -c 1 -o gpurun_out/${TAG}_prof \
  python bench.py --kernel fast --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-transfer > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
