#!/bin/bash
# GPU parity tests against every lib/variants/*.so (DF11_LIB), then the A/B bench (scripts/ab.sh).
TAG=${1:-vt}
mkdir -p gpurun_out
{
for v in paper_2504_11651_b200/lib/variants/*.so; do
  echo "== $(basename $v)"
  DF11_LIB=$v timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
done
} > gpurun_out/${TAG}_vtests.log 2>&1
cat gpurun_out/${TAG}_vtests.log
CONFIGS=${CONFIGS:-llama8b_block llama70b_block} bash scripts/ab.sh ${TAG}
