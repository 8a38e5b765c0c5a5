#!/bin/bash
# NEXT-4 format variants on one box: GPU parity of the variants, the full GPU suite, an A/B of the
# BF16 product kernel against prevtree/ (the previous revision), and one bench line per variant.
mkdir -p gpurun_out
TAG=${1:-next4}
{
echo "== variant parity"
timeout 1200 python -m pytest tests/test_gpu_variants.py -x -q 2>&1 | tail -15
echo "== full GPU suite"
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
echo "== A/B BF16 (prevtree = previous revision, . = this tree)"
bash scripts/gpu_abtrees.sh ${TAG}_ab "llama8b_block llama70b_block" prevtree . 2>&1
echo "== variant bench lines"
for a in "--vf fp16" "--vf fp8_e4m3" "--vf fp8_e5m2" "--lut-bits 5" "--lut-bits 12" "--vf fp16 --lut-bits mono" "--vf fp8_e4m3 --format 128x16"; do
  echo "-- $a"
  timeout 900 python bench.py --steps 200 --warmup 5 --no-e2e --no-transfer --no-cpu-baseline $a 2>&1 | tail -1
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
