#!/bin/bash
# GPU tests (all), NEXT-1 overlap bench, compute-sanitizer on small cases.
mkdir -p gpurun_out
TAG=${1:-extra}
{
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python scripts/bench_overlap.py --blocks 8 2>&1 | tail -5
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py fast 2>&1 | tail -6
done
echo "== memcheck alg1"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_case.py alg1 2>&1 | tail -4
} > gpurun_out/${TAG}.log 2>&1
tail -30 gpurun_out/${TAG}.log
