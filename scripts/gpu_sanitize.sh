#!/bin/bash
# compute-sanitizer passes over small decode cases (bounded by timeouts).
mkdir -p gpurun_out
TAG=${1:-san}
{
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  DF11_MAX_GRID=2 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py fast 2>&1 | tail -4
  echo "rc=$?"
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
