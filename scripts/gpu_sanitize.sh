#!/bin/bash
# compute-sanitizer passes over small decode cases (bounded by timeouts); the exit code printed is
# compute-sanitizer's own (--error-exitcode 9 on any report), not the pipeline's.
# usage: bash scripts/gpu_sanitize.sh [TAG]   (the SP12_SM_BARRIER A/B variant must be built as
# paper_2504_11651_b200/lib/variants/smbar.so for the racecheck comparison)
mkdir -p gpurun_out
TAG=${1:-san}
{
for tool in memcheck racecheck synccheck; do
  echo "== $tool (product kernel)"
  DF11_MAX_GRID=2 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py fast > /tmp/san_$tool.log 2>&1
  echo "rc=$?"
  tail -4 /tmp/san_$tool.log
done
if [ -f paper_2504_11651_b200/lib/variants/smbar.so ]; then
  echo "== racecheck (A/B variant: group barrier before the PackedSignMantissa TMA refill)"
  DF11_LIB=paper_2504_11651_b200/lib/variants/smbar.so DF11_MAX_GRID=2 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_case.py fast > /tmp/san_rb.log 2>&1
  echo "rc=$?"
  tail -4 /tmp/san_rb.log
fi
echo "== memcheck over test_corrupt_metadata_never_faults (both kernels)"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_parity.py -k corrupt > /tmp/san_corrupt.log 2>&1
echo "rc=$?"
tail -4 /tmp/san_corrupt.log
echo "== memcheck over every parity case of both kernels (DF11_MAX_GRID=4)"
DF11_MAX_GRID=4 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_parity.py -k "parity_cases" > /tmp/san_parity.log 2>&1
echo "rc=$?"
tail -4 /tmp/san_parity.log
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
