#!/bin/bash
# Closing sanitizer pass on the final build: memcheck over the parity, variant, fuzz and encoder tests
# (DF11_MAX_GRID=4: every group walks many tiles and tensor switches), racecheck / synccheck on small
# cases of every value format.  The exit codes printed are compute-sanitizer's own (--error-exitcode 9).
TAG=${1:-sanfinal}
mkdir -p gpurun_out
{
echo "== memcheck: parity + variants + fuzz (DF11_MAX_GRID=4)"
DF11_MAX_GRID=4 timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x \
  tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fuzz.py -k "not full_size and not llama8b and not 405b and not embed" > /tmp/s1.log 2>&1
echo "rc=$?"; tail -3 /tmp/s1.log
echo "== memcheck: GPU encoder tests"
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_encoder.py -k "not llama" > /tmp/s2.log 2>&1
echo "rc=$?"; tail -3 /tmp/s2.log
for tool in racecheck synccheck; do
  echo "== $tool: value-format parity (product kernel, gauss / escapes / 1-bit cases, DF11_MAX_GRID=2)"
  DF11_MAX_GRID=2 timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -x tests/test_gpu_variants.py \
    -k "value_format_parity and fast and (gauss- or escapes or constant_1bit) and not 1m" > /tmp/s3.log 2>&1
  echo "rc=$?"; grep -E "SUMMARY|passed|failed|hazard" /tmp/s3.log | tail -6
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
