#!/bin/bash
# compute-sanitizer initcheck (reads of uninitialised device memory) over small decode and encode cases.
TAG=${1:-initcheck}
mkdir -p gpurun_out
{
echo "== initcheck: parity cases of both kernels + value formats (DF11_MAX_GRID=4)"
DF11_MAX_GRID=4 timeout 2400 compute-sanitizer --tool initcheck --error-exitcode 9 python -m pytest -q -x \
  tests/test_gpu_parity.py tests/test_gpu_variants.py -k "parity_cases or (value_format_parity and not 1m)" > /tmp/i1.log 2>&1
echo "rc=$?"; tail -3 /tmp/i1.log
echo "== initcheck: GPU encoder"
timeout 1800 compute-sanitizer --tool initcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_encoder.py -k "not llama" > /tmp/i2.log 2>&1
echo "rc=$?"; tail -3 /tmp/i2.log
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
