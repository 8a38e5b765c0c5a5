#!/bin/bash
# NEXT-4 follow-up: runtime hook + variant tests, b-bit lines with SMEM-staged tables, memcheck /
# racecheck over the variant parity cases.  usage: bash scripts/gpu_next4b.sh TAG
TAG=${1:-n4b}
mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_variants.py -x -q 2>&1 | tail -3
for a in "--lut-bits 5" "--lut-bits 12" "--lut-bits 10" "--vf fp16 --lut-bits mono" "--vf fp8_e4m3 --lut-bits mono"; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-e2e --no-transfer --no-cpu-baseline $a 2>> gpurun_out/${TAG}_err.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']; r=d['roofline']
print('$a', c['value_format'], c['lut_bits'], round(c['bits_per_weight'],3), round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],1))"
done
echo "== memcheck over the variant parity cases (DF11_MAX_GRID=4)"
DF11_MAX_GRID=4 timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_variants.py -k "parity and not full_size" > /tmp/san_var.log 2>&1
echo "rc=$?"; tail -3 /tmp/san_var.log
echo "== racecheck, FP16 / FP8 cases"
DF11_MAX_GRID=2 timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_variants.py -k "value_format_parity and gauss and fast and not 1m" > /tmp/san_var_rc.log 2>&1
echo "rc=$?"; grep -E "RACECHECK SUMMARY|hazard|passed|failed" /tmp/san_var_rc.log | tail -5
if [ -f paper_2504_11651_b200/lib/variants/smbar.so ]; then
  echo "== racecheck, same cases, A/B variant with a group barrier before the residual TMA refill"
  DF11_LIB=$PWD/paper_2504_11651_b200/lib/variants/smbar.so DF11_MAX_GRID=2 timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_variants.py -k "value_format_parity and gauss and fast and not 1m" > /tmp/san_var_rb.log 2>&1
  echo "rc=$?"; grep -E "RACECHECK SUMMARY|hazard|passed|failed" /tmp/san_var_rb.log | tail -5
fi
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
