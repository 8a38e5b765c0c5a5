#!/bin/bash
# A/B: griddepcontrol.wait before the first global write of each tile (pdllate.so, -DSP12_PDL_LATE)
# vs after the table build (the product); GPU parity under the variant first.
TAG=${1:-abpdllate}
V=paper_2504_11651_b200/lib/variants
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=d.get('graph') or {}; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2), 'graph', round(g.get('value',0),1))" 2>&1 | tail -1; }
{
echo "== parity under pdllate.so"
DF11_LIB=$V/pdllate.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for round in 1 2; do
for c in llama8b_block matrix4096 flux_single_block flux_double_block llama70b_block; do
  echo "$round base $c $(run --config $c)"
  echo "$round pdl  $c $(DF11_LIB=$V/pdllate.so run --config $c)"
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
