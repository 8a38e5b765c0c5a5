#!/bin/bash
# A/B: parity of the default lib (fast-kernel cases), then bench default vs variants on the 8B block
# (two rounds), then an ncu capture of the default lib.  usage: bash scripts/gpu_ab2.sh TAG VARIANT [VARIANT...]
TAG=$1; shift
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -x -q -k "fast or split or unaligned or block or scratch or corrupt" 2>&1 | tail -4
for round in 1 2; do
for v in default "$@"; do
  if [ "$v" = default ]; then L=""; else L=paper_2504_11651_b200/lib/variants/$v.so; fi
  for c in ${CONFIGS:-llama8b_block}; do
    r=$(DF11_LIB=$L timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4))" 2>&1 | tail -1)
    echo "$round $v $c $r"
  done
done
done
} > gpurun_out/${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"(sp12|wt)_kernel" -s 2 -c 1 -o gpurun_out/${TAG}_prof \
  python bench.py --kernel fast --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-transfer > gpurun_out/${TAG}_ncu.log 2>&1
cat gpurun_out/${TAG}.log
