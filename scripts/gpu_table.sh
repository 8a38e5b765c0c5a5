#!/bin/bash
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -x -q 2>&1 | tail -3
for round in 1 2; do
for c in llama8b_block llama70b_block flux_double_block matrix4096; do
  for v in prev default inkernel sw3 sw5; do
    L=""; E=""
    [ "$v" = prev ] && L=paper_2504_11651_b200/lib/variants/prev.so
    [ "$v" = inkernel ] && E="DF11_NO_PREBUILT_TABLE=1"
    [ "$v" = sw3 ] && E="DF11_SWITCH_TILES_ENV=3"
    [ "$v" = sw5 ] && E="DF11_SWITCH_TILES_ENV=5"
    r=$(env $E DF11_LIB=$L timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4))" 2>&1 | tail -1)
    echo "$round $v $c $r"
  done
done
done
} > gpurun_out/table.log 2>&1
cat gpurun_out/table.log
