#!/bin/bash
# A/B: warp-specialised kernel with setmaxnreg register redistribution (variants built from a tree with
# decode_ws.cu restored; ws_a: no setmaxnreg, ws_b: decode warps 72 / merge warps 56 registers at 1 024
# threads, ws_c: 768 threads, decode 96 / merge 64) against the product kernel.
TAG=${1:-abwsreg}
V=paper_2504_11651_b200/lib/variants
mkdir -p gpurun_out
run() { timeout 300 python bench.py --config $1 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer --no-graph 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2))" 2>&1 | tail -1; }
{
for v in ws_b ws_c; do
  echo "== $v parity (no 1-bit-code cases)"
  DF11_LIB=$V/$v.so DF11_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "(parity_cases and fast and not notable and not constant_1bit and not two_symbol and not one_bit) or (full_size and fast)" 2>&1 | tail -2
done
for round in 1 2; do
for c in llama8b_block llama70b_block flux_double_block; do
  echo "$round sp12 $c $(run $c)"
  for v in ws_a ws_b ws_c; do echo "$round $v $c $(DF11_LIB=$V/$v.so DF11_WS=1 run $c)"; done
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
