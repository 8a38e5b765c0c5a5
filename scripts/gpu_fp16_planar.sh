#!/bin/bash
# FP16 planar residual layout (R25: byte plane + 3-bit plane): GPU parity (variants, fuzz, encoder,
# alg1) and the FP16 bench lines.
TAG=${1:-fp16planar}
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer --no-graph "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2), round(d['config']['bits_per_weight'],3))" 2>&1 | tail -1; }
{
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fuzz.py tests/test_gpu_encoder.py -q -x 2>&1 | tail -4
for round in 1 2; do
  for a in "--vf fp16" "--vf fp16 --format 128x16" "--vf bf16"; do echo "$round $a $(run $a)"; done
done
for a in "--vf fp16 --lut-bits mono" "--config llama70b_block --vf fp16"; do echo "$a $(run $a)"; done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
