#!/bin/bash
# GPU encoder for every value format: parity tests + per-block timing on the Llama-8B block.
TAG=${1:-encvf}
mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests/test_gpu_encoder.py -x -q 2>&1 | tail -3
for vf in bf16 fp16 fp8_e4m3 fp8_e5m2; do
  timeout 600 python scripts/bench_encode.py --configs llama8b_block --vf $vf --host 2>&1 | tail -1
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
