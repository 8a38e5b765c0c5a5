#!/bin/bash
# NEXT-3 GPU encoder: tests + encode-time bench.
mkdir -p gpurun_out
TAG=${1:-enc}
{
timeout 900 python -m pytest tests/test_gpu_encoder.py -q -x 2>&1 | tail -15
timeout 900 python scripts/bench_encode.py --configs llama8b_block,llama70b_block --host 2>&1 | tail -5
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
