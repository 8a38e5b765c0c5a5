#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runtime.py -x -q 2>&1 | tail -3 > gpurun_out/r2n1.log
timeout 1500 python scripts/bench_overlap.py --tokens 1,16,256,2048 > gpurun_out/r2n1_overlap.jsonl 2>> gpurun_out/r2n1.log
cat gpurun_out/r2n1.log gpurun_out/r2n1_overlap.jsonl
