#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fast or block or split" 2>&1 | tail -2 > gpurun_out/fb.log
bash scripts/gpu_abtree.sh fb_ab "llama8b_block llama70b_block flux_double_block" DF11_FEEDBACK=0 >> gpurun_out/fb.log 2>&1
cat gpurun_out/fb.log
