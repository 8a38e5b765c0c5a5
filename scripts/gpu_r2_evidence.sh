#!/bin/bash
# Round-2 evidence pass: full-size parity tests, default bench line (e2e + cpu baseline), every config,
# batching and size sweep.  usage: bash scripts/gpu_r2_evidence.sh TAG
TAG=${1:-r2ev}
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv,noheader
lscpu | grep -E "Model name|^CPU\(s\)"; free -g | head -2
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -4
} > gpurun_out/${TAG}_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
for c in matrix4096 llama70b_block flux_double_block flux_single_block llama405b_block; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-transfer --no-e2e >> gpurun_out/${TAG}_configs.jsonl 2>> gpurun_out/${TAG}_bench.err
done
timeout 900 python scripts/bench_batching.py > gpurun_out/${TAG}_batching.jsonl 2>> gpurun_out/${TAG}_bench.err
timeout 900 python scripts/bench_size_sweep.py > gpurun_out/${TAG}_sweep.jsonl 2>> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_tests.log; tail -c 1500 gpurun_out/${TAG}_bench.jsonl; tail -3 gpurun_out/${TAG}_bench.err
