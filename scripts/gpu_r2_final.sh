#!/bin/bash
# Round-2 closing evidence on one box: smoke + every GPU test, the default bench line (e2e, cpu
# baseline on all host cores, transfer baseline, CUDA-graph replay), the reference arm, every config,
# the ncu launch list of the bench command and one --set full capture of the product kernel.
TAG=${1:-r2final}
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv,noheader
lscpu | grep -E "Model name|^CPU\(s\)"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4
} > gpurun_out/${TAG}_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${TAG}_ref.jsonl 2> gpurun_out/${TAG}_ref.err
for c in matrix4096 llama70b_block flux_double_block flux_single_block llama405b_block; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-transfer --no-e2e >> gpurun_out/${TAG}_configs.jsonl 2>> gpurun_out/${TAG}_bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-transfer --no-graph > /dev/null 2>&1
bash scripts/gpu_prof_only.sh ${TAG}
cat gpurun_out/${TAG}_tests.log; tail -c 1500 gpurun_out/${TAG}_bench.jsonl; tail -c 400 gpurun_out/${TAG}_ref.jsonl; tail -5 gpurun_out/${TAG}_bench.err
