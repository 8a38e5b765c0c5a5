#!/bin/bash
# Iteration pass: smoke, GPU parity, bench, ncu launch list + full capture of the product kernel.
# usage: bash scripts/gpu_iter.sh [tag] [pytest -k expr]
TAG=${1:-iter}
KEXPR=${2:-}
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$KEXPR" 2>&1 | tail -15
else
  timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
fi
timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-e2e --no-transfer 2>&1 | tail -1
} > gpurun_out/${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sp12_kernel" -s 2 -c 1 -o gpurun_out/${TAG}_prof \
  python bench.py --kernel fast --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-transfer > gpurun_out/${TAG}_ncu.log 2>&1
tail -8 gpurun_out/${TAG}.log
