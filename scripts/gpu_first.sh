#!/bin/bash
# First GPU pass: smoke, GPU parity (Alg. 1 kernel), bench, ncu launch list + one full capture.
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fast" 2>&1 | tail -15
timeout 600 python bench.py --kernel alg1 --steps 100 --warmup 5 2>&1 | tail -3
} > gpurun_out/first.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches_alg1.csv \
  python bench.py --kernel alg1 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:alg1 -s 2 -c 1 -o gpurun_out/prof_alg1 \
  python bench.py --kernel alg1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/first.log
