#!/bin/bash
# ncu of the GPU encoder on the Llama-8B block: launch list + full capture of pack_kernel.
mkdir -p gpurun_out
TAG=${1:-encprof}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python scripts/bench_encode.py --configs llama8b_block --reps 1 > gpurun_out/${TAG}_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 20 -c 1 -o gpurun_out/${TAG}_pack \
  python scripts/bench_encode.py --configs llama8b_block --reps 1 > gpurun_out/${TAG}_p.log 2>&1
tail -3 gpurun_out/${TAG}_p.log
