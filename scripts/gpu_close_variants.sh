#!/bin/bash
# Closing re-measurement with the PDL product kernel: NEXT-4 variant lines, block batching and
# the NEXT-1 overlap benchmark.  usage: bash scripts/gpu_close_variants.sh TAG
TAG=${1:-closevar}
mkdir -p gpurun_out
for a in "--vf fp16" "--vf fp8_e4m3" "--vf fp8_e5m2" "--vf fp16 --format 128x16" "--format 128x16" "--lut-bits 5" "--lut-bits 12" \
         "--vf fp16 --lut-bits mono" "--vf fp8_e4m3 --lut-bits mono" "--config llama70b_block --vf fp16" \
         "--config llama70b_block --vf fp8_e4m3"; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-e2e --no-transfer --no-cpu-baseline $a >> gpurun_out/${TAG}_variants.jsonl 2>> gpurun_out/${TAG}_err.log
done
timeout 900 python scripts/bench_batching.py > gpurun_out/${TAG}_batching.jsonl 2>> gpurun_out/${TAG}_err.log
timeout 1200 python scripts/bench_overlap.py > gpurun_out/${TAG}_overlap.jsonl 2>> gpurun_out/${TAG}_err.log
python -c "
import json,sys
for l in open('gpurun_out/${TAG}_variants.jsonl'):
    d=json.loads(l); c=d['config']; r=d['roofline']
    print(c['workload'], c['value_format'], c['lut_bits'], c['format'], round(c['bits_per_weight'],3), round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],1))
"
cat gpurun_out/${TAG}_batching.jsonl | cut -c1-220
cat gpurun_out/${TAG}_overlap.jsonl | cut -c1-400
tail -3 gpurun_out/${TAG}_err.log
