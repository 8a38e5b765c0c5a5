#!/bin/bash
# GPU fuzz sweep + the NEXT-4 variant lines with the current timing (back-to-back launches).
TAG=${1:-var2}
mkdir -p gpurun_out
{
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q 2>&1 | tail -3
for a in "--vf fp16" "--vf fp16 --format 128x16" "--vf fp8_e4m3" "--vf fp8_e5m2" "--lut-bits 5" "--lut-bits 10" "--lut-bits 12" \
         "--vf fp16 --lut-bits mono" "--vf fp8_e4m3 --lut-bits mono" "--format 128x16" "--config llama70b_block --vf fp16" \
         "--config llama70b_block --vf fp8_e4m3"; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-e2e --no-transfer --no-cpu-baseline $a 2>> gpurun_out/${TAG}_err.log | tail -1 >> gpurun_out/${TAG}_variants.jsonl
done
python -c "
import json
for l in open('gpurun_out/${TAG}_variants.jsonl'):
    d=json.loads(l); c=d['config']; r=d['roofline']; g=d.get('graph') or {}
    print(c['workload'], c['value_format'], c['lut_bits'], c['format'], round(c['bits_per_weight'],3), round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],1), 'graph', round(g.get('value',0),1))
"
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
