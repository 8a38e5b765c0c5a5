#!/bin/bash
# NEXT-4 evidence: every GPU test, one bench line per format variant, and one ncu --set full capture
# of the product kernel for FP16 and FP8 E4M3.  usage: bash scripts/gpu_next4_evidence.sh TAG
TAG=${1:-n4ev}
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
} > gpurun_out/${TAG}_tests.log 2>&1
for a in "" "--vf fp16" "--vf fp8_e4m3" "--vf fp8_e5m2" "--vf fp16 --format 128x16" "--lut-bits 5" "--lut-bits 12" \
         "--vf fp16 --lut-bits mono" "--vf fp8_e4m3 --lut-bits mono" "--config llama70b_block --vf fp16" \
         "--config llama70b_block --vf fp8_e4m3"; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-e2e --no-transfer --no-cpu-baseline $a >> gpurun_out/${TAG}_variants.jsonl 2>> gpurun_out/${TAG}_err.log
done
for vf in fp16 fp8_e4m3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sp12_kernel" -s 2 -c 1 -o gpurun_out/${TAG}_${vf}_prof \
    python bench.py --vf $vf --kernel fast --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-transfer > gpurun_out/${TAG}_${vf}_ncu.log 2>&1
  tail -1 gpurun_out/${TAG}_${vf}_ncu.log
done
cat gpurun_out/${TAG}_tests.log
python -c "
import json,sys
for l in open('gpurun_out/${TAG}_variants.jsonl'):
    d=json.loads(l); c=d['config']; r=d['roofline']
    print(c['workload'], c['value_format'], c['lut_bits'], c['format'], round(c['bits_per_weight'],3), round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],1))
"
