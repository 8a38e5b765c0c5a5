#!/bin/bash
# BASELINE configs[2] and [4] on one GPU (whole-model sweeps) + the realism variants, closing timing.
TAG=${1:-models}
mkdir -p gpurun_out
{
for a in "--config llama70b_model --steps 3 --warmup 1" "--config llama405b_model --steps 3 --warmup 1" \
         "--dist t5 --steps 200 --warmup 5" "--dist sigma-lu --steps 200 --warmup 5"; do
  timeout 1500 python bench.py $a --no-e2e --no-cpu-baseline --no-transfer 2>>gpurun_out/${TAG}_err.log | tail -1
done
} > gpurun_out/${TAG}.jsonl
python -c "
import json
for l in open('gpurun_out/${TAG}.jsonl'):
    d=json.loads(l); c=d['config']; r=d['roofline']
    print(c['workload'], c.get('dist',''), round(d['value'],1), round(r['frac'],4), d['ms_per_step'])
"
tail -3 gpurun_out/${TAG}_err.log
