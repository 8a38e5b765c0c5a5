#!/bin/bash
# The default bench line (full: e2e, cpu baseline, transfer, graph) + every config with the graph replay.
TAG=${1:-line}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
for c in matrix4096 llama70b_block flux_double_block flux_single_block llama405b_block; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-transfer --no-e2e >> gpurun_out/${TAG}_configs.jsonl 2>> gpurun_out/${TAG}_bench.err
done
python -c "
import json
for f in ('gpurun_out/${TAG}_bench.jsonl', 'gpurun_out/${TAG}_configs.jsonl'):
    for l in open(f):
        d=json.loads(l); c=d['config']; r=d['roofline']; g=d.get('graph') or {}
        print(c['workload'], round(d['value'],1), round(r['frac'],4), round(d['ms_per_step']*1e3,2), 'graph', round(g.get('value',0),1), round(g.get('ms_per_step',0)*1e3,2))
"
tail -3 gpurun_out/${TAG}_bench.err
