#!/bin/bash
# A/B: FP16 / FP8 merge loop with a warp-uniform trip count (this tree) vs the per-unit loop (variant
# oldmerge.so); GPU parity of the variants first.
TAG=${1:-abvf}
V=paper_2504_11651_b200/lib/variants
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer --no-graph "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), round(r['avg_launch_us'],2))" 2>&1 | tail -1; }
{
echo "== variant parity"
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
for round in 1 2; do
for a in "--vf fp16" "--vf fp8_e4m3" "--vf fp8_e5m2" "--vf fp16 --format 128x16" "--vf bf16"; do
  echo "$round new  $a $(run $a)"
  echo "$round old  $a $(DF11_LIB=$V/oldmerge.so run $a)"
done
done
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
