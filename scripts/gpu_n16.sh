#!/bin/bash
mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "n16 or split or fast" 2>&1 | tail -4
for f in 256x8 128x16; do for c in llama8b_block llama70b_block; do
  timeout 600 python bench.py --config $c --format $f --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-transfer 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', '$c', round(d['value'],1), round(d['roofline']['frac'],4), round(d['config']['bits_per_weight'],4), d['config']['df11_bytes_per_gpu'])"
done; done
} > gpurun_out/n16.log 2>&1
cat gpurun_out/n16.log
