#!/bin/bash
# Functional check of the N-rank bench path on a 1-GPU box: torchrun with 2 (and 4) ranks sharing the
# GPU (DF11_BENCH_OVERSUBSCRIBE=1): gloo host group, per-rank decode, whole-job aggregation, one JSON
# line from rank 0.  The numbers are not throughputs (ranks share one GPU).
TAG=${1:-mrank}
mkdir -p gpurun_out
{
for n in 2 4; do
  echo "== $n ranks, llama8b_block"
  DF11_BENCH_OVERSUBSCRIBE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-900
done
echo "== 2 ranks, llama70b_model (strong scaling placement)"
DF11_BENCH_OVERSUBSCRIBE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config llama70b_model --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-900
} > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
