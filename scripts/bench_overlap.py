#!/usr/bin/env python
"""NEXT-1: on-the-fly DF11 weights in a transformer-block forward.

For a stack of Llama-3.1-8B-shaped blocks, time one forward pass (the block's seven GEMMs) with
  (a) BF16 weights resident in HBM (no decode),
  (b) DF11 weights decoded right before each block (serial: decode then GEMMs),
  (c) DF11 weights decoded one block ahead on a side stream (OverlapRunner, prefetch), with an SM
      budget for the decode (df11_decompress_block_budget: the decode runs on `ctas` SMs and leaves
      the others to the GEMMs; 0 = every SM).
Prints one JSON line per token-batch size (every budget, the best one named).  GEMMs are
torch.matmul (cuBLAS); the decode is ours.

    python scripts/bench_overlap.py [--blocks 8] [--tokens 1,16,256,2048] [--budgets 0,112,96,74,56,40]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--tokens", default="1,16,256,2048")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--budgets", default="0,120,104,88,74,60,48")
    args = ap.parse_args()
    import torch

    from paper_2504_11651_b200 import df11
    from paper_2504_11651_b200.runtime import BlockWeights, OverlapRunner
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ts = workloads.config_tensors("llama8b_block", layer=0)
    hosts = [df11.encode(w) for _, w in ts]
    proto = BlockWeights.from_host(hosts, dev)
    blocks = [proto]
    for _ in range(args.blocks - 1):                     # device copies (same sizes / entropy)
        blocks.append(BlockWeights([df11.clone_device_tensor(d) for d in proto.dts]))
    resident = [[torch.from_numpy(w.reshape(-1).view(np.int16)).to(dev).view(torch.bfloat16).view(w.shape)
                 for _, w in ts] for _ in range(args.blocks)]

    def fwd(x, W):
        q, k, v, o, g, u, dn = W
        a = x @ q.T + x @ k.T.repeat(1, 4) + x @ v.T.repeat(1, 4)
        h = a @ o.T
        return (torch.nn.functional.silu(h @ g.T) * (h @ u.T)) @ dn.T

    def time_it(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / args.reps

    budgets = [int(x) for x in args.budgets.split(",")]
    serial = OverlapRunner(blocks, dev, prefetch=False)
    runners = {c: OverlapRunner(blocks, dev, prefetch=True, decode_ctas=c) for c in budgets}
    # correctness: the decoded weights equal the resident BF16 weights, for every budget
    for r in [serial] + list(runners.values()):
        for i, W in r.iterate():
            for a, b in zip(W, resident[0]):
                assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    for t in [int(x) for x in args.tokens.split(",")]:
        x0 = torch.randn(t, 4096, device=dev, dtype=torch.bfloat16) * 0.1

        def run_resident():
            x = x0
            for W in resident:
                x = fwd(x, W)
            return x

        def run_df11(r):
            def f():
                x = x0
                for _, W in r.iterate():
                    x = fwd(x, W)
                return x
            return f

        plans = [b.plan(serial.scratch[0]) for b in blocks]

        def decode_only():
            for p in plans:
                p.run()

        ms_res = time_it(run_resident)
        ms_ser = time_it(run_df11(serial))
        ms_ovl = {c: time_it(run_df11(r)) for c, r in runners.items()}
        ms_dec = time_it(decode_only)
        best = min(ms_ovl, key=ms_ovl.get)
        print(json.dumps({"tokens": t, "blocks": args.blocks, "ms_bf16_resident": ms_res,
                          "ms_df11_serial": ms_ser, "ms_df11_overlap": ms_ovl[best], "best_decode_ctas": best,
                          "ms_df11_overlap_by_ctas": {str(c): round(v, 4) for c, v in ms_ovl.items()},
                          "ms_decode_only": ms_dec,
                          "overhead_serial": ms_ser / ms_res - 1, "overhead_overlap": ms_ovl[best] / ms_res - 1,
                          "bit_exact": True, "gemm": "torch.matmul (cuBLAS)",
                          "decode": "df11_decompress_block_budget (ours)"}), flush=True)


if __name__ == "__main__":
    main()
