#!/usr/bin/env python
"""Block batching evidence ("decompress all ... matrices within a transformer block as a single
batch"): one df11_decompress_block launch per block vs one
df11_decompress launch per tensor, each issued from Python and captured in a CUDA graph (the graph
removes the host's per-call cost, so the remaining gap is GPU-side: launch gaps, small grids, tails).
One JSON line per (config, mode).  Inputs rotate over device copies until a step sequence moves >= 4x
L2, so no timed launch reads its inputs from L2.

    python scripts/bench_batching.py [--configs llama8b_block flux_double_block flux_single_block]
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
    ap.add_argument("--configs", nargs="+", default=["llama8b_block", "flux_double_block", "flux_single_block"])
    ap.add_argument("--steps", type=int, default=30)
    args = ap.parse_args()
    import torch

    from paper_2504_11651_b200 import df11
    dev = torch.device("cuda", 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    l2 = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20) or (126 << 20))
    for cfg in args.configs:
        ts = workloads.config_tensors(cfg)
        hs = [df11.encode(w) for _, w in ts]
        base = [df11.to_device(h, dev) for h in hs]
        N = sum(h.num_elements for h in hs)
        algo = sum(d.compressed_bytes for d in base) + 2 * N
        copies = 1 if algo >= 4 * l2 else -(-4 * l2 // algo)
        sets = [base] + [[df11.clone_device_tensor(d) for d in base] for _ in range(copies - 1)]
        for dts in sets:                                   # every copy decodes bit-exactly
            outs = df11.decompress_block(dts)
            torch.cuda.synchronize()
            for (name, w), o in zip(ts, outs):
                assert torch.equal(o.reshape(-1).view(torch.int16),
                                   torch.from_numpy(w.reshape(-1).view(np.int16)).to(dev)), (cfg, name)
        plans = [df11.BlockPlan(dts) for dts in sets]

        def batched(i):
            plans[i % copies].run()

        def per_tensor(i):
            for d in sets[i % copies]:
                df11.decompress(d)

        for mode, fn, launches in (("batched", batched, 1), ("per_tensor", per_tensor, len(hs))):
            for graph in (False, True):
                stream = torch.cuda.Stream(dev)
                stream.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.stream(stream):
                    for i in range(3):
                        fn(i)
                    torch.cuda.synchronize()
                    if graph:
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=stream):
                            for i in range(args.steps):
                                fn(i)
                        g.replay()
                        torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    if graph:
                        g.replay()
                    else:
                        for i in range(args.steps):
                            fn(i)
                    b.record(stream)
                    torch.cuda.synchronize()
                us = a.elapsed_time(b) * 1e3 / args.steps
                print(json.dumps({"config": cfg, "mode": mode + ("+cuda_graph" if graph else "+python_calls"),
                                  "tensors": len(hs), "launches_per_step": launches, "us_per_step": round(us, 2),
                                  "gbs_bf16": round(2 * N / us / 1e3, 1), "frac_of_measured_hbm": round(algo / us / 1e3 / peak, 4),
                                  "l2_copies": copies, "bf16_bytes": 2 * N, "algorithmic_bytes": algo}), flush=True)
        del plans, sets, base
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
