#!/usr/bin/env python
"""NEXT-3: compression time per transformer block (the paper's Table `time`: 191 / 547 /
2133 s per block for Llama 3.1 8B / 70B / 405B on one CPU thread).

For each config: the GPU encoder (histogram kernel -> host codebook -> pack + gaps kernels) timed end to
end per block (CUDA events around the whole call sequence, including the histogram read-back), the
pack kernel alone, and the multithreaded host encoder (df11_encode) on the same tensors.  One JSON
line per config.

    python scripts/bench_encode.py [--configs llama8b_block,llama70b_block] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="llama8b_block,llama70b_block,llama405b_block")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--host", action="store_true", help="also time the host encoder (slow for 405B)")
    ap.add_argument("--vf", default="bf16", choices=list(workloads.VALUE_FORMATS),
                    help="value format of the weights (NEXT-4): bf16 / fp16 / fp8_e4m3 / fp8_e5m2")
    args = ap.parse_args()
    import torch

    from paper_2504_11651_b200 import df11
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    for cfg in args.configs.split(","):
        shapes = workloads.CONFIGS[cfg]
        vf = args.vf
        if vf == "bf16":
            xs = [torch.from_numpy(workloads.gaussian_bf16_torch(sh, workloads.seed_for(cfg, 0, name), dev)
                                   .view(np.int16)).to(dev) for name, sh in shapes]
        else:
            xs = []
            for name, sh in shapes:
                w = workloads.gaussian_values(sh, workloads.seed_for(cfg, 0, name), vf)
                xs.append(torch.from_numpy(w.view(np.int16) if w.dtype == np.uint16 else w).to(dev))
        wb = xs[0].element_size()
        wv = torch.int16 if wb == 2 else torch.uint8
        numel = sum(x.numel() for x in xs)
        # correctness: round trip
        dts = [df11.encode_device(x, vf=vf) for x in xs]
        outs = df11.decompress_block(dts)
        torch.cuda.synchronize()
        for x, o in zip(xs, outs):
            assert torch.equal(o.reshape(-1).view(wv), x.reshape(-1))
        comp = sum(d.compressed_bytes for d in dts)

        def full():   # histograms of the whole block first (one read-back), then the plans and packing
            return df11.encode_device_group(xs, shared_codebook=False, vf=vf)

        for _ in range(2):
            full()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.reps):
            full()
        e.record()
        torch.cuda.synchronize()
        ms_full = s.elapsed_time(e) / args.reps
        wall_full = (time.perf_counter() - t0) * 1e3 / args.reps
        # pack stage alone (plans prebuilt)
        plans = []
        for x in xs:
            h = df11.histogram_device(x, vf=vf).cpu().numpy().view(np.uint64)
            plans.append(df11.EncodePlan(h, h, vf=vf))
        for _ in range(2):
            [df11.encode_device_with_plan(x, p) for x, p in zip(xs, plans)]
        torch.cuda.synchronize()
        s.record()
        for _ in range(args.reps):
            [df11.encode_device_with_plan(x, p) for x, p in zip(xs, plans)]
        e.record()
        torch.cuda.synchronize()
        ms_pack = s.elapsed_time(e) / args.reps
        hbuf = torch.zeros(256, dtype=torch.int64, device=dev)
        for _ in range(2):
            [df11.histogram_device(x, out=hbuf, vf=vf) for x in xs]
        s.record()
        for _ in range(args.reps):
            [df11.histogram_device(x, out=hbuf, vf=vf) for x in xs]
        e.record()
        torch.cuda.synchronize()
        ms_hist = s.elapsed_time(e) / args.reps
        line = {"config": cfg, "value_format": vf, "elements": numel, "input_bytes": wb * numel, "df11_bytes": comp,
                "ratio": comp / (wb * numel), "gpu_encode_ms_per_block": ms_full, "gpu_encode_wall_ms": wall_full,
                "gpu_pack_ms_per_block": ms_pack, "gpu_hist_ms_per_block": ms_hist,
                "hist_gbs": wb * numel / ms_hist / 1e6, "gpu_encode_gelem_s": numel / ms_full / 1e6,
                "paper_single_thread_s_per_block": {"llama8b_block": 191, "llama70b_block": 547,
                                                    "llama405b_block": 2133}.get(cfg)}
        if args.host:
            ws = [x.cpu().numpy().view(workloads.word_dtype(vf)) for x in xs]
            t0 = time.perf_counter()
            for w in ws:
                df11.encode(w, vf=vf)
            line["host_encode_ms_per_block"] = (time.perf_counter() - t0) * 1e3
            line["host_threads"] = os.cpu_count()
        print(json.dumps(line), flush=True)
        del xs, dts, outs, plans
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
