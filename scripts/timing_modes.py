"""Timing-method check: K block decodes timed (a) eager with per-launch events, (b) eager with only
start/end events, (c) as one CUDA graph replay.  Prints us per step for each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2504_11651_b200 import df11  # noqa: E402

K = 200
for cfg in sys.argv[1:] or ["llama8b_block", "matrix4096"]:
    ts = workloads.config_tensors(cfg)
    hs = [df11.encode(w) for _, w in ts]
    base = [df11.to_device(h) for h in hs]
    algo = sum(d.compressed_bytes for d in base) + 2 * sum(h.num_elements for h in hs)
    copies = max(1, min(32, -(-4 * (126 << 20) // algo)))
    plans = [df11.BlockPlan(base)] + [df11.BlockPlan([df11.clone_device_tensor(d) for d in base]) for _ in range(copies - 1)]
    s = torch.cuda.Stream()
    res = {"config": cfg, "copies": copies}
    with torch.cuda.stream(s):
        for i in range(10):
            plans[i % copies].run(s)
        torch.cuda.synchronize()
        for mode in ("eager_events", "eager_plain", "graph", "eager_events", "eager_plain", "graph"):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if mode == "graph":
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for i in range(K):
                        plans[i % copies].run(s)
                g.replay()
                torch.cuda.synchronize()
                a.record(s)
                g.replay()
                b.record(s)
            else:
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
                a.record(s)
                for i in range(K):
                    if mode == "eager_events":
                        ev[i][0].record(s)
                    plans[i % copies].run(s)
                    if mode == "eager_events":
                        ev[i][1].record(s)
                b.record(s)
            torch.cuda.synchronize()
            res.setdefault(mode, []).append(round(a.elapsed_time(b) * 1e3 / K, 2))
    print(json.dumps(res), flush=True)
