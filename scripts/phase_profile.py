"""Per-phase cycle breakdown of the sp12 kernel (clock64 instrumentation, -DSP12_PROF variant build).

    DF11_LIB=paper_2504_11651_b200/lib/variants/prof.so python scripts/phase_profile.py [config]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2504_11651_b200 import df11  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama8b_block"
if cfg.startswith("n="):                                   # one Gaussian tensor of n elements
    tensors = [("w", workloads.gaussian_bf16((int(cfg[2:]),), 1))]
else:
    tensors = workloads.config_tensors(cfg)
dts = [df11.to_device(df11.encode(w)) for _, w in tensors]
plan = df11.BlockPlan(dts, None)
for _ in range(3):
    plan.run(kernel="fast")
torch.cuda.synchronize()
buf = np.zeros((148 * 32, 8), np.uint64)
rc = df11.lib().df11_debug_sp12_prof(buf.ctypes.data_as(ctypes.c_void_p))
assert rc == 0, rc
names = ["merge+tail (prev tile)", "stage wait", "decode", "scan", "barrier", "range + slot loads",
         "compaction stores+heads", "merge setup + sm wait"]
tot = buf.astype(np.float64).sum(1)
act = tot > 0
print(f"{cfg}: warps {act.sum()}, mean cycles per warp {tot[act].mean():.0f}, max {tot.max():.0f}")
if len(sys.argv) > 2:
    for i in range(8):
        print("   max", names[i], int(buf[act, i].max()))
for i, n in enumerate(names):
    v = buf[act, i].astype(np.float64)
    print(f"  {n:24s} {100 * v.sum() / tot[act].sum():5.1f} %   mean {v.mean():9.0f}")
