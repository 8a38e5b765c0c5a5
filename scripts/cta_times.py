"""Per-CTA timeline of one product-kernel launch (globaltimer instrumentation, -DSP12_TIMES build):
start skew, table build, group end spread (the tail) and CTA exit spread.

    DF11_LIB=paper_2504_11651_b200/lib/variants/times.so python scripts/cta_times.py [config]
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
ts = workloads.config_tensors(cfg)
if os.environ.get("REVERSE"):                   # does a slow CTA range follow the tensor or the CTA index?
    ts = ts[::-1]
dts = [df11.to_device(df11.encode(w)) for _, w in ts]
plan = df11.BlockPlan(dts, None)
for _ in range(5):
    plan.run(kernel="fast")
torch.cuda.synchronize()
buf = np.zeros((256, 12), np.uint64)
assert df11.lib().df11_debug_sp12_times(buf.ctypes.data_as(ctypes.c_void_p)) == 0
used = buf[:, 0] > 0
b = buf[used].astype(np.float64)
t0 = b[:, 0].min()
ent, built, ext, grp = (b[:, 0] - t0) / 1e3, (b[:, 1] - t0) / 1e3, (b[:, 2] - t0) / 1e3, (b[:, 3:11] - t0) / 1e3
print(f"{cfg}: CTAs {used.sum()}, kernel span {ext.max():.1f} us")
print(f"  entry skew: max {ent.max():.2f} us; first table built at {np.median(built):.2f} us (median), max {built.max():.2f}")
print(f"  CTA exit: min {ext.min():.1f} median {np.median(ext):.1f} max {ext.max():.1f} us")
print(f"  group end within a CTA (max - min): median {np.median(grp.max(1) - grp.min(1)):.2f} us, max {(grp.max(1) - grp.min(1)).max():.2f}")
print(f"  idle SM-time after a CTA's exit: {np.mean(ext.max() - ext):.2f} us mean per SM ({100 * np.mean(ext.max() - ext) / ext.max():.1f} %)")
print(f"  idle group-time inside CTAs: {np.mean(grp.max(1)[:, None] - grp):.2f} us mean per group")
if len(sys.argv) > 2:
    # per-CTA exit time vs the CTA's tile range and tensors (static plan from df11_plan_cta_ranges)
    order = np.argsort(ext)
    print("  slowest CTAs:", [(int(i), round(float(ext[i]), 1)) for i in order[-8:]])
    print("  fastest CTAs:", [(int(i), round(float(ext[i]), 1)) for i in order[:8]])
    print("  exit time by CTA index (16 per row):")
    for r in range(0, len(ext), 16):
        print("   ", " ".join(f"{v:6.1f}" for v in ext[r:r + 16]))
if len(sys.argv) > 2:
    smid = buf[used, 11].astype(int)
    rel = (ext - ext.mean()) / ext.mean() * 100
    print("  exit time vs SM id (relative %, sorted by smid):")
    o = np.argsort(smid)
    for r in range(0, len(o), 16):
        print("   ", " ".join(f"{smid[i]:3d}:{rel[i]:+4.1f}" for i in o[r:r + 16]))
