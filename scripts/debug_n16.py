"""Debug helper (not a test): first mismatches of the n = 16 product kernel on a Gaussian tensor."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import workloads
from paper_2504_11651_b200 import df11
for n in (4096 * 3, 1 << 20):
    w = workloads.gaussian_bf16((n,), seed=1)
    h = df11.encode(w, T=128, n=16)
    dt = df11.to_device(h)
    out = df11.decompress(dt, kernel="fast")
    torch.cuda.synchronize()
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    bad = np.nonzero(got != w)[0]
    bop = h.block_output_pos
    print(n, "B", h.B, "mismatches", bad.size, "max code", h.max_code_len)
    if bad.size:
        i = bad[0]
        b = int(np.searchsorted(bop, i, side="right") - 1)
        print(" first", i, "block", b, "bop", bop[b], bop[b + 1], "got/want", hex(got[i]), hex(w[i]))
        print(" got ", [hex(x) for x in got[i - 3:i + 5]])
        print(" want", [hex(x) for x in w[i - 3:i + 5]])
        print(" exp got", (got[i - 3:i + 5] >> 7) & 255, "want", (w[i - 3:i + 5] >> 7) & 255)
        blocks = np.unique(np.searchsorted(bop, bad, side="right") - 1)
        print(" bad blocks", blocks[:20], blocks.size)
