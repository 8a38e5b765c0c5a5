"""Small decode cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2504_11651_b200 import df11  # noqa: E402

cases = [workloads.gaussian_bf16((150001,), seed=1), workloads.constant(40000),
         workloads.from_exponent_histogram({e: max(1, int(40000 * 0.72 ** i)) for i, e in enumerate(range(60, 200))}, 3),
         workloads.all_bf16_patterns(),
         workloads.from_exponent_histogram({110 + i: 20000 for i in range(4)}, seed=12),      # 2-bit codes
         workloads.from_exponent_histogram({e: max(1, int(200000 * 0.829 ** i)) for i, e in enumerate(range(90, 130))}, 11)]
# run with DF11_MAX_GRID=2: every group walks several tiles (stage/sign-mantissa refills, tensor switches)
kernels = sys.argv[1:] or ["fast", "alg1"]
for kernel in kernels:
    dts = [df11.to_device(df11.encode(w)) for w in cases]
    outs = df11.decompress_block(dts, kernel=kernel)
    torch.cuda.synchronize()
    for w, o in zip(cases, outs):
        assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), w.reshape(-1))
print("sanitize cases ok", kernels)
