"""GPU: the on-the-fly runtime (NEXT-1) yields bit-exact BF16 weights per block, with and without
prefetch on the side stream, and the block forward it feeds matches the resident-weight forward."""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prefetch", [False, True])
def test_overlap_runner_bit_exact(prefetch):
    from paper_2504_11651_b200 import df11
    from paper_2504_11651_b200.runtime import BlockWeights, OverlapRunner
    dev = torch.device("cuda", 0)
    shapes = [("a", (1000, 96)), ("b", (257, 96)), ("c", (96, 4099))]
    blocks, refs = [], []
    for layer in range(5):
        ts = [(n, workloads.gaussian_bf16(sh, workloads.seed_for("rt", layer, n))) for n, sh in shapes]
        blocks.append(BlockWeights.from_host([df11.encode(w) for _, w in ts], dev))
        refs.append([torch.from_numpy(w.view(np.int16)).to(dev) for _, w in ts])
    runner = OverlapRunner(blocks, dev, prefetch=prefetch)
    x = torch.randn(7, 96, device=dev, dtype=torch.bfloat16)
    y_ref = x.clone()
    y = x.clone()
    seen = []
    for i, W in runner.iterate():
        seen.append(i)
        for got, ref in zip(W, refs[i]):
            assert torch.equal(got.view(torch.int16), ref)
        y = y @ W[0].T @ W[0] / 100                       # uses the weights on the main stream
        y_ref = y_ref @ refs[i][0].view(torch.bfloat16).T @ refs[i][0].view(torch.bfloat16) / 100
    torch.cuda.synchronize()
    assert seen == list(range(5))
    assert torch.equal(y, y_ref)
