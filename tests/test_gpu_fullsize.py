"""Full-size GPU parity for the model configs of BASELINE.json (SURVEY.md 8(a) shapes):
one df11_decompress_block launch per transformer block (the launch configuration bench.py times),
GPU == original for EVERY element (the plain definition of lossless decode, P:8), and oracle D2
(Alg. 1 emulator, oracle/) on sampled format blocks of every tensor, including the last ones.

Inputs are generated on the GPU with a seeded torch generator (workloads.gaussian_bf16_torch; the
multi-GB shapes would take minutes with numpy) and encoded by the host encoder; expected values are
the generator's tensors and oracle D2's outputs only.
"""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def df11():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2504_11651_b200 import df11 as m
    m.lib()
    return m


def _sampled_blocks(B):
    return sorted(b for b in {0, 1, B // 3, B // 2, (2 * B) // 3, B - 2, B - 1} if 0 <= b < B)


@pytest.mark.parametrize("config", ["flux_double_block", "llama70b_block", "llama405b_block", "llama405b_embed"])
def test_full_size_config(df11, oracle_mod, config):
    """FLUX.1 double block (24 tensors incl. biases and 128-element norm scales), a Llama-3.3-70B
    block, a Llama-3.1-405B block (3.19 G elements) and the 405B embedding (2.10 G elements: output
    positions past 2^30, uint32 position arithmetic near its range)."""
    dev = torch.device("cuda")
    names, ws, hs, dts = [], [], [], []
    for name, shape in workloads.CONFIGS[config]:
        w = workloads.gaussian_bf16_torch(shape, workloads.seed_for(config, 0, name), dev)
        h = df11.encode(w)
        names.append(name)
        hs.append(h)
        dts.append(df11.to_device(h))
        ws.append(w)
    before = df11.launch_count()
    outs = df11.decompress_block(dts, kernel="auto")
    torch.cuda.synchronize()
    assert df11.launch_count() - before == 1, "one launch for the whole block (P:157)"
    assert df11.last_kernels() == {"fast"}
    for name, w, o, h in zip(names, ws, outs, hs):
        ref = torch.from_numpy(w.reshape(-1).view(np.int16)).to(dev)
        got = o.reshape(-1).view(torch.int16)
        assert got.numel() == ref.numel()
        assert torch.equal(got, ref), name           # every element bit-exact
        fmt_like = dict(h.arrays(), num_elements=h.num_elements, T=h.T, n=h.n, B=h.B, k=h.k,
                        lut_entry_bytes=h.lut_entry_bytes)
        for b, (lo, vals) in oracle_mod.decode_alg1_blocks(fmt_like, _sampled_blocks(h.B)).items():
            assert np.array_equal(got[lo:lo + vals.size].cpu().numpy().view(np.uint16), vals), (name, b)
        if config == "llama405b_embed":
            assert int(h.block_output_pos[-2]) > (1 << 30)   # the sampled last blocks sit past 2^30
        del ref, got
    del outs, dts
    torch.cuda.empty_cache()
