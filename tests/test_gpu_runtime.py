"""GPU: the on-the-fly runtime (NEXT-1) yields bit-exact BF16 weights per block, with and without
prefetch on the side stream, and the block forward it feeds matches the resident-weight forward."""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prefetch,ctas", [(False, 0), (True, 0), (True, 3)])
def test_overlap_runner_bit_exact(prefetch, ctas):
    from paper_2504_11651_b200 import df11
    from paper_2504_11651_b200.runtime import BlockWeights, OverlapRunner
    dev = torch.device("cuda", 0)
    shapes = [("a", (1000, 96)), ("b", (257, 96)), ("c", (96, 4099))]
    blocks, refs = [], []
    for layer in range(5):
        ts = [(n, workloads.gaussian_bf16(sh, workloads.seed_for("rt", layer, n))) for n, sh in shapes]
        blocks.append(BlockWeights.from_host([df11.encode(w) for _, w in ts], dev))
        refs.append([torch.from_numpy(w.view(np.int16)).to(dev) for _, w in ts])
    runner = OverlapRunner(blocks, dev, prefetch=prefetch, decode_ctas=ctas)
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


def test_decompress_host_block_pipelined():
    """df11_decompress_host_block: H2D + decode on one stream, D2H overlapped on a second; the BF16
    results in host memory equal the originals bit for bit (P:8 lossless), including an empty tensor."""
    from paper_2504_11651_b200 import df11
    dev = torch.device("cuda", 0)
    # "big" has 2 654 format blocks: two chunks of the pipeline
    shapes = [("q", (512, 1000)), ("empty", (0,)), ("k", (33, 4097)), ("big", (4096, 4096)), ("v", (3000, 700))]
    ws = [workloads.gaussian_bf16(sh, workloads.seed_for("hb", 0, n)) if sh != (0,) else np.zeros(0, np.uint16)
          for n, sh in shapes]
    hs = [df11.encode(w) for w in ws]
    dts = [df11.DeviceTensor(h, dev) for h in hs]
    outs = [torch.empty(max(w.size, 1), dtype=torch.bfloat16, pin_memory=True) for w in ws]
    for rep in range(2):                                  # twice: the staging buffers are reused
        for o in outs:
            o.fill_(0)
        df11.decompress_host_block(hs, dts, outs, copy_stream=torch.cuda.Stream(dev))
        torch.cuda.current_stream(dev).synchronize()
        for w, o in zip(ws, outs):
            got = o[: w.size].view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got, w.reshape(-1))


@pytest.mark.parametrize("max_grid", [1, 3])
def test_capped_grid_many_tiles_and_switches(max_grid):
    """DF11_MAX_GRID caps the persistent grid (read once per process, so a subprocess): one or three
    CTAs then walk every tile of a mixed block — long tile loops per group, stage and sign/mantissa
    refills, decode-table rebuilds at every tensor switch — and the result stays bit-exact."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, workloads\n"
        "from paper_2504_11651_b200 import df11\n"
        "ts = [workloads.gaussian_bf16((n,), seed=n) for n in (300001, 17, 123457, 64000, 5)]\n"
        "ts.append(workloads.student_t_bf16((200003,), seed=2))\n"
        "dts = [df11.to_device(df11.encode(w)) for w in ts]\n"
        "outs = df11.decompress_block(dts, kernel='fast')\n"
        "torch.cuda.synchronize()\n"
        "for w, o in zip(ts, outs):\n"
        "    assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1), w.reshape(-1))\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DF11_MAX_GRID=str(max_grid), PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("max_ctas", [1, 5, 37, 100000])
def test_sm_budget_bit_exact(max_ctas):
    """df11_decompress_block_budget: the same bytes for every SM budget (a budget above the SM count
    means every SM), one launch, on a mixed block (small and large tensors, several CTAs' worth)."""
    from paper_2504_11651_b200 import df11
    dev = torch.device("cuda", 0)
    shapes = [("a", (4096, 1024)), ("b", (128,)), ("c", (3000, 777)), ("d", (1, 5))]
    ws = [workloads.gaussian_bf16(sh, workloads.seed_for("budget", 0, n)) for n, sh in shapes]
    dts = [df11.to_device(df11.encode(w), dev) for w in ws]
    before = df11.launch_count()
    outs = df11.decompress_block(dts, max_ctas=max_ctas)
    torch.cuda.synchronize()
    assert df11.launch_count() - before == 1
    for w, o in zip(ws, outs):
        assert np.array_equal(o.reshape(-1).view(torch.int16).cpu().numpy().view(np.uint16), w.reshape(-1))


def test_module_hook_bit_exact():
    """DF11Hook: a BF16 MLP block whose weights exist only as DF11 in HBM produces bit-identical outputs
    (one decode launch per forward); two blocks share one scratch (decoded weights discarded)."""
    from paper_2504_11651_b200 import df11, runtime
    torch.manual_seed(0)

    def block():
        return torch.nn.Sequential(torch.nn.Linear(1024, 2816, bias=False), torch.nn.SiLU(),
                                   torch.nn.Linear(2816, 1024, bias=False)).to("cuda", torch.bfloat16)
    b1, b2 = block(), block()
    x = torch.randn(8, 1024, device="cuda", dtype=torch.bfloat16)
    ref = b2(b1(x))
    shared = torch.empty(2 * 2816 * 1024 + 4096, dtype=torch.bfloat16, device="cuda")
    h1 = runtime.compress_module(b1, scratch=shared)
    h2 = runtime.compress_module(b2, scratch=shared)
    assert b1[0].weight is None and b2[2].weight is None
    n0 = df11.launch_count()
    out = b2(b1(x))
    torch.cuda.synchronize()
    assert df11.launch_count() - n0 == 2
    assert torch.equal(out, ref)
    assert b1[0].weight is None                           # unbound after the forward
    h1.remove()
    h2.remove()


@pytest.mark.parametrize("dtype", ["bfloat16", "float16"])
def test_compress_blocks_llama_bit_exact(dtype):
    """A randomly initialised (offline, no weights downloaded) Llama-architecture model from
    `transformers` whose decoder blocks, embedding and LM head exist only as DF11 in HBM: one decode
    launch per block / embedding / head per forward into one shared scratch, and the logits are
    bit-identical to the BF16 model's (lossless, P:8)."""
    transformers = pytest.importorskip("transformers")
    from paper_2504_11651_b200 import df11, runtime
    torch.manual_seed(0)
    cfg = transformers.LlamaConfig(vocab_size=1024, hidden_size=256, intermediate_size=704, num_hidden_layers=3,
                                   num_attention_heads=4, num_key_value_heads=2, tie_word_embeddings=False)
    model = transformers.LlamaForCausalLM(cfg).to("cuda", getattr(torch, dtype)).eval()
    ids = torch.randint(0, 1024, (2, 17), device="cuda")
    with torch.no_grad():
        ref = model(ids).logits.clone()
    mods = list(model.model.layers) + [model.model.embed_tokens, model.lm_head]
    hooks = runtime.compress_blocks(mods)
    assert model.model.layers[0].self_attn.q_proj.weight is None
    n0 = df11.launch_count()
    with torch.no_grad():
        out = model(ids).logits
    torch.cuda.synchronize()
    assert df11.launch_count() - n0 == len(mods)
    assert torch.equal(out, ref)
    for h in hooks:
        h.remove()


def test_back_to_back_decodes_into_one_buffer():
    """The product kernel is a programmatic dependent launch (df11.h stream semantics): a decode that
    follows a decode on the same stream may read its own inputs early but must not write before the
    previous decode is complete.  Write-after-write through one output buffer, no host sync in between:
    a large decode (58.7 M elements) followed by a small one into the tail of the same buffer (the
    region the large decode writes last), and two equal-size tensors alternating; the last decode's values must survive every time.
    (A regression check: a build without the wait, -DSP12_PDL_NOWAIT, also passed on B200 - the second
    decode's table build outlasts the first one's CTA-exit spread - so the wait is required by the PTX
    memory model, not caught by timing.)"""
    from paper_2504_11651_b200 import df11
    dev = torch.device("cuda", 0)
    big = workloads.gaussian_bf16((14336, 4096), workloads.seed_for("pdl", 0, "big"))
    small = workloads.gaussian_bf16((1 << 20,), workloads.seed_for("pdl", 0, "small"), sigma=0.05)
    other = workloads.gaussian_bf16((14336, 4096), workloads.seed_for("pdl", 1, "big"), sigma=0.01)
    d_big, d_small, d_other = (df11.to_device(df11.encode(w), dev) for w in (big, small, other))
    buf = torch.empty(big.size, dtype=torch.bfloat16, device=dev)
    ref_small = torch.from_numpy(small.view(np.int16)).to(dev)
    ref_big = torch.from_numpy(big.reshape(-1).view(np.int16)).to(dev)
    ref_other = torch.from_numpy(other.reshape(-1).view(np.int16)).to(dev)
    # the small decodes target the tail of the buffer, which the big decode's last CTA writes last:
    # one tile (4 096 elements, one CTA that starts on the first SM the big decode frees) and 1 M
    tiny = workloads.gaussian_bf16((4096,), workloads.seed_for("pdl", 0, "tiny"), sigma=0.05)
    d_tiny = df11.to_device(df11.encode(tiny), dev)
    ref_tiny = torch.from_numpy(tiny.view(np.int16)).to(dev)
    bad = 0
    for i in range(40):
        df11.decompress(d_big, out=buf)
        if i % 2:
            df11.decompress(d_small, out=buf[-small.size:])
            bad += not torch.equal(buf[-small.size:].view(torch.int16), ref_small)
        else:
            df11.decompress(d_tiny, out=buf[-tiny.size:])
            bad += not torch.equal(buf[-tiny.size:].view(torch.int16), ref_tiny)
    torch.cuda.synchronize()
    assert bad == 0, f"{bad} of 40 back-to-back pairs lost the second decode's values"
    # SM-budgeted decodes (df11_decompress_block_budget): the dependent grid's CTAs land on idle SMs at
    # once and must still wait before writing
    for ctas in (8, 37):
        for i in range(10):
            df11.decompress_block([d_big], outs=[buf], max_ctas=ctas)
            df11.decompress_block([d_tiny], outs=[buf[-tiny.size:]], max_ctas=ctas)
            bad += not torch.equal(buf[-tiny.size:].view(torch.int16), ref_tiny)
    assert bad == 0, f"{bad} budgeted back-to-back pairs lost the second decode's values"
    assert torch.equal(buf[: -small.size].view(torch.int16), ref_big[: -small.size])
    for i in range(21):
        df11.decompress(d_other if i % 2 == 0 else d_big, out=buf)
    torch.cuda.synchronize()
    assert torch.equal(buf.view(torch.int16), ref_other)
    assert df11.lib().df11_last_kernel_mask() & 2, "the product kernel ran"


def test_decodes_captured_in_cuda_graph():
    """Block decodes captured in a CUDA graph (the dependent launches become graph edges) replay
    bit-exactly, including back-to-back decodes through one output buffer."""
    from paper_2504_11651_b200 import df11
    dev = torch.device("cuda", 0)
    ws = [workloads.gaussian_bf16(sh, workloads.seed_for("graph", 0, str(i)))
          for i, sh in enumerate([(4096, 4096), (1024, 4096), (14336, 512), (3, 1000)])]
    dts = [df11.to_device(df11.encode(w), dev) for w in ws]
    refs = [torch.from_numpy(w.reshape(-1).view(np.int16)).to(dev) for w in ws]
    shared = torch.empty(ws[0].size, dtype=torch.bfloat16, device=dev)
    plan = df11.BlockPlan(dts)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):                      # warm-up outside the capture (attributes, LUT copies)
        plan.run(stream=s)
        df11.decompress(dts[1], out=shared[: ws[1].size], stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(stream=s)
        df11.decompress(dts[0], out=shared, stream=s)
        df11.decompress(dts[1], out=shared[: ws[1].size], stream=s)
    for _ in range(3):
        for o in plan.outputs():
            o.view(torch.int16).zero_()
        shared.view(torch.int16).fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        for o, r in zip(plan.outputs(), refs):
            assert torch.equal(o.reshape(-1).view(torch.int16), r)
        assert torch.equal(shared[: ws[1].size].view(torch.int16), refs[1])
        assert torch.equal(shared[ws[1].size:].view(torch.int16), refs[0][ws[1].size:])
