"""GPU parity: the CUDA path (through the C ABI) vs the oracle and the original tensor, bit for bit.

Decode of DF11 is lossless: the plain definition of the result is the original tensor (P:8, P:36,
P:264).  Every case checks GPU == original, and GPU == oracle D1 (sequential) on the same arrays.
Inputs come from workloads.py; expected values from the generator or from oracle/ only.
"""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KERNELS = ["alg1", "fast"]


@pytest.fixture(scope="module")
def df11():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2504_11651_b200 import df11 as m
    m.lib()
    return m


def _fast_ok(df11, meta):
    return (meta["T"], meta["n"]) in ((256, 8), (128, 16))


def _gpu_decode_arrays(df11, meta, arrays, kernel, shape=None):
    dt = df11.DeviceTensor.from_arrays(meta, arrays, shape=shape)
    out = df11.decompress(dt, kernel=kernel)
    torch.cuda.synchronize()
    return out.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1)


def _check_oracle_format(df11, oracle_mod, w, kernel, **kw):
    """Oracle-encoded arrays -> GPU decode == original == oracle D1."""
    fmt = oracle_mod.encode(w, **kw)
    meta = {k: fmt[k] for k in ("num_elements", "T", "n", "B", "k", "lut_entry_bytes", "encoded_bits",
                                "max_code_len")}
    if kernel == "fast" and not _fast_ok(df11, meta):
        with pytest.raises(df11.Df11Error):
            _gpu_decode_arrays(df11, meta, fmt, kernel)
        return
    got = _gpu_decode_arrays(df11, meta, fmt, kernel)
    assert np.array_equal(got[: w.size], w.reshape(-1))
    if w.size <= 5_000_000:
        assert np.array_equal(got[: w.size], oracle_mod.decode_sequential(fmt))


CASES = ["gauss_1m", "gauss_ragged", "constant_1bit", "two_symbol", "all_patterns_wide", "overflow_wide",
         "fibonacci_32bit", "one_element", "tiny_17", "sigma_large", "random_bits", "escape_heavy", "escape_deep",
         "uniform8_short_codes", "one_bit_with_tail", "maxlen_12", "maxlen_13", "four_symbol_2bit", "student_t5",
         "sigma_loguniform"]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("case", CASES)
def test_parity_cases(df11, oracle_mod, kernel, case):
    _check_oracle_format(df11, oracle_mod, _case_weights(case), kernel)


@pytest.mark.parametrize("case", CASES)
def test_parity_cases_n16_fast(df11, oracle_mod, case):
    """NEXT-4: the product kernel on the format T = 128, n = 16 (half the gap bits), every
    parity case, oracle-encoded arrays: GPU == original == oracle D1."""
    _check_oracle_format(df11, oracle_mod, _case_weights(case), "fast", T=128, n=16)


def _case_weights(case):
    if case == "gauss_1m":
        w = workloads.gaussian_bf16((1 << 20,), seed=1)
    elif case == "gauss_ragged":
        w = workloads.gaussian_bf16((3 * 16384 * 3 + 12345,), seed=2)      # several tiles + ragged tail
    elif case == "constant_1bit":
        w = workloads.constant(16384 * 5 + 3)                              # 8nT elements per block
    elif case == "two_symbol":
        w = workloads.from_exponent_histogram({100: 70000, 101: 3}, seed=1)
    elif case == "all_patterns_wide":
        w = workloads.all_bf16_patterns()
    elif case == "overflow_wide":
        counts = {120: 1 << 18}
        counts.update({e: 1 + e % 3 for e in range(1, 120)})
        w = workloads.from_exponent_histogram(counts, seed=5)
    elif case == "fibonacci_32bit":
        w = workloads.from_exponent_histogram(workloads.fibonacci_histogram(34, 80), seed=1)
    elif case == "one_element":
        w = np.array([0xC040], np.uint16)
    elif case == "tiny_17":
        w = workloads.gaussian_bf16((17,), seed=3)
    elif case == "sigma_large":
        w = workloads.gaussian_bf16((777777,), seed=4, sigma=3.0)
    elif case == "escape_heavy":
        # 16 frequent exponents (~4-bit codes) + 200 rare ones (~12-bit codes): many codes are
        # longer than the 9-bit root (~9 %: (escape rows, second-level tables, bit-buffer refills)
        counts = {100 + i: 24000 for i in range(16)}
        counts.update({i: 200 for i in range(1, 100)})
        counts.update({116 + i: 200 for i in range(101)})
        w = workloads.from_exponent_histogram(counts, seed=7)
    elif case == "uniform8_short_codes":
        # 8 equally likely exponents: every code is 3 bits (no code longer than the 9-bit root, so
        # the kernel cannot use one-bit chain-end sentinels and walks back instead)
        w = workloads.from_exponent_histogram({100 + i: 40000 for i in range(8)}, seed=9)
    elif case == "one_bit_with_tail":
        # a 1-bit codeword (p > 1/2) plus a geometric tail of long codes: count + direct path
        counts = {127: 600000}
        counts.update({e: max(1, int(50000 * 0.6 ** i)) for i, e in enumerate(range(100, 127))})
        w = workloads.from_exponent_histogram(counts, seed=10)
    elif case == "maxlen_12" or case == "maxlen_13":
        # geometric exponent distribution whose longest code is exactly 12 (every code fits the
        # 12-bit decode table: chain ends are found by walking back) or 13 bits (the all-ones row
        # is an escape: exact chain ends through one-bit sentinels)
        L = 12 if case == "maxlen_12" else 13
        from oracle import huffman
        for r in np.linspace(0.76, 0.90, 300):
            counts = {90 + i: max(1, int(200000 * r ** i)) for i in range(40)}
            h = np.zeros(256, np.int64)
            for e, c in counts.items():
                h[e] = c
            if max(huffman.code_lengths(h)) == L:
                break
        else:
            pytest.fail("no histogram with the requested maximum code length")
        w = workloads.from_exponent_histogram(counts, seed=11)
    elif case == "four_symbol_2bit":
        # four equally likely exponents: 2-bit codes, 8192 outputs per format block, more than the
        # kernel stages in SMEM per tile (its PackedSignMantissa is read from global memory instead)
        w = workloads.from_exponent_histogram({110 + i: 60000 for i in range(4)}, seed=12)
    elif case == "student_t5":
        # heavy-tailed realism variant: more exponents, longer codes, more escapes
        w = workloads.student_t_bf16((3 * 16384 * 5 + 999,), seed=13)
    elif case == "sigma_loguniform":
        # per-tensor sigma drawn log-uniform in [0.01, 0.04]; here the extremes
        w = np.concatenate([workloads.gaussian_bf16((200003,), seed=14, sigma=0.01),
                            workloads.gaussian_bf16((200003,), seed=15, sigma=0.04)])
    elif case == "escape_deep":
        # geometric tail: codes up to ~26 bits, some beyond the second level (walk path)
        counts = {e: max(1, int(400000 * 0.72 ** i)) for i, e in enumerate(range(60, 200))}
        w = workloads.from_exponent_histogram(counts, seed=8)
    else:
        w = np.random.default_rng(5).integers(0, 1 << 16, size=400001, dtype=np.uint32).astype(np.uint16)
    return w


@pytest.mark.parametrize("T,n", [(32, 4), (64, 8), (128, 16), (256, 8), (512, 8), (1024, 8), (96, 5), (1024, 32)])
def test_alg1_geometry_grid(df11, oracle_mod, T, n):
    w = workloads.gaussian_bf16((300001,), seed=T * 100 + n)
    _check_oracle_format(df11, oracle_mod, w, "alg1", T=T, n=n)


def test_empty_tensor_is_noop(df11):
    h = df11.encode(np.zeros(0, np.uint16))
    dt = df11.to_device(h)
    df11.decompress(dt)
    torch.cuda.synchronize()
    assert h.B == 0


@pytest.mark.parametrize("kernel", KERNELS)
def test_block_batch_flux_single(df11, oracle_mod, kernel):
    """One launch for a mixed FLUX.1 single block (3 matrices + biases + 128-element norm scales):
    tiny tensors, ragged sizes, different codebooks per tensor."""
    ts = workloads.config_tensors("flux_single_block")
    hs = [df11.encode(w) for _, w in ts]
    dts = [df11.to_device(h) for h in hs]
    before = df11.launch_count()
    outs = df11.decompress_block(dts, kernel=kernel)
    torch.cuda.synchronize()
    assert df11.launch_count() - before == 1
    for (name, w), o in zip(ts, outs):
        got = o.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, w), name


def test_outputs_into_shared_scratch_with_unaligned_views(df11):
    """Per-tensor outputs as views into one reused scratch buffer at odd element offsets."""
    ts = [workloads.gaussian_bf16((n,), seed=n) for n in (5000, 777, 123457, 16)]
    dts = [df11.to_device(df11.encode(w)) for w in ts]
    scratch = torch.zeros(sum(w.size for w in ts) + 8, dtype=torch.bfloat16, device="cuda")
    offs, o = [], 3
    for w in ts:
        offs.append(o)
        o += w.size
    outs = [scratch[a:a + w.size] for a, w in zip(offs, ts)]
    df11.decompress_block(dts, outs=outs)
    torch.cuda.synchronize()
    got = scratch.view(torch.int16).cpu().numpy().view(np.uint16)
    for a, w in zip(offs, ts):
        assert np.array_equal(got[a:a + w.size], w)
    assert not got[:3].any()


def test_invalid_descriptor_names_index(df11):
    dts = [df11.to_device(df11.encode(workloads.gaussian_bf16((1000,), seed=i))) for i in range(3)]
    plan = df11.BlockPlan(dts)
    plan.arr[2].T = 33
    with pytest.raises(df11.Df11Error) as e:
        plan.run()
    assert "descriptor 2" in str(e.value)


def test_corrupt_metadata_never_faults(df11):
    """Malformed metadata may give wrong output but never an out-of-bounds access (df11.h)."""
    w = workloads.gaussian_bf16((200000,), seed=9)
    h = df11.encode(w)
    a = h.arrays()
    rng = np.random.default_rng(0)
    meta = dict(num_elements=h.num_elements, T=h.T, n=h.n, B=h.B, k=h.k, lut_entry_bytes=1,
                encoded_bits=h.encoded_bits, max_code_len=h.max_code_len)
    for trial in range(6):
        b = {k: np.array(v, copy=True) for k, v in a.items()}
        if trial == 0:
            b["block_output_pos"] = rng.integers(0, 1 << 32, size=b["block_output_pos"].size, dtype=np.uint64).astype(np.uint32)
        elif trial == 1:
            b["luts"] = rng.integers(0, 256, size=b["luts"].size, dtype=np.uint8)
        elif trial == 2:
            b["code_lengths"] = rng.integers(0, 256, size=256, dtype=np.uint8)
        elif trial == 3:
            b["gaps"] = rng.integers(0, 256, size=b["gaps"].size, dtype=np.uint8)
        elif trial == 4:
            b["encoded_exponent"] = rng.integers(0, 256, size=b["encoded_exponent"].size, dtype=np.uint8)
        else:
            b["luts"][:] = 240
        for kernel in KERNELS:
            dt = df11.DeviceTensor.from_arrays(meta, b)
            df11.decompress(dt, kernel=kernel)
            torch.cuda.synchronize()   # a fault would raise here


@pytest.mark.parametrize("kernel", KERNELS)
def test_full_size_matrix4096(df11, oracle_mod, kernel):
    """configs[0]: 4096x4096 N(0,0.02): oracle-encoded arrays, GPU == original == oracle D1."""
    w = workloads.gaussian_bf16((4096, 4096), seed=workloads.seed_for("matrix4096", 0, "w"))
    _check_oracle_format(df11, oracle_mod, w, kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_full_size_llama8b_block(df11, oracle_mod, kernel):
    """configs[1] at full size in the launch configuration bench.py times (one df11_decompress_block
    over the 7 tensors): GPU == original for every element; library arrays == oracle arrays for the
    largest tensor; sampled format blocks == oracle D2 (Alg. 1 emulator)."""
    ts = workloads.config_tensors("llama8b_block")
    hs = [df11.encode(w) for _, w in ts]
    dts = [df11.to_device(h) for h in hs]
    outs = df11.decompress_block(dts, kernel=kernel)
    torch.cuda.synchronize()
    for (name, w), o, h in zip(ts, outs, hs):
        got = o.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, w), name
        fmt_like = dict(h.arrays(), num_elements=h.num_elements, T=h.T, n=h.n, B=h.B, k=h.k,
                        lut_entry_bytes=h.lut_entry_bytes)
        blocks = [0, 1, h.B // 2, h.B - 1]
        for b, (lo, vals) in oracle_mod.decode_alg1_blocks(fmt_like, blocks).items():
            assert np.array_equal(got.reshape(-1)[lo:lo + vals.size], vals), (name, b)
    # oracle encoder on the down projection (58.7M elements): byte-identical, and GPU-decodable
    name, w = ts[-1]
    fmt = oracle_mod.encode(w)
    a = hs[-1].arrays()
    for key in ("code_lengths", "luts", "encoded_exponent", "packed_sign_mantissa", "gaps", "block_output_pos"):
        assert np.array_equal(a[key], fmt[key]), key


def test_unaligned_sign_mantissa_buffer(df11):
    """PackedSignMantissa at an odd device address (a view into a larger buffer): the fast kernel
    needs 16-byte aligned streams (TMA bulk copies), so `auto` routes the tensor to the Algorithm 1
    kernel and an explicit `fast` request is refused; the auto result is still the original tensor bit
    for bit (P:8)."""
    w = workloads.gaussian_bf16((700001,), seed=21)
    dt = df11.to_device(df11.encode(w))
    psm = dt.packed_sign_mantissa
    big = torch.zeros(psm.numel() + 16, dtype=torch.uint8, device=psm.device)
    big[1:1 + psm.numel()].copy_(psm)
    dt.packed_sign_mantissa = big[1:1 + psm.numel()]                  # data_ptr() % 16 == 1
    assert dt.packed_sign_mantissa.data_ptr() % 16 == 1
    with pytest.raises(df11.Df11Error):
        df11.decompress(dt, kernel="fast")
    out = df11.decompress(dt, kernel="auto")
    assert df11.last_kernels() == {"alg1"}
    torch.cuda.synchronize()
    got = out.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1)
    assert np.array_equal(got, w.reshape(-1))


def test_auto_splits_a_mixed_batch(df11):
    """A block where one tensor cannot take the product kernel (unaligned PackedSignMantissa view, or
    other format parameters): `auto` sends only that tensor to the Algorithm 1 kernel and the rest of
    the block to ONE product-kernel launch; the Alg. 1 kernel takes one launch per distinct T (3
    launches in all here); every output is the original."""
    ws = [workloads.gaussian_bf16((n,), seed=30 + i) for i, n in enumerate((300001, 65536, 123457))]
    hs = [df11.encode(ws[0]), df11.encode(ws[1], T=64, n=8), df11.encode(ws[2])]
    dts = [df11.to_device(h) for h in hs]
    psm = dts[2].packed_sign_mantissa
    big = torch.zeros(psm.numel() + 16, dtype=torch.uint8, device=psm.device)
    big[3:3 + psm.numel()].copy_(psm)
    dts[2].packed_sign_mantissa = big[3:3 + psm.numel()]
    before = df11.launch_count()
    outs = df11.decompress_block(dts)
    assert df11.launch_count() - before == 3
    assert df11.last_kernels() == {"alg1", "fast"}
    torch.cuda.synchronize()
    for w, o in zip(ws, outs):
        assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), w)
    df11.decompress_block([dts[0]])
    assert df11.last_kernels() == {"fast"}


def test_full_size_llama8b_block_n16(df11, oracle_mod):
    """NEXT-4: the Llama-3.1-8B block encoded with T = 128, n = 16 decodes in ONE product-kernel
    launch, every element bit-exact, oracle D2 on sampled blocks; a mixed n = 8 / n = 16 batch takes
    one launch per chunk size."""
    ts = workloads.config_tensors("llama8b_block")
    hs = [df11.encode(w, T=128, n=16) for _, w in ts]
    dts = [df11.to_device(h) for h in hs]
    before = df11.launch_count()
    outs = df11.decompress_block(dts)
    assert df11.launch_count() - before == 1 and df11.last_kernels() == {"fast"}
    torch.cuda.synchronize()
    for (name, w), o, h in zip(ts, outs, hs):
        got = o.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, w), name
        fmt_like = dict(h.arrays(), num_elements=h.num_elements, T=h.T, n=h.n, B=h.B, k=h.k,
                        lut_entry_bytes=h.lut_entry_bytes)
        for b, (lo, vals) in oracle_mod.decode_alg1_blocks(fmt_like, [0, 1, h.B // 2, h.B - 1]).items():
            assert np.array_equal(got.reshape(-1)[lo:lo + vals.size], vals), (name, b)
    mixed = [df11.to_device(df11.encode(ts[1][1])), dts[2]]
    before = df11.launch_count()
    outs = df11.decompress_block(mixed)
    assert df11.launch_count() - before == 2
    torch.cuda.synchronize()
    for (name, w), o in zip([ts[1], ts[2]], outs):
        assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), w), name
