"""GPU: the device encoder (NEXT-3, df11_histogram_device / df11_encode_plan_create / df11_encode_device)
writes exactly the bytes of the oracle encoder (oracle/oracle.py E1..E8), padding included.

Expected values come from oracle/ only; inputs from workloads.py.
"""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ARRAYS = ("encoded_exponent", "packed_sign_mantissa", "gaps", "luts", "code_lengths", "block_output_pos")


@pytest.fixture(scope="module")
def df11():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2504_11651_b200 import df11 as m
    m.lib()
    return m


def _dev(w):
    return torch.from_numpy(np.ascontiguousarray(w).view(np.int16)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint8)


def _compare(dt, fmt):
    torch.cuda.synchronize()
    for key in ("T", "n", "B", "k", "lut_entry_bytes", "encoded_bits", "max_code_len"):
        assert dt.meta[key] == fmt[key], key
    assert dt.num_elements == fmt["num_elements"]
    for key in ARRAYS:
        want = np.ascontiguousarray(fmt[key]).view(np.uint8)
        got = _host(getattr(dt, key))
        if key == "luts" and want.size == 0:
            continue
        assert got.size >= want.size, key
        assert np.array_equal(got[: want.size], want), key


def _case(name):
    if name == "gauss_1m":
        return workloads.gaussian_bf16((1 << 20,), seed=21)
    if name == "gauss_ragged":
        return workloads.gaussian_bf16((3 * 16384 * 3 + 12345,), seed=22)
    if name == "constant_1bit":
        return workloads.constant(16384 * 5 + 3)
    if name == "two_symbol":
        return workloads.from_exponent_histogram({100: 70000, 101: 3}, seed=1)
    if name == "all_patterns":
        return workloads.all_bf16_patterns()
    if name == "fibonacci_32bit":
        return workloads.from_exponent_histogram(workloads.fibonacci_histogram(34, 80), seed=1)
    if name == "one_element":
        return np.array([0xC040], np.uint16)
    if name == "tiny_17":
        return workloads.gaussian_bf16((17,), seed=3)
    if name == "escape_deep":
        counts = {e: max(1, int(400000 * 0.72 ** i)) for i, e in enumerate(range(60, 200))}
        return workloads.from_exponent_histogram(counts, seed=8)
    return np.random.default_rng(5).integers(0, 1 << 16, size=400001, dtype=np.uint32).astype(np.uint16)


@pytest.mark.parametrize("case", ["gauss_1m", "gauss_ragged", "constant_1bit", "two_symbol", "all_patterns",
                                  "fibonacci_32bit", "one_element", "tiny_17", "escape_deep", "random_bits"])
def test_encoder_matches_oracle(df11, oracle_mod, case):
    w = _case(case)
    fmt = oracle_mod.encode(w)
    dt = df11.encode_device(_dev(w))
    _compare(dt, fmt)
    out = df11.decompress(dt)                                   # and it decodes back
    torch.cuda.synchronize()
    assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1), w.reshape(-1))


@pytest.mark.parametrize("T,n", [(32, 4), (64, 8), (128, 16), (96, 5), (256, 13), (1024, 8), (1024, 32)])
def test_encoder_geometry(df11, oracle_mod, T, n):
    w = workloads.gaussian_bf16((300001,), seed=T * 7 + n)
    _compare(df11.encode_device(_dev(w), T=T, n=n), oracle_mod.encode(w, T=T, n=n))


@pytest.mark.parametrize("lut_mode", ["narrow", "wide"])
def test_encoder_lut_modes(df11, oracle_mod, lut_mode):
    w = workloads.gaussian_bf16((100003,), seed=31)
    _compare(df11.encode_device(_dev(w), lut_mode=lut_mode), oracle_mod.encode(w, lut_mode=lut_mode))


def test_encoder_unaligned_input_view(df11, oracle_mod):
    """A tensor view starting 2 bytes past a 16-byte boundary (scalar head + vector body)."""
    w = workloads.gaussian_bf16((70001,), seed=41)
    big = torch.zeros(70001 + 8, dtype=torch.int16, device="cuda")
    for off in (1, 3, 7):
        big[off: off + w.size] = _dev(w)
        _compare(df11.encode_device(big[off: off + w.size]), oracle_mod.encode(w))


def test_encoder_shared_codebook_group(df11, oracle_mod):
    """One codebook from the block's summed histogram (R5), then per-tensor packing."""
    ts = [w for _, w in workloads.config_tensors("flux_single_block")]
    dts = df11.encode_device_group([_dev(w) for w in ts], shared_codebook=True)
    group = sum(oracle_mod.histogram(oracle_mod.split(w)[0]) for w in ts)
    for w, dt in zip(ts, dts):
        _compare(dt, oracle_mod.encode(w, codebook_hist=group))
    outs = df11.decompress_block(dts)
    torch.cuda.synchronize()
    for w, o in zip(ts, outs):
        assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), w)


def test_encoder_histogram_and_empty(df11, oracle_mod):
    w = workloads.gaussian_bf16((123457,), seed=51)
    h = df11.histogram_device(_dev(w)).cpu().numpy()
    assert np.array_equal(h, oracle_mod.histogram(oracle_mod.split(w)[0]).astype(np.int64))
    e = np.zeros(0, np.uint16)
    dt = df11.encode_device(_dev(e))
    torch.cuda.synchronize()
    assert dt.meta["B"] == 0 and dt.num_elements == 0
    assert _host(dt.block_output_pos)[:4].view(np.uint32)[0] == 0


def test_encoder_rejects_uncoded_exponent(df11):
    hist = np.zeros(256, np.uint64)
    hist[120] = 10
    own = hist.copy()
    own[121] = 1
    with pytest.raises(df11.Df11Error):
        df11.EncodePlan(hist, own)


def test_encoder_full_size_block(df11, oracle_mod):
    """Llama-3.1-8B block at full size: byte parity for the largest tensor (oracle encoder), and the
    GPU encoder's output decodes back to the original for every tensor."""
    ts = workloads.config_tensors("llama8b_block")
    name, w = max(ts, key=lambda t: t[1].size)
    _compare(df11.encode_device(_dev(w)), oracle_mod.encode(w))
    for name, w in ts:
        dt = df11.encode_device(_dev(w))
        out = df11.decompress(dt)
        torch.cuda.synchronize()
        assert torch.equal(out.reshape(-1).view(torch.int16), _dev(w).reshape(-1)), name


@pytest.mark.parametrize("vf", ["fp16", "fp8_e4m3", "fp8_e5m2"])
@pytest.mark.parametrize("case", ["gauss", "patterns", "ragged", "tiny"])
def test_encoder_value_formats_match_oracle(df11, oracle_mod, vf, case):
    """NEXT-3 x NEXT-4: the device encoder writes the oracle's bytes for FP16 / FP8 words (R-bit residual
    stream included), for aligned and unaligned (view) inputs, and the result decodes back."""
    import workloads as wl
    if case == "gauss":
        w = wl.gaussian_values((1 << 20,), 71, vf)
    elif case == "patterns":
        w = np.tile(wl.all_patterns(vf), 5 if vf == "fp16" else 1000)
        np.random.default_rng(2).shuffle(w)
    elif case == "ragged":
        w = wl.gaussian_values((300007,), 72, vf)
    else:
        w = wl.gaussian_values((19,), 73, vf)
    tdt = torch.int16 if w.dtype == np.uint16 else torch.uint8
    x = torch.from_numpy(w.view(np.int16) if w.dtype == np.uint16 else w).to("cuda")
    fmt = oracle_mod.encode(w, vf=vf)
    _compare(df11.encode_device(x, vf=vf), fmt)
    big = torch.zeros(w.size + 16, dtype=tdt, device="cuda")
    big[3: 3 + w.size] = x
    dt = df11.encode_device(big[3: 3 + w.size], vf=vf)           # unaligned view: scalar head path
    _compare(dt, fmt)
    out = df11.decompress(dt)
    torch.cuda.synchronize()
    got = out.view(tdt).cpu().numpy().view(w.dtype).reshape(-1)
    assert np.array_equal(got, w)


@pytest.mark.parametrize("lut_bits", [3, 12, "mono"])
def test_encoder_lut_bits_match_oracle(df11, oracle_mod, lut_bits):
    w = workloads.gaussian_values((200003,), 74, "fp16")
    x = torch.from_numpy(w.view(np.int16)).to("cuda").view(torch.float16)
    _compare(df11.encode_device(x, lut_bits=lut_bits), oracle_mod.encode(w, vf="fp16", lut_bits=lut_bits))
