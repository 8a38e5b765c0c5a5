"""GPU parity of the NEXT-4 format variants through the C ABI: value formats FP16 / FP8 E4M3 / FP8 E5M2
(R25-R27) and b-bit hierarchical / monolithic LUTs (App. I.1-I.2, R28), on both kernels.

Every case: GPU decode == original words (the definition of lossless, P:8) == oracle D1 on the same
oracle-encoded arrays; at full size, every element vs the original plus oracle D2 (Alg. 1) on sampled
format blocks including the last.  Inputs from workloads.py; expected values from the generator or
oracle/ only.
"""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VFS = ["bf16", "fp16", "fp8_e4m3", "fp8_e5m2"]
E_BITS = {"bf16": 8, "fp16": 5, "fp8_e4m3": 4, "fp8_e5m2": 5}


@pytest.fixture(scope="module")
def df11():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2504_11651_b200 import df11 as m
    m.lib()
    return m


def _meta(fmt):
    return {k: fmt[k] for k in ("num_elements", "T", "n", "B", "k", "lut_entry_bytes", "encoded_bits",
                                "max_code_len", "value_format", "lut_bits")}


def _words(out, vf):
    wt = workloads.word_dtype(vf)
    return out.view(torch.int16 if wt is np.uint16 else torch.uint8).cpu().numpy().view(wt).reshape(-1)


def _decode(df11, fmt, kernel):
    dt = df11.DeviceTensor.from_arrays(_meta(fmt), fmt)
    out = df11.decompress(dt, kernel=kernel)
    torch.cuda.synchronize()
    assert df11.last_kernels() == {kernel}
    return _words(out, df11.VF_NAMES[fmt["value_format"]])


def _check(df11, oracle_mod, w, vf, kernel, **kw):
    fmt = oracle_mod.encode(w, vf=vf, **kw)
    got = _decode(df11, fmt, kernel)
    assert np.array_equal(got, w.reshape(-1))
    if w.size <= 3_000_000:
        assert np.array_equal(got, oracle_mod.decode_sequential(fmt))


def _weights(case, vf):
    E = E_BITS[vf]
    top = (1 << E) - 1
    if case == "gauss":
        return workloads.gaussian_values((3 * 16384 * 3 + 12345,), 21, vf)
    if case == "gauss_1m":
        return workloads.gaussian_values((1 << 20,), 22, vf)
    if case == "patterns":
        pats = workloads.all_patterns(vf)
        w = np.tile(pats, 1 if pats.size > 256 else 400)
        np.random.default_rng(1).shuffle(w)
        return w
    if case == "tiny":
        return workloads.gaussian_values((17,), 23, vf)
    if case == "one":
        return workloads.gaussian_values((1,), 24, vf)
    if case == "constant_1bit":          # one symbol: 1-bit codes, count + direct path
        return workloads.from_exponent_histogram_vf({top // 2: 16384 * 5 + 3}, vf, seed=2)
    if case == "one_bit_tail":           # p > 1/2 symbol + geometric tail
        counts = {top // 2: 300000}
        counts.update({e: max(1, int(40000 * 0.5 ** i)) for i, e in enumerate(range(top // 2))})
        return workloads.from_exponent_histogram_vf(counts, vf, seed=3)
    if case == "uniform4_2bit":          # 2-bit codes: the most elements per tile (FP16: residuals
        #                                  above the SMEM staging cap, read per element)
        return workloads.from_exponent_histogram_vf({i + 1: 70000 for i in range(4)}, vf, seed=4)
    if case == "escapes":                # geometric: codes longer than the 12-bit decode table
        counts = {e: int(300000 * 0.7 ** i) + 1 for i, e in enumerate(range(min(top + 1, 40)))}
        return workloads.from_exponent_histogram_vf(counts, vf, seed=5)
    raise ValueError(case)


CASES = ["gauss", "gauss_1m", "patterns", "tiny", "one", "constant_1bit", "one_bit_tail", "uniform4_2bit",
         "escapes"]


@pytest.mark.parametrize("kernel", ["alg1", "fast"])
@pytest.mark.parametrize("vf", VFS)
@pytest.mark.parametrize("case", CASES)
def test_value_format_parity(df11, oracle_mod, case, vf, kernel):
    _check(df11, oracle_mod, _weights(case, vf), vf, kernel)


@pytest.mark.parametrize("vf", VFS)
def test_value_format_n16(df11, oracle_mod, vf):
    """The product kernel's T = 128, n = 16 build with every value format."""
    for case in ("gauss", "escapes", "constant_1bit"):
        _check(df11, oracle_mod, _weights(case, vf), vf, "fast", T=128, n=16)


@pytest.mark.parametrize("kernel", ["alg1", "fast"])
@pytest.mark.parametrize("lut_bits", [1, 2, 5, 7, 8, 11, 12, 16, "mono"])
def test_lut_bits_parity(df11, oracle_mod, lut_bits, kernel):
    """b-bit tables: decode through them (Alg. 1 walks them for every code; the product kernel builds
    its 12-bit table from them and walks them for codes longer than 12 bits)."""
    cases = [("bf16", workloads.gaussian_bf16((200001,), seed=31)),
             ("bf16", workloads.from_exponent_histogram(workloads.fibonacci_histogram(34, 80), seed=32)),
             ("fp16", _weights("escapes", "fp16")),
             ("fp8_e4m3", _weights("gauss", "fp8_e4m3"))]
    for vf, w in cases:
        try:
            fmt = oracle_mod.encode(w, vf=vf, lut_bits=lut_bits)
        except oracle_mod.FormatError:
            assert lut_bits == "mono"
            continue
        got = _decode(df11, fmt, kernel)
        assert np.array_equal(got, w.reshape(-1)), (vf, lut_bits)


@pytest.mark.parametrize("vf", ["fp16", "fp8_e4m3", "fp8_e5m2"])
def test_value_format_llama8b_block_full_size(df11, oracle_mod, vf):
    """The Llama-3.1-8B block (configs[1]) in another value format, library-encoded, one batched
    product launch: every element == original; oracle D2 on sampled blocks incl. the last of each."""
    ws = workloads.config_tensors("llama8b_block", vf=vf)
    hs = [df11.encode(w, vf=vf) for _, w in ws]
    dts = [df11.to_device(h) for h in hs]
    outs = df11.decompress_block(dts)
    torch.cuda.synchronize()
    assert df11.last_kernels() == {"fast"}
    for (name, w), h, o in zip(ws, hs, outs):
        got = _words(o, vf)
        assert np.array_equal(got, w.reshape(-1)), name
        fmt = dict(h.arrays(), num_elements=h.num_elements, T=h.T, n=h.n, B=h.B, k=h.k,
                   lut_entry_bytes=h.lut_entry_bytes, value_format=h.value_format, lut_bits=h.lut_bits)
        for b, (lo, vals) in oracle_mod.decode_alg1_blocks(fmt, [0, h.B // 2, h.B - 1]).items():
            assert np.array_equal(got[lo: lo + vals.size], vals), (name, b)


def test_mixed_value_format_batch(df11):
    """One df11_decompress_block over tensors of all four value formats (and both n): one product
    launch per (n, format), results bit-exact."""
    items = []
    for i, vf in enumerate(VFS):
        w = workloads.gaussian_values((300000 + 1000 * i,), 40 + i, vf)
        items.append((vf, w, df11.encode(w, vf=vf, T=128 if i % 2 else 256, n=16 if i % 2 else 8)))
    dts = [df11.to_device(h) for _, _, h in items]
    n0 = df11.launch_count()
    outs = df11.decompress_block(dts)
    torch.cuda.synchronize()
    assert df11.launch_count() - n0 == 4 and df11.last_kernels() == {"fast"}
    for (vf, w, _), o in zip(items, outs):
        assert np.array_equal(_words(o, vf), w)


def test_value_format_host_path(df11):
    """df11_decompress_host with FP8 / FP16: the D2H copy moves N words of the format's width."""
    for vf in ("fp16", "fp8_e5m2"):
        w = workloads.gaussian_values((123457,), 50, vf)
        h = df11.encode(w, vf=vf)
        dt = df11.to_device(h)
        host = torch.empty(w.size, dtype=df11.out_dtype(vf)).pin_memory()
        df11.decompress_host(h, dt, host)
        torch.cuda.synchronize()
        assert np.array_equal(_words(host, vf), w)


def test_fp16_large_tensor_offsets(df11):
    """FP16 with 420 M elements: residual bit positions (11 * index) pass 2^32, which the product kernel
    handles in modular 32-bit arithmetic relative to the staged range.  Every element == original."""
    N = 420_000_000
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.randn(N, generator=g, device="cuda") * 0.02).to(torch.float16)
    dt = df11.encode_device(x)                                      # GPU encoder (byte parity elsewhere)
    out = df11.decompress(dt, kernel="fast")
    torch.cuda.synchronize()
    assert df11.last_kernels() == {"fast"}
    assert torch.equal(out.view(torch.int16), x.view(torch.int16))


@pytest.mark.parametrize("vf,lut_bits", [("fp16", 8), ("fp8_e4m3", 8), ("fp8_e5m2", 5), ("bf16", 5), ("fp16", "mono")])
def test_corrupt_metadata_variants_never_fault(df11, vf, lut_bits):
    """df11.h robustness contract for the format variants: random Gaps / BlockOutputPos / LUTs /
    CodeLengths / stream bytes may give wrong output but never an out-of-bounds access (run under
    compute-sanitizer memcheck in profiles/r02_final_sanitizer.log)."""
    w = workloads.gaussian_values((150001,), 81, vf)
    h = df11.encode(w, vf=vf, lut_bits=lut_bits)
    a = h.arrays()
    rng = np.random.default_rng(3)
    meta = dict(num_elements=h.num_elements, T=h.T, n=h.n, B=h.B, k=h.k, lut_entry_bytes=h.lut_entry_bytes,
                encoded_bits=h.encoded_bits, max_code_len=h.max_code_len, value_format=h.value_format,
                lut_bits=h.lut_bits)
    for trial in range(6):
        b = {k: np.array(v, copy=True) for k, v in a.items()}
        key = ["block_output_pos", "luts", "code_lengths", "gaps", "encoded_exponent", "packed_sign_mantissa"][trial]
        if key == "block_output_pos":
            b[key] = rng.integers(0, 1 << 32, size=b[key].size, dtype=np.uint64).astype(np.uint32)
        else:
            b[key] = rng.integers(0, 256, size=b[key].size, dtype=np.uint8)
        for kernel in ("alg1", "fast"):
            dt = df11.DeviceTensor.from_arrays(meta, b)
            df11.decompress(dt, kernel=kernel)
            torch.cuda.synchronize()   # a fault would raise here
