"""Host encoder (libdf11.so df11_encode) vs the oracle, byte for byte (CPU only).

The library encoder and oracle/ share no code; both implement DESIGN.md §2.  Every array of the DF11
format must be identical, including the zero padding.
"""
import ctypes

import numpy as np
import pytest

import workloads
from paper_2504_11651_b200 import df11


def _cmp(fmt, h):
    assert h.num_elements == fmt["num_elements"]
    assert h.encoded_bits == fmt["encoded_bits"]
    assert (h.T, h.n, h.B, h.k) == (fmt["T"], fmt["n"], fmt["B"], fmt["k"])
    assert h.lut_entry_bytes == fmt["lut_entry_bytes"] and h.max_code_len == fmt["max_code_len"]
    a = h.arrays()
    for key in ("code_lengths", "luts", "encoded_exponent", "packed_sign_mantissa", "gaps", "block_output_pos"):
        assert np.array_equal(a[key], fmt[key]), key


def test_library_exports_every_header_symbol():
    """The C-ABI library loads and exports every function include/df11.h declares."""
    import re
    import os
    hdr = open(os.path.join(os.path.dirname(df11.library_path()), "..", "..", "include", "df11.h")).read()
    declared = set(re.findall(r"^(?:df11_status|void|int|uint32_t|uint64_t|const char)\s+\*?\s*(df11_\w+)\s*\(",
                              hdr, flags=re.M))
    L = ctypes.CDLL(df11.library_path())
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(df11.EXPORTED_SYMBOLS)
    assert df11.lib().df11_version().decode().startswith("df11-b200")


@pytest.mark.parametrize("case", ["gauss_small", "gauss_ragged", "constant", "two_symbol", "all_patterns",
                                  "overflow_wide", "fibonacci", "one", "empty"])
def test_encoder_bytes_equal_oracle(oracle_mod, case):
    rng = np.random.default_rng(3)
    T, n = 256, 8
    if case == "gauss_small":
        w = workloads.gaussian_bf16((1 << 20,), seed=1)
    elif case == "gauss_ragged":
        w = workloads.gaussian_bf16((1234567,), seed=2, sigma=0.01)
        T, n = 128, 16
    elif case == "constant":
        w = workloads.constant(200003)
    elif case == "two_symbol":
        w = workloads.from_exponent_histogram({100: 7000, 101: 3}, seed=1)
    elif case == "all_patterns":
        w = workloads.all_bf16_patterns()
    elif case == "overflow_wide":
        counts = {120: 1 << 18}
        counts.update({e: 1 + e % 3 for e in range(1, 120)})
        w = workloads.from_exponent_histogram(counts, seed=5)
    elif case == "fibonacci":
        w = workloads.from_exponent_histogram(workloads.fibonacci_histogram(34, 80), seed=1)
        T, n = 64, 4
    elif case == "one":
        w = np.array([0xBF80], np.uint16)
    else:
        w = np.zeros(0, np.uint16)
    fmt = oracle_mod.encode(w, T=T, n=n)
    for threads in (1, 0):
        h = df11.encode(w, T=T, n=n, num_threads=threads)
        _cmp(fmt, h)


def test_encoder_fuzz_vs_oracle(oracle_mod):
    rng = np.random.default_rng(9)
    geoms = [(32, 4), (64, 8), (256, 8), (512, 8), (96, 5), (1024, 16), (32, 32)]
    for i in range(150):
        N = int(rng.integers(1, 200000))
        kind = i % 4
        if kind == 0:
            w = workloads.gaussian_bf16((N,), seed=100 + i, sigma=float(rng.choice([0.003, 0.02, 0.2])))
        elif kind == 1:
            w = rng.integers(0, 1 << 16, size=N, dtype=np.uint32).astype(np.uint16)
        elif kind == 2:
            nsym = int(rng.integers(1, 50))
            counts = {int(e): int(c) for e, c in zip(rng.choice(256, nsym, replace=False),
                                                    rng.geometric(0.05, nsym))}
            w = workloads.from_exponent_histogram(counts, seed=i)
        else:
            w = workloads.constant(N, int(rng.integers(0, 1 << 16)))
        T, n = geoms[i % len(geoms)]
        fmt = oracle_mod.encode(w, T=T, n=n)
        h = df11.encode(w, T=T, n=n, num_threads=int(rng.choice([0, 1, 3])))
        _cmp(fmt, h)


def test_encoder_errors(oracle_mod):
    with pytest.raises(df11.Df11Error) as e:
        df11.encode(workloads.all_bf16_patterns(), lut_mode="narrow")
    assert e.value.kind == "DF11_E_RESERVED_EXPONENT"
    counts = {120: 1 << 18}
    counts.update({e: 1 + e % 3 for e in range(1, 120)})
    with pytest.raises(df11.Df11Error) as e:
        df11.encode(workloads.from_exponent_histogram(counts, seed=5), lut_mode="narrow")
    assert e.value.kind == "DF11_E_LUT_OVERFLOW"
    for T, n in ((33, 8), (2048, 8), (256, 3), (256, 33)):
        with pytest.raises(df11.Df11Error) as e:
            df11.encode(workloads.constant(10), T=T, n=n)
        assert e.value.kind == "DF11_E_INVALID_ARGUMENT"
    h = df11.encode(workloads.all_bf16_patterns(), lut_mode="wide")
    assert h.lut_entry_bytes == 2


def test_encode_group_shared_codebook(oracle_mod):
    ts = workloads.config_tensors("flux_single_block")
    small = [w.reshape(-1)[: 50000 + 7 * i] for i, (_, w) in enumerate(ts)]
    hs = df11.encode_group(small, shared_codebook=True)
    assert len({bytes(h.code_lengths) for h in hs}) == 1
    # the shared codebook is the one the oracle builds from the concatenation
    fmt = oracle_mod.encode(np.concatenate(small))
    assert np.array_equal(hs[0].code_lengths, fmt["code_lengths"])
    assert np.array_equal(hs[0].luts, fmt["luts"])
    per = df11.encode_group(small, shared_codebook=False)
    for w, h in zip(small, per):
        _cmp(oracle_mod.encode(w), h)


def test_encoder_speed_8b_block():
    """The host encoder must keep setup practical: > 50 M elements/s."""
    import time
    w = workloads.gaussian_bf16((14336, 4096), seed=7)
    t = time.perf_counter()
    h = df11.encode(w)
    dt = time.perf_counter() - t
    assert h.num_elements == w.size
    assert w.size / dt > 50e6, w.size / dt


def test_plan_cta_ranges_cover_and_balance():
    """Launcher planning (row a9): the per-CTA tile ranges are non-decreasing, cover every tile
    exactly once, and a CTA whose range holds a tensor start gets about `switch_tiles` fewer tiles."""
    import ctypes
    from paper_2504_11651_b200 import df11
    rng = np.random.default_rng(3)
    L = df11.lib()
    for trial in range(200):
        count = int(rng.integers(1, 20))
        sizes = rng.integers(1, 5000, size=count)
        if trial % 3 == 0:
            sizes[rng.integers(0, count)] = int(rng.integers(1, 16))          # a small tensor
        starts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
        total = int(starts[-1])
        grid = int(rng.integers(1, 200))
        for P in (0, 12):
            out = np.zeros(grid + 1, np.uint32)
            L.df11_plan_cta_ranges(starts.ctypes.data_as(ctypes.c_void_p), count, grid, P,
                                   out.ctypes.data_as(ctypes.c_void_p))
            assert out[0] == 0 and out[-1] == total
            assert np.all(np.diff(out.astype(np.int64)) >= 0)
            if P == 0:          # plain equal split (rounding down)
                assert np.array_equal(out, (np.arange(grid + 1, dtype=np.uint64) * total // grid).astype(np.uint32))
            # work per CTA (tiles + P per interior entry start) differs by at most P + 1 across CTAs
            work = []
            for c in range(grid):
                inner = int(np.sum((starts[1:-1] > out[c]) & (starts[1:-1] < out[c + 1])))
                work.append(int(out[c + 1]) - int(out[c]) + P * inner)
            if total >= grid * (P + 2):
                assert max(work) - min(work) <= 2 * P + 2, (work, P)


# ---------------------------------------------------------------------------- NEXT-4 format variants
def _cmp_variant(fmt, h):
    _cmp(fmt, h)
    assert h.value_format == fmt["value_format"] and h.lut_bits == fmt["lut_bits"]


@pytest.mark.parametrize("vf", ["fp16", "fp8_e4m3", "fp8_e5m2"])
@pytest.mark.parametrize("case", ["gauss", "patterns", "ragged"])
def test_encoder_value_formats_equal_oracle(oracle_mod, vf, case):
    """FP16 / FP8 (R25-R27): the library encoder writes the oracle's bytes (residual stream included),
    single- and multi-threaded, for Gaussian weights, every bit pattern and ragged sizes."""
    if case == "gauss":
        w = workloads.gaussian_values((1 << 19,), 4, vf)
    elif case == "patterns":
        rng = np.random.default_rng(8)
        w = np.tile(workloads.all_patterns(vf), 3 if vf == "fp16" else 300)
        rng.shuffle(w)
    else:
        w = workloads.gaussian_values((300007,), 5, vf)
    fmt = oracle_mod.encode(w, vf=vf)
    for threads in (1, 0):
        _cmp_variant(fmt, df11.encode(w, num_threads=threads, vf=vf))


@pytest.mark.parametrize("lut_bits", [1, 3, 5, 8, 11, 12, 16, "mono"])
def test_encoder_lut_bits_equal_oracle(oracle_mod, lut_bits):
    """b-bit hierarchical tables (App. I.2) and the monolithic table (b = L, App. I.1): same bytes."""
    cases = [workloads.gaussian_bf16((1 << 18,), seed=6),
             workloads.gaussian_values((1 << 18,), 7, "fp8_e4m3"),
             workloads.from_exponent_histogram(workloads.fibonacci_histogram(34, 80), seed=3)]
    for i, w in enumerate(cases):
        vf = "fp8_e4m3" if i == 1 else "bf16"
        try:
            fmt = oracle_mod.encode(w, vf=vf, lut_bits=lut_bits)
        except oracle_mod.FormatError as e:
            assert lut_bits == "mono" and e.kind == "invalid_argument"
            with pytest.raises(df11.Df11Error) as ei:
                df11.encode(w, vf=vf, lut_bits=lut_bits)
            assert ei.value.kind == "DF11_E_INVALID_ARGUMENT"
            continue
        _cmp_variant(fmt, df11.encode(w, vf=vf, lut_bits=lut_bits))


def test_encoder_rejects_bad_variant_options():
    w = workloads.gaussian_bf16((1000,), seed=1)
    for kw in (dict(lut_bits=17), dict(lut_bits=40)):
        with pytest.raises(df11.Df11Error):
            df11.encode(w, **kw)


@pytest.mark.parametrize("vf", ["bf16", "fp16", "fp8_e4m3", "fp8_e5m2"])
def test_device_plan_matches_host_encoder(vf):
    """df11_encode_plan_create (the GPU encoder's host half) plans the host encoder's codebook and sizes
    for every value format and b."""
    w = workloads.gaussian_values((100003,), 3, vf)
    E, M = {"bf16": (8, 7), "fp16": (5, 10), "fp8_e4m3": (4, 3), "fp8_e5m2": (5, 2)}[vf]
    hist = np.bincount((w.astype(np.uint32) >> M) & ((1 << E) - 1), minlength=256).astype(np.uint64)
    for lut_bits in (8, 5, "mono"):
        h = df11.encode(w, vf=vf, lut_bits=lut_bits)
        plan = df11.EncodePlan(hist, vf=vf, lut_bits=lut_bits)
        assert (plan.value_format, plan.lut_bits, plan.k, plan.B) == (h.value_format, h.lut_bits, h.k, h.B)
        assert plan.packed_sign_mantissa_bytes == h.packed_sign_mantissa.size
        assert np.array_equal(plan.code_lengths, h.code_lengths)


def test_encoder_variant_fuzz_vs_oracle(oracle_mod):
    """Seeded sweep: value format x b (incl. monolithic) x (T, n) x lut mode x size x distribution;
    the library encoder writes the oracle's bytes every time."""
    rng = np.random.default_rng(77)
    vfs = ["bf16", "fp16", "fp8_e4m3", "fp8_e5m2"]
    checked = 0
    for i in range(40):
        vf = vfs[i % 4]
        N = int(rng.choice([1, 33, 4097, 70001, 262147]))
        if rng.random() < 0.5:
            w = workloads.gaussian_values((N,), 500 + i, vf, sigma=float(rng.choice([0.003, 0.02, 0.4])))
        else:
            pats = workloads.all_patterns(vf)
            w = pats[rng.integers(0, pats.size, size=N)]
        T, n = [(256, 8), (128, 16), (64, 4), (32, 32)][int(rng.integers(0, 4))]
        lut_bits = [8, 2, 7, 11, 16, "mono"][int(rng.integers(0, 6))]
        mode = ["auto", "wide"][int(rng.integers(0, 2))]
        try:
            fmt = oracle_mod.encode(w, T=T, n=n, lut_mode=mode, vf=vf, lut_bits=lut_bits)
        except oracle_mod.FormatError:
            assert lut_bits == "mono"
            continue
        _cmp_variant(fmt, df11.encode(w, T=T, n=n, lut_mode=mode, vf=vf, lut_bits=lut_bits))
        checked += 1
    assert checked >= 30


def test_missing_library_fails_loudly():
    """The product path has no fallback: without the CUDA library every call raises (no oracle, no CPU
    decode behind the binding)."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np\nfrom paper_2504_11651_b200 import df11\n"
            "try:\n    df11.encode(np.zeros(64, np.uint16))\nexcept ImportError as e:\n    print('RAISED', e)\n")
    env = dict(os.environ, DF11_LIB="/nonexistent/libdf11.so")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "RAISED" in r.stdout and "not built" in r.stdout, r.stdout + r.stderr
    src = open(df11.__file__).read()
    assert "oracle" not in src.replace("# oracle", ""), "the binding must not reach oracle/"
