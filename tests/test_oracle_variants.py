"""Pins for the NEXT-4 format variants in the oracle: value formats FP16 / FP8 E4M3 / FP8 E5M2 (R25-R27)
and b-bit hierarchical LUTs incl. the monolithic table (App. I.1-I.2, R28).

Independent pins:
* split_v is checked against the VALUE of every bit pattern, as evaluated by numpy (float16) or torch
  (float8_e4m3fn / float8_e5m2): sign, exponent and mantissa are recovered from the value by the
  textbook formulas of each format (normal: (-1)^s 2^(e-bias) (1 + m/2^M); subnormal: 2^(1-bias) m/2^M),
  and the packed residual bits are re-read with numpy's unpackbits;
* b-bit tables: a bit-by-bit code-tree walk written here (the unique codeword that prefixes the stream)
  on fuzzed codebooks for every b in [1, 16]; b = L reproduces the paper's monolithic LUT (P:537-539,
  tests/golden/paper_appendix_I.json) exactly;
* decoders D1 / D2: round trip = identity (the definition of lossless) for every bit pattern of every
  format and every b.
"""
import math

import numpy as np
import pytest

import workloads
from conftest import load_golden
from oracle import huffman

FORMATS = {  # name: (word bits, exponent bits, mantissa bits, bias)
    "fp16": (16, 5, 10, 15),
    "fp8_e4m3": (8, 4, 3, 7),
    "fp8_e5m2": (8, 5, 2, 15),
}


def _values(vf, words):
    """float64 values of the bit patterns, evaluated by numpy / torch (not by bit manipulation here)."""
    if vf == "fp16":
        return words.view(np.float16).astype(np.float64)
    import torch
    dt = torch.float8_e4m3fn if vf == "fp8_e4m3" else torch.float8_e5m2
    return torch.from_numpy(words.copy()).view(dt).to(torch.float64).numpy()


def _fields_from_value(vf, v):
    """(sign, exponent, mantissa) of a finite value from the format's textbook definition."""
    _, E, M, bias = FORMATS[vf]
    s = 1 if math.copysign(1.0, v) < 0 else 0
    a = abs(v)
    if a < 2.0 ** (1 - bias):                       # subnormal or zero: a = 2^(1-bias) m / 2^M
        m = a / 2.0 ** (1 - bias) * (1 << M)
        assert m == int(m)
        return s, 0, int(m)
    e = math.floor(math.log2(a))
    m = (a / 2.0 ** e - 1.0) * (1 << M)
    assert m == int(m)
    return s, e + bias, int(m)


def _residual_fields(res, R, n):
    """Read the residuals back by the R25 layout: R >= 8: byte plane of the low 8 bits (roundup(n, 16)
    bytes) + the (R - 8)-bit plane MSB-first; R < 8: one R-bit plane MSB-first."""
    def plane(buf, r):
        bits = np.unpackbits(buf)[: r * n].reshape(n, r)
        return bits.dot(1 << np.arange(r - 1, -1, -1)).astype(np.int64)
    if R < 8:
        return plane(res, R)
    lo = res[:n].astype(np.int64)
    if R == 8:
        return lo
    L = (n + 15) // 16 * 16
    return (plane(res[L:], R - 8) << 8) | lo


@pytest.mark.parametrize("vf", sorted(FORMATS))
def test_split_v_against_values(oracle_mod, vf):
    """Every bit pattern: exponent symbol and residual (sign << M | mantissa, stored by the R25 layout)
    equal the fields recovered from the numpy/torch value; infinities and NaNs by class."""
    W, E, M, bias = FORMATS[vf]
    words = workloads.all_patterns(vf)
    exp, res = oracle_mod.split_v(words, vf)
    R = oracle_mod.residual_bits(vf)
    assert R == 1 + M
    assert res.size == oracle_mod.residual_array_bytes(words.size, vf)
    r = _residual_fields(res, R, words.size)
    vals = _values(vf, words)
    checked = 0
    for i in range(words.size):
        v = float(vals[i])
        s_got, m_got = int(r[i]) >> M, int(r[i]) & ((1 << M) - 1)
        if math.isnan(v):
            # E5M2 / FP16: all-ones exponent, nonzero mantissa; E4M3 (fn): only S.1111.111
            assert int(exp[i]) == (1 << E) - 1 and m_got != 0
            continue
        if math.isinf(v):
            assert int(exp[i]) == (1 << E) - 1 and m_got == 0 and s_got == (1 if v < 0 else 0)
            continue
        assert (s_got, int(exp[i]), m_got) == _fields_from_value(vf, v), hex(int(words[i]))
        checked += 1
    assert checked >= (words.size * 7) // 8


@pytest.mark.parametrize("vf", ["bf16", "fp16", "fp8_e4m3", "fp8_e5m2"])
def test_compose_v_inverts_split_v(oracle_mod, vf):
    words = workloads.all_patterns(vf)
    exp, res = oracle_mod.split_v(words, vf)
    R = oracle_mod.residual_bits(vf)
    r = _residual_fields(res, R, words.size)
    idx = range(0, words.size, 7 if words.size > 256 else 1)
    assert all(oracle_mod.compose_v(vf, int(exp[i]), int(r[i])) == int(words[i]) for i in idx)


def test_split_v_bf16_is_the_paper_layout(oracle_mod):
    """For BF16, R = 8 and the residual stream is one byte per element, sign in bit 7 and mantissa in
    bits 6..0: identical to the BF16 split E1."""
    w = workloads.all_patterns("bf16")
    e1, p1 = oracle_mod.split(w)
    e2, p2 = oracle_mod.split_v(w, "bf16")
    assert np.array_equal(e1, e2) and np.array_equal(p1, p2[: w.size])
    assert not p2[w.size:].any()


@pytest.mark.parametrize("b", list(range(1, 17)))
def test_b_bit_tables_equal_tree_walk(b):
    """App. I.2 with generic b: every lookup chain over the b-bit tables decodes the unique codeword
    prefixing the stream (fuzzed codebooks, lengths up to 32)."""
    rng = np.random.default_rng(100 + b)
    for trial in range(30):
        nsym = int(rng.integers(2, 48))
        syms = rng.choice(256, size=nsym, replace=False)
        h = [0] * 256
        for s in syms:
            h[int(s)] = int(rng.pareto(0.6) * 10) + 1
        lengths = huffman.code_lengths(h)
        codes = huffman.canonical_codes(lengths)
        tables, depth = huffman.hierarchical_luts(lengths, codes, b=b)
        assert all(len(t) == 1 << b for t in tables)
        assert max(depth) <= (max(lengths) - 1) // b
        present = [s for s in range(256) if lengths[s]]
        for _ in range(10):
            s = int(rng.choice(present))
            bits = format(codes[s], f"0{lengths[s]}b") + "".join(rng.choice(["0", "1"], size=40))
            want = None
            for t in present:
                if bits.startswith(format(codes[t], f"0{lengths[t]}b")):
                    want = (t, lengths[t])
            assert want == (s, lengths[s])
            assert huffman.lut_decode_step(tables, lengths, bits, b=b) == want


def test_monolithic_is_b_equal_L():
    """App. I.1: with b = L the hierarchy is ONE table, equal to the paper's monolithic LUT
    of the L = 4 example (A..F)."""
    g = load_golden("paper_appendix_I.json")
    names = "ABCDEF"
    lengths = [0] * 256
    for i, nm in enumerate(names):
        lengths[i] = g["code_lengths"][nm]
    codes = huffman.canonical_codes(lengths)
    tables, depth = huffman.hierarchical_luts(lengths, codes, b=max(lengths))
    assert len(tables) == 1 and depth == [0] and len(tables[0]) == 16
    for idx, nm in g["monolithic_lut_L4"]["entries"].items():
        assert tables[0][int(idx)] == names.index(nm)


@pytest.mark.parametrize("vf", ["bf16", "fp16", "fp8_e4m3", "fp8_e5m2"])
def test_round_trip_all_patterns(oracle_mod, vf):
    """D1 and D2 rebuild every bit pattern of the format (each pattern present, shuffled, plus a
    Gaussian tensor), for the paper's tables and for b = 5 and the monolithic table."""
    rng = np.random.default_rng(11)
    pats = workloads.all_patterns(vf)
    reps = 1 if pats.size > 256 else 40
    w = np.concatenate([np.tile(pats, reps), workloads.gaussian_values((30011,), 3, vf)])
    rng.shuffle(w)
    for lut_bits in (8, 5):
        fmt = oracle_mod.encode(w, lut_bits=lut_bits, vf=vf)
        assert fmt["value_format"] == oracle_mod.vf_code(vf) and fmt["lut_bits"] == lut_bits
        assert fmt["luts"].size == fmt["k"] * (1 << lut_bits) * fmt["lut_entry_bytes"]
        assert np.array_equal(oracle_mod.decode_sequential(fmt), w)
        assert np.array_equal(oracle_mod.decode_alg1(fmt), w)
    if vf != "bf16":                                  # <= 32 symbols: L <= 16 here
        fmt = oracle_mod.encode(w, lut_bits="mono", vf=vf)
        assert fmt["k"] == 1 and fmt["lut_bits"] == fmt["max_code_len"]
        assert np.array_equal(oracle_mod.decode_alg1(fmt), w)


@pytest.mark.parametrize("lut_bits", [1, 2, 3, 4, 6, 7, 9, 10, 11, 12, 13, 16, "mono"])
def test_round_trip_generic_b(oracle_mod, lut_bits):
    """D2 over b-bit tables on LLM-like BF16 exponents (L typically 12-20) and on a Fibonacci
    histogram (L = 32 through package-merge), and the monolithic table when L <= 16."""
    w1 = workloads.gaussian_bf16((3, 20001), seed=5)
    w2 = workloads.from_exponent_histogram(workloads.fibonacci_histogram(34), seed=2)
    for w in (w1, w2):
        try:
            fmt = oracle_mod.encode(w, lut_bits=lut_bits)
        except oracle_mod.FormatError as e:
            assert lut_bits == "mono" and e.kind == "invalid_argument"
            continue
        assert np.array_equal(oracle_mod.decode_alg1(fmt), w.reshape(-1))
    # the monolithic table at L <= 16: one table of 2^L entries
    w3 = workloads.from_exponent_histogram({100 + i: 2 ** (12 - i) for i in range(12)}, seed=4)
    fmt = oracle_mod.encode(w3, lut_bits="mono")
    assert fmt["k"] == 1 and fmt["lut_bits"] == fmt["max_code_len"] <= 16
    assert np.array_equal(oracle_mod.decode_alg1(fmt), w3)


def test_fp_formats_compress(oracle_mod):
    """Sanity of the variant formats on N(0, 0.02) weights: the exponent costs between H and H + 1 bits
    (Huffman), the residual exactly R bits, and the stored size follows (R + L_bar + gaps) / 8."""
    for vf in ("fp16", "fp8_e4m3", "fp8_e5m2"):
        w = workloads.gaussian_values((1 << 18,), 9, vf)
        fmt = oracle_mod.encode(w, vf=vf)
        N = w.size
        H = oracle_mod.entropy_bits(fmt["histogram"])
        Lbar = fmt["encoded_bits"] / N
        assert H <= Lbar < H + 1
        R = oracle_mod.residual_bits(vf)
        size = oracle_mod.compressed_bytes(fmt)
        meta = 4 * (fmt["B"] + 1) + fmt["luts"].size + 256           # BlockOutputPos, LUTs, CodeLengths
        assert abs(size - (N * (R + Lbar) / 8 + 5 * fmt["B"] * fmt["T"] / 8 + meta)) <= 3
