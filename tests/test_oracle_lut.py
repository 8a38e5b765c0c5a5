"""Pins for oracle E5 (hierarchical LUTs) and the monolithic LUT.

Independent pins: the paper's App. I worked examples (tests/golden/paper_appendix_I.json), and a
bit-by-bit code-tree walk written here from the codebook (decode = the unique codeword that is a
prefix of the stream) on fuzzed codebooks.
"""
import numpy as np
import pytest

from conftest import load_golden

from oracle import huffman

NAMES = "ABCDEF"


def _paper_codebook():
    g = load_golden("paper_appendix_I.json")
    lengths = [0] * 256
    for i, nm in enumerate(NAMES):
        lengths[i] = g["code_lengths"][nm]
    return g, lengths, huffman.canonical_codes(lengths)


def test_monolithic_example():
    g, lengths, codes = _paper_codebook()
    table = huffman.monolithic_lut(lengths, codes)
    assert len(table) == 16
    for idx, nm in g["monolithic_lut_L4"]["entries"].items():
        assert table[int(idx)] == NAMES.index(nm)


def test_hierarchical_b2_example():
    """with b = 2 the tree splits into exactly LUT_0, LUT_1, LUT_2 as printed."""
    g, lengths, codes = _paper_codebook()
    tables, depth = huffman.hierarchical_luts(lengths, codes, b=2)
    assert len(tables) == 3 and depth == [0, 1, 1]
    for t in range(3):
        want = g["hierarchical_luts_b2"][f"LUT_{t}"]
        got = []
        for e in tables[t]:
            got.append(f"->{e[1]}" if isinstance(e, tuple) else NAMES[e])
        assert got == want


def _tree_walk(lengths, codes, bits):
    """Reference decode step: the codeword that is a prefix of `bits` (prefix-free => unique)."""
    for s in range(256):
        l = lengths[s]
        if l and bits[:l] == format(codes[s], f"0{l}b"):
            return s, l
    raise AssertionError("no codeword matches")


def _random_codebook(rng, nsym, cap=32):
    syms = rng.choice(256, size=nsym, replace=False)
    h = [0] * 256
    # heavy-tailed counts so that long codes (several LUT levels) appear
    for s in syms:
        h[int(s)] = int(rng.pareto(0.6) * 10) + 1
    lengths = huffman.code_lengths(h, cap)
    return lengths, huffman.canonical_codes(lengths)


def test_hierarchical_equals_tree_walk_fuzz():
    rng = np.random.default_rng(7)
    checked = 0
    for trial in range(400):
        nsym = int(rng.integers(2, 64))
        lengths, codes = _random_codebook(rng, nsym)
        tables, _ = huffman.hierarchical_luts(lengths, codes, b=8)
        present = [s for s in range(256) if lengths[s]]
        for _ in range(20):
            s = int(rng.choice(present))
            tail = "".join(rng.choice(["0", "1"], size=40))
            bits = format(codes[s], f"0{lengths[s]}b") + tail
            assert huffman.lut_decode_step(tables, lengths, bits) == _tree_walk(lengths, codes, bits) == (s, lengths[s])
            checked += 1
    assert checked == 8000


def test_hierarchical_equals_monolithic_small_L():
    rng = np.random.default_rng(8)
    for _ in range(200):
        nsym = int(rng.integers(2, 30))
        lengths, codes = _random_codebook(rng, nsym, cap=12)
        L = max(lengths)
        mono = huffman.monolithic_lut(lengths, codes)
        tables, _ = huffman.hierarchical_luts(lengths, codes, b=8)
        for i in range(0, 1 << L, max(1, (1 << L) // 512)):
            bits = format(i, f"0{L}b")
            assert huffman.lut_decode_step(tables, lengths, bits)[0] == mono[i]


def test_narrow_pointer_encoding():
    """Alg. 1: an entry >= 240 is a pointer and LUT_{257-v} (1-based) must be the child;
    the serialized narrow table stores child j as 256-j."""
    rng = np.random.default_rng(9)
    for _ in range(100):
        lengths, codes = _random_codebook(rng, int(rng.integers(20, 60)))
        lengths = [l if s < 240 else 0 for s, l in enumerate(lengths)]
        if sum(1 for l in lengths if l) < 2:
            continue
        # rebuild a valid codebook over symbols < 240
        h = [1 << (32 - l) if l else 0 for l in lengths]
        lengths = huffman.code_lengths(h)
        codes = huffman.canonical_codes(lengths)
        tables, _ = huffman.hierarchical_luts(lengths, codes, b=8)
        if len(tables) - 1 > 16:
            continue
        raw = huffman.serialize_luts(tables, wide=False)
        assert len(raw) == 256 * len(tables)
        for t, table in enumerate(tables):
            for i, e in enumerate(table):
                v = raw[t * 256 + i]
                if isinstance(e, tuple):
                    assert v >= 240 and (257 - v) - 1 == e[1]
                else:
                    assert v == e and v < 240


def test_single_symbol_table_total():
    lengths = [0] * 256
    lengths[50] = 1
    codes = huffman.canonical_codes(lengths)
    tables, _ = huffman.hierarchical_luts(lengths, codes)
    assert len(tables) == 1 and all(e == 50 for e in tables[0])


@pytest.mark.parametrize("sigma", [0.01, 0.02, 0.04])
def test_gaussian_k_in_paper_range(oracle_mod, sigma):
    """'k ranges from 4 to 8'; L 24-32 for LLMs (ours smaller for 1M elements)."""
    import workloads
    w = workloads.gaussian_bf16((1 << 20,), seed=11, sigma=sigma)
    exp, _ = oracle_mod.split(w)
    h = [int(x) for x in oracle_mod.histogram(exp)]
    lengths = huffman.code_lengths(h)
    tables, _ = huffman.hierarchical_luts(lengths, huffman.canonical_codes(lengths))
    g = load_golden("table1_ratios.json")
    assert 2 <= len(tables) <= g["k_max"]
    assert huffman.narrow_is_legal(lengths, tables)
