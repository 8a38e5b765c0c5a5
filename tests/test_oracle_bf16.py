"""Pins for oracle E1 (split) and the Alg. 1 compose step, and Eq. 2 entropy.

Pins are independent of the oracle's own code: the exhaustive check compares against numpy's view of
the word as a float32 value (Eq. 1), and the worked examples come from tests/golden/.
"""
import math

import numpy as np

from conftest import load_golden


def test_split_compose_exhaustive(oracle_mod):
    """compose(split(w)) == w for all 65 536 BF16 bit patterns (Alg. 1 compose P:429-434)."""
    w = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    exp, psm = oracle_mod.split(w)
    # the split must agree with the bit layout of Eq. 1 (sign 15, exponent 14..7, mantissa 6..0)
    assert np.array_equal(exp, ((w >> 7) & 0xFF).astype(np.uint8))
    assert np.array_equal(psm >> 7, (w >> 15).astype(np.uint8))
    assert np.array_equal(psm & 0x7F, (w & 0x7F).astype(np.uint8))
    back = np.array([oracle_mod.compose(int(e), int(p)) for e, p in zip(exp[::97], psm[::97])], np.uint16)
    assert np.array_equal(back, w[::97])


def test_value_formula_eq1(oracle_mod):
    """Eq. 1: value = (-1)^s 2^(e-127) (1 + m/128) for normal exponents; the BF16 word is
    the top half of the fp32 word, so numpy's float32 view is an independent evaluator."""
    rng = np.random.default_rng(1)
    w = rng.integers(0, 1 << 16, size=4000, dtype=np.uint32).astype(np.uint16)
    exp, psm = oracle_mod.split(w)
    f = (w.astype(np.uint32) << 16).view(np.float32)
    for i in range(w.size):
        e = int(exp[i])
        if e in (0, 255):
            continue
        s = int(psm[i]) >> 7
        m = int(psm[i]) & 0x7F
        assert float(f[i]) == (-1) ** s * 2.0 ** (e - 127) * (1 + m / 128)


def test_split_worked_examples(oracle_mod):
    for ex in load_golden("spec_examples.json")["split"]:
        w = np.array([int(ex["word"], 16)], np.uint16)
        exp, psm = oracle_mod.split(w)
        assert int(exp[0]) == ex["exponent"]
        assert int(psm[0]) >> 7 == ex["sign"] and int(psm[0]) & 0x7F == ex["mantissa"]
        assert oracle_mod.compose(ex["exponent"], (ex["sign"] << 7) | ex["mantissa"]) == int(ex["word"], 16)


def test_entropy_eq2(oracle_mod):
    for ex in load_golden("spec_examples.json")["entropy"]:
        assert abs(oracle_mod.entropy_bits(ex["hist"]) - ex["bits"]) < 1e-12
    # uniform over n symbols -> log2 n exactly; single symbol -> 0
    for n in (1, 2, 3, 7, 256):
        assert abs(oracle_mod.entropy_bits([5] * n) - math.log2(n)) < 1e-12


def test_histogram(oracle_mod):
    rng = np.random.default_rng(2)
    e = rng.integers(0, 256, size=10000, dtype=np.uint8)
    assert np.array_equal(oracle_mod.histogram(e), np.bincount(e, minlength=256).astype(np.uint64))
