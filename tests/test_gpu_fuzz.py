"""Seeded random sweep over the format space on the GPU: value format, LUT width b (incl. the monolithic
table), (T, n), lut mode, tensor size (tiny .. several thousand format blocks) and exponent
distribution, each decoded by both kernels through the C ABI and compared element by element with the
original words and oracle D1 (expected values from workloads.py / oracle/ only)."""
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


def _case(i):
    rng = np.random.default_rng(1000 + i)
    vf = VFS[i % 4]
    N = int(rng.choice([1, 7, 255, 4097, 65536 + 13, 300001, 1 << 20, 2_500_003]))
    kind = ["gauss", "geometric", "uniform", "patterns"][int(rng.integers(0, 4))]
    top = (1 << E_BITS[vf]) - 1
    if kind == "gauss":
        w = workloads.gaussian_values((N,), 2000 + i, vf, sigma=float(rng.choice([0.002, 0.02, 0.5])))
    elif kind == "geometric":
        r = float(rng.uniform(0.3, 0.85))
        syms = rng.choice(top + 1, size=min(top + 1, int(rng.integers(2, 48))), replace=False)
        counts = {int(s): max(1, int(N * (1 - r) * r ** k)) for k, s in enumerate(syms)}
        w = workloads.from_exponent_histogram_vf(counts, vf, seed=i)
    elif kind == "uniform":
        syms = rng.choice(top + 1, size=int(rng.integers(1, min(top + 1, 40) + 1)), replace=False)
        w = workloads.from_exponent_histogram_vf({int(s): max(1, N // len(syms)) for s in syms}, vf, seed=i)
    else:
        pats = workloads.all_patterns(vf)
        w = pats[rng.integers(0, pats.size, size=N)]
    T, n = [(256, 8), (128, 16), (64, 4), (512, 8), (32, 32)][int(rng.integers(0, 5))]
    lut_bits = [8, 8, 8, 3, 6, 10, 13, "mono"][int(rng.integers(0, 8))]
    lut_mode = ["auto", "auto", "wide"][int(rng.integers(0, 3))]
    return vf, w, dict(T=T, n=n, lut_bits=lut_bits, lut_mode=lut_mode), kind


@pytest.mark.parametrize("i", range(48))
def test_fuzz_parity(df11, oracle_mod, i):
    vf, w, kw, kind = _case(i)
    try:
        fmt = oracle_mod.encode(w, vf=vf, **kw)
    except oracle_mod.FormatError as e:                  # e.g. monolithic with L > 16
        assert kw["lut_bits"] == "mono", e
        return
    meta = {k: fmt[k] for k in ("num_elements", "T", "n", "B", "k", "lut_entry_bytes", "encoded_bits",
                                "max_code_len", "value_format", "lut_bits")}
    want = w.reshape(-1)
    if want.size <= 1_100_000:
        assert np.array_equal(oracle_mod.decode_sequential(fmt), want)
    fast_ok = (kw["T"], kw["n"]) in ((256, 8), (128, 16))
    wt = workloads.word_dtype(vf)
    for kernel in ("alg1", "fast"):
        dt = df11.DeviceTensor.from_arrays(meta, fmt)
        if kernel == "fast" and not fast_ok:
            with pytest.raises(df11.Df11Error):
                df11.decompress(dt, kernel=kernel)
            continue
        out = df11.decompress(dt, kernel=kernel)
        torch.cuda.synchronize()
        got = out.view(torch.int16 if wt is np.uint16 else torch.uint8).cpu().numpy().view(wt).reshape(-1)
        assert np.array_equal(got, want), (i, vf, kind, kw, kernel)
