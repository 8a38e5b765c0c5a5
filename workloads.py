"""Seeded synthetic workloads shared by tests/, bench.py and smoke() — inputs only.

This module holds none of DF11's arithmetic (no splitting, coding or packing).  It only produces BF16
bit patterns (as uint16) with the shapes and value distribution of the paper's workloads
(DESIGN.md §5 "Input recipe"), so that the oracle and the CUDA path can be fed identical inputs.

* Value distribution: w = fp32 N(0, sigma^2) rounded to BF16 (round-to-nearest-even), sigma = 0.02.
  Real LLM linear weights have ~2.6-bit exponent entropy and ~40 used exponents; BF16
  N(0, 0.02) gives 2.545 bits and 27-42 symbols depending on N.
* Shapes: public model configs cross-checked against Table 1 byte counts.
* Seed per tensor: (base_seed * 1_000_003 + crc32(f"{config}/{layer}/{name}")) mod 2^63.
"""
from __future__ import annotations

import zlib

import numpy as np

SIGMA = 0.02


def _llama_block(h, ffn, kv):
    return [("q_proj", (h, h)), ("k_proj", (kv, h)), ("v_proj", (kv, h)), ("o_proj", (h, h)),
            ("gate_proj", (ffn, h)), ("up_proj", (ffn, h)), ("down_proj", (h, ffn))]


def _flux_double_block():
    ts = []
    for stream in ("img", "txt"):
        ts += [(f"{stream}_mod", (18432, 3072)), (f"{stream}_qkv", (9216, 3072)),
               (f"{stream}_proj", (3072, 3072)), (f"{stream}_mlp0", (12288, 3072)),
               (f"{stream}_mlp2", (3072, 12288))]
        ts += [(f"{stream}_mod_b", (18432,)), (f"{stream}_qkv_b", (9216,)), (f"{stream}_proj_b", (3072,)),
               (f"{stream}_mlp0_b", (12288,)), (f"{stream}_mlp2_b", (3072,))]
        ts += [(f"{stream}_q_norm", (128,)), (f"{stream}_k_norm", (128,))]
    return ts


def _flux_single_block():
    return [("linear1", (21504, 3072)), ("linear2", (3072, 15360)), ("mod", (9216, 3072)),
            ("linear1_b", (21504,)), ("linear2_b", (3072,)), ("mod_b", (9216,)),
            ("q_norm", (128,)), ("k_norm", (128,))]


# One "unit" per config = the tensors decoded by ONE df11_decompress_block call.
CONFIGS = {
    "matrix4096": [("w", (4096, 4096))],
    "llama8b_block": _llama_block(4096, 14336, 1024),
    "llama70b_block": _llama_block(8192, 28672, 1024),
    "llama405b_block": _llama_block(16384, 53248, 1024),
    "flux_double_block": _flux_double_block(),
    "flux_single_block": _flux_single_block(),
    "llama70b_embed": [("embed_tokens", (128256, 8192))],
    "llama405b_embed": [("embed_tokens", (128256, 16384))],      # 2.10 G elements: positions past 2^30
}

# BASELINE.json configs -> workload names
BASELINE_CONFIGS = {
    0: "matrix4096",        # single 4096x4096 matrix: the oracle finishes it in seconds
    1: "llama8b_block",     # Llama-3.1-8B-shaped transformer block, block-batched on 1 B200
    2: "llama70b_block",    # swept per block at 1/2/4/8 GPUs
    3: "flux_double_block",
    4: "llama405b_block",
}


def seed_for(config: str, layer: int, name: str, base_seed: int = 0) -> int:
    return (base_seed * 1_000_003 + zlib.crc32(f"{config}/{layer}/{name}".encode())) % (1 << 63)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> BF16 bit pattern, round-to-nearest-even (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def gaussian_bf16(shape, seed: int, sigma: float = SIGMA) -> np.ndarray:
    """BF16(N(0, sigma^2)) as uint16, numpy PCG64 with the given seed."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal(size=int(np.prod(shape)), dtype=np.float32)
    x *= np.float32(sigma)
    return f32_to_bf16_bits(x).reshape(shape)


def student_t_bf16(shape, seed: int, nu: float = 5.0, scale: float = SIGMA) -> np.ndarray:
    """Heavy-tailed realism variant: BF16(scale * Student-t(nu)) as uint16, PCG64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_t(nu, size=int(np.prod(shape))).astype(np.float32)
    x *= np.float32(scale)
    return f32_to_bf16_bits(x).reshape(shape)


def gaussian_bf16_torch(shape, seed: int, device, sigma: float = SIGMA):
    """BF16(N(0, sigma^2)) generated on `device` with torch's Philox (fast, for the multi-GB model
    configs); returned as a host uint16 array (the host encoder's input)."""
    import torch
    g = torch.Generator(device=device).manual_seed(int(seed))
    w = (torch.randn(tuple(shape), generator=g, device=device, dtype=torch.float32) * sigma).to(torch.bfloat16)
    return w.view(torch.int16).cpu().numpy().view(np.uint16)


# --------------------------------------------------------------------------- other value formats
# (NEXT-4, R25-R27): the same N(0, sigma^2) weights stored as FP16, or as FP8 with one
# per-tensor scale that maps the tensor's absolute maximum to the format's largest finite value (the
# usual FP8 weight recipe).  Inputs only: conversions are numpy's / torch's round-to-nearest-even.
VALUE_FORMATS = ("bf16", "fp16", "fp8_e4m3", "fp8_e5m2")
FP8_MAX = {"fp8_e4m3": 448.0, "fp8_e5m2": 57344.0}


def word_dtype(vf: str):
    return np.uint8 if vf.startswith("fp8") else np.uint16


def gaussian_values(shape, seed: int, vf: str = "bf16", sigma: float = SIGMA) -> np.ndarray:
    """N(0, sigma^2) weights as bit patterns of value format vf (uint16 for bf16/fp16, uint8 for fp8)."""
    if vf == "bf16":
        return gaussian_bf16(shape, seed, sigma)
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal(size=int(np.prod(shape)), dtype=np.float32)
    x *= np.float32(sigma)
    if vf == "fp16":
        return x.astype(np.float16).view(np.uint16).reshape(shape)
    import torch
    amax = float(np.abs(x).max()) if x.size else 1.0
    t = torch.from_numpy(x) * (FP8_MAX[vf] / (amax or 1.0))
    dt = torch.float8_e4m3fn if vf == "fp8_e4m3" else torch.float8_e5m2
    return t.to(dt).view(torch.uint8).numpy().copy().reshape(shape)


def all_patterns(vf: str = "bf16") -> np.ndarray:
    """Every bit pattern of the format (65 536 or 256 words)."""
    return np.arange(1 << (8 if vf.startswith("fp8") else 16), dtype=np.uint32).astype(word_dtype(vf))


# Whole-model sweeps: units = transformer blocks (+ embedding first, LM head last).
MODELS = {
    "llama70b_model": dict(block="llama70b_block", blocks=80, vocab=128256, hidden=8192),
    "llama405b_model": dict(block="llama405b_block", blocks=126, vocab=128256, hidden=16384),
}


def config_tensors(config: str, layer: int = 0, base_seed: int = 0, sigma: float = SIGMA, dist: str = "gauss",
                   vf: str = "bf16"):
    """[(name, uint16 array)] for one unit of `config`.  dist: "gauss" (the headline recipe), or the
    realism variants of SURVEY 8(d), reported separately: "t5" (scale * Student-t(5)) and "sigma-lu"
    (per-tensor sigma log-uniform in [0.01, 0.04], drawn from the tensor's seed).  vf != "bf16": the
    Gaussian recipe in another value format (gaussian_values; uint8 arrays for fp8)."""
    out = []
    for name, shape in CONFIGS[config]:
        seed = seed_for(config, layer, name, base_seed)
        if vf != "bf16":
            out.append((name, gaussian_values(shape, seed, vf, sigma)))
        elif dist == "t5":
            out.append((name, student_t_bf16(shape, seed, 5.0, sigma)))
        elif dist == "sigma-lu":
            s = float(np.exp(np.random.Generator(np.random.PCG64(seed ^ 0x5F5F)).uniform(np.log(0.01), np.log(0.04))))
            out.append((name, gaussian_bf16(shape, seed, s)))
        else:
            out.append((name, gaussian_bf16(shape, seed, sigma)))
    return out


def config_numel(config: str) -> int:
    return sum(int(np.prod(s)) for _, s in CONFIGS[config])


# --------------------------------------------------------------------------- adversarial inputs
def all_bf16_patterns() -> np.ndarray:
    """Every one of the 65 536 BF16 bit patterns (incl. inf/NaN/subnormals)."""
    return np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)


def constant(n: int, word: int = 0x3C00) -> np.ndarray:
    return np.full(n, word, np.uint16)


def from_exponent_histogram(counts: dict, seed: int = 0) -> np.ndarray:
    """Words whose exponent histogram is exactly `counts` ({exponent: count}), shuffled, with random
    sign and mantissa bits."""
    rng = np.random.Generator(np.random.PCG64(seed))
    exps = np.concatenate([np.full(int(c), int(e), np.uint16) for e, c in counts.items() if c > 0])
    rng.shuffle(exps)
    sm = rng.integers(0, 256, size=exps.size, dtype=np.uint16)
    return (((sm & 0x80) << 8) | (exps << 7) | (sm & 0x7F)).astype(np.uint16)


def from_exponent_histogram_vf(counts: dict, vf: str, seed: int = 0) -> np.ndarray:
    """from_exponent_histogram for any value format: words of vf whose exponent field histogram is
    exactly `counts`, shuffled, with random sign and mantissa bits."""
    if vf == "bf16":
        return from_exponent_histogram(counts, seed)
    E, M = {"fp16": (5, 10), "fp8_e4m3": (4, 3), "fp8_e5m2": (5, 2)}[vf]
    rng = np.random.Generator(np.random.PCG64(seed))
    exps = np.concatenate([np.full(int(c), int(e), np.uint32) for e, c in counts.items() if c > 0])
    assert exps.max() < (1 << E)
    rng.shuffle(exps)
    sm = rng.integers(0, 1 << (M + 1), size=exps.size, dtype=np.uint32)
    words = ((sm >> M) << (E + M)) | (exps << M) | (sm & ((1 << M) - 1))
    return words.astype(word_dtype(vf))


def fibonacci_histogram(nsym: int = 40, first_exponent: int = 90) -> dict:
    """Fibonacci counts over `nsym` exponents: the unconstrained Huffman tree has depth nsym-1."""
    a, b = 1, 1
    counts = {}
    for i in range(nsym):
        counts[first_exponent + i] = a
        a, b = b, a + b
    return counts
