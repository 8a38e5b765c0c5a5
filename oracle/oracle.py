"""DF11 CPU oracle — orchestration of E1..E9 and the decoders D1/D2 over numpy arrays.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this module.  It shares no code with paper_2504_11651_b200/ and
neither imports the other.

The bulk loops live in plain C (df11_oracle.c, compiled to liboracle.so by build_oracle()); the
per-codebook steps live in huffman.py.  Citations "P:n" = PAPER.md line n; R-numbers = DESIGN.md §3.

Format produced ("DF11 format"):
    num_elements N, encoded_bits, T, n, B, k, lut_entry_bytes (1 narrow | 2 wide), max_code_len,
    value_format (bf16 | fp16 | fp8_e4m3 | fp8_e5m2, R25), lut_bits b (8 = the paper; R28)
    code_lengths          uint8[256]
    luts                  uint8[k*2^b*lut_entry_bytes]          (App. I.2)
    encoded_exponent      uint8[B*T*n + 16], MSB-first stream
    packed_sign_mantissa  uint8[roundup(R*roundup(N,16)/8,16) + 16], R-bit residuals MSB-first
                          (R = 8 for BF16: one byte per element)
    gaps                  uint8[roundup(ceil(5BT/8),16) + 16]
    block_output_pos      uint32[B+1]
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

from . import huffman

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "df11_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile the plain-C oracle with gcc -O2 (no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        U64, U32, I = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        lib.df11o_split.argtypes = [P, U64, P, P]
        lib.df11o_compose.argtypes = [ctypes.c_uint8, ctypes.c_uint8]
        lib.df11o_compose.restype = ctypes.c_uint16
        lib.df11o_split_v.argtypes = [P, U64, I, P, P]
        lib.df11o_compose_v.argtypes = [I, U32, U32]
        lib.df11o_compose_v.restype = U32
        lib.df11o_vf_residual_bits.argtypes = [I]
        lib.df11o_vf_residual_bits.restype = I
        lib.df11o_histogram.argtypes = [P, U64, P]
        lib.df11o_pack_bits.argtypes = [P, U64, P, P, P]
        lib.df11o_pack_bits.restype = U64
        lib.df11o_gaps_bop.argtypes = [P, U64, P, U32, U32, U32, P, P]
        lib.df11o_gaps_bop.restype = I
        lib.df11o_pack_gaps.argtypes = [P, U64, P]
        lib.df11o_decode_sequential.argtypes = [P, U64, P, P, U64, U64, I, P]
        lib.df11o_decode_sequential.restype = I
        lib.df11o_decode_sequential_range.argtypes = [P, U64, P, P, U64, U64, U64, U64, U64, I, P]
        lib.df11o_decode_sequential_range.restype = I
        lib.df11o_decode_alg1.argtypes = [P, U32, U32, U32, P, P, U64, P, U64, P, P, U64, U32, U32, U32, U64, I, I,
                                          P]
        lib.df11o_decode_alg1.restype = I
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _roundup(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# --------------------------------------------------------------------------- value formats (R25)
VALUE_FORMATS = {"bf16": 0, "fp16": 1, "fp8_e4m3": 2, "fp8_e5m2": 3}
WORD_DTYPE = {0: np.uint16, 1: np.uint16, 2: np.uint8, 3: np.uint8}


def vf_code(vf) -> int:
    return VALUE_FORMATS[vf] if isinstance(vf, str) else int(vf)


def residual_bits(vf) -> int:
    """R = 1 + mantissa bits: BF16 8, FP16 11, FP8 E4M3 4, FP8 E5M2 3."""
    return int(_load().df11o_vf_residual_bits(vf_code(vf)))


def residual_array_bytes(N: int, vf) -> int:
    """PackedSignMantissa bytes (R25): R >= 8: a byte plane of roundup(N, 16) bytes + the (R - 8)-bit
    plane rounded to 16 bytes; R < 8: one R-bit plane rounded to 16 bytes; + 16 bytes of zero pad."""
    R = residual_bits(vf)
    if R >= 8:
        L = _roundup(N, 16)
        return L + _roundup((R - 8) * L // 8, 16) + 16
    return _roundup(R * _roundup(N, 16) // 8, 16) + 16


def split_v(w: np.ndarray, vf):
    """E1 for value format vf (R25): words -> (exponent symbols, R-bit residuals packed MSB-first)."""
    v = vf_code(vf)
    w = np.ascontiguousarray(w, dtype=WORD_DTYPE[v]).reshape(-1)
    exp = np.empty(w.size, np.uint8)
    res = np.zeros(residual_array_bytes(w.size, v), np.uint8)
    if w.size:
        _load().df11o_split_v(_ptr(w), w.size, v, _ptr(exp), _ptr(res))
    return exp, res


def compose_v(vf, exponent: int, residual: int) -> int:
    return int(_load().df11o_compose_v(vf_code(vf), exponent, residual))


# --------------------------------------------------------------------------- E1, E2
def split(w: np.ndarray):
    """E1: uint16 BF16 words -> (exponent bytes, packed sign/mantissa bytes)."""
    w = np.ascontiguousarray(w, dtype=np.uint16).reshape(-1)
    exp = np.empty(w.size, np.uint8)
    psm = np.empty(w.size, np.uint8)
    if w.size:
        _load().df11o_split(_ptr(w), w.size, _ptr(exp), _ptr(psm))
    return exp, psm


def compose(exponent: int, psm: int) -> int:
    return int(_load().df11o_compose(exponent, psm))


def histogram(exp: np.ndarray) -> np.ndarray:
    """E2."""
    hist = np.zeros(256, np.uint64)
    if exp.size:
        _load().df11o_histogram(_ptr(exp), exp.size, _ptr(hist))
    return hist


def entropy_bits(hist) -> float:
    """Eq. 2: H(X) = -sum p log2 p, with 0 log 0 := 0."""
    total = float(sum(int(h) for h in hist))
    h = 0.0
    for c in hist:
        c = int(c)
        if c:
            p = c / total
            h -= p * math.log2(p)
    return h


# --------------------------------------------------------------------------- full encoder
class FormatError(ValueError):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


def encode(w: np.ndarray, T: int = 256, n: int = 8, lut_mode: str = "auto", codebook_hist=None,
           vf="bf16", lut_bits=8) -> dict:
    """E1..E8 for one tensor.  Codebook scope (R5): the tensor's own histogram, or `codebook_hist`
    (e.g. the summed histogram of a group sharing "a Huffman tree based on the distribution of
    exponents in model weights"); it must give every exponent of `w` a code.
    vf: value format (R25; words are uint16 for bf16/fp16, uint8 for the fp8 formats).  lut_bits: b of
    the b-bit hierarchical tables (App. I.2; 8 = the paper), or "mono" for the monolithic table of
    App. I.1 (b = L, L <= 16; R28)."""
    v = vf_code(vf)
    w = np.ascontiguousarray(w, dtype=WORD_DTYPE[v]).reshape(-1)
    N = int(w.size)
    if N >= 1 << 32:
        raise FormatError("too_large", "N >= 2^32 (BlockOutputPos is uint32, P:387)")
    lib = _load()
    exp, psm = split_v(w, v)
    hist = histogram(exp)
    cb_hist = hist if codebook_hist is None else np.asarray(codebook_hist)
    lengths = huffman.code_lengths([int(h) for h in cb_hist])
    if any(int(hist[s]) and not lengths[s] for s in range(256)):
        raise FormatError("invalid_argument", "codebook_hist gives an exponent of w no code")
    codes = huffman.canonical_codes(lengths)
    L = max(lengths)
    if L > 8 * n:
        raise FormatError("invalid_argument", "max code length exceeds the 8n-bit chunk")
    if lut_bits == "mono":
        if L > 16:
            raise FormatError("invalid_argument", "monolithic LUT needs L <= 16")
        b = max(L, 1)
    else:
        b = int(lut_bits)
        if not 1 <= b <= 16:
            raise FormatError("invalid_argument", "lut_bits must be in [1, 16]")
    tables, _depth = huffman.hierarchical_luts(lengths, codes, b=b)
    narrow_ok = huffman.narrow_is_legal(lengths, tables)
    if lut_mode == "narrow":
        if any(lengths[s] for s in range(240, 256)):
            raise FormatError("reserved_exponent", "exponent >= 240 present (P:130)")
        if len(tables) - 1 > 16:
            raise FormatError("lut_overflow", "more than 16 child LUTs")
        wide = False
    elif lut_mode == "wide":
        wide = True
    elif lut_mode == "auto":
        wide = not narrow_ok
    else:
        raise ValueError(lut_mode)
    luts = np.frombuffer(huffman.serialize_luts(tables, wide), np.uint8).copy()

    code_len = np.array(lengths, np.uint8)
    code_arr = np.array(codes, np.uint32)
    encoded_bits = int(sum(int(hist[s]) * lengths[s] for s in range(256)))
    block_bits = 8 * T * n
    B = (encoded_bits + block_bits - 1) // block_bits
    stream = np.zeros(B * T * n + 16, np.uint8)
    if N:
        written = lib.df11o_pack_bits(_ptr(exp), N, _ptr(code_len), _ptr(code_arr), _ptr(stream))
        assert written == encoded_bits
    gap_values = np.zeros(max(B * T, 1), np.uint8)
    bop = np.zeros(B + 1, np.uint32)
    if N:
        rc = lib.df11o_gaps_bop(_ptr(exp), N, _ptr(code_len), T, n, B, _ptr(gap_values), _ptr(bop))
        if rc != 0:
            raise FormatError("invalid_argument", "gap does not fit in 5 bits")
    gaps = np.zeros(_roundup((5 * B * T + 7) // 8, 16) + 16, np.uint8)
    if B:
        lib.df11o_pack_gaps(_ptr(gap_values), B * T, _ptr(gaps))
    return dict(
        num_elements=N, encoded_bits=encoded_bits, T=T, n=n, B=B, k=len(tables),
        lut_entry_bytes=2 if wide else 1, max_code_len=L, value_format=v, lut_bits=b,
        code_lengths=code_len, luts=luts, encoded_exponent=stream,
        packed_sign_mantissa=psm, gaps=gaps, block_output_pos=bop,
        # oracle-side extras for tests
        histogram=hist, codes=code_arr, gap_values=gap_values[: B * T],
    )


def compressed_bytes(fmt: dict) -> int:
    """Bytes of the DF11 representation that the method must store/read (excluding alignment pad):
    encoded stream + sign/mantissa (R bits per element) + 5-bit gaps + 32-bit BlockOutputPos + LUTs +
    CodeLengths."""
    B, T = fmt["B"], fmt["T"]
    R = residual_bits(fmt.get("value_format", 0))
    return ((fmt["encoded_bits"] + 7) // 8 + (R * fmt["num_elements"] + 7) // 8 + (5 * B * T + 7) // 8
            + 4 * (B + 1) + len(fmt["luts"]) + 256)


# --------------------------------------------------------------------------- decoders
def _vf(fmt) -> int:
    return int(fmt.get("value_format", 0))


def decode_sequential(fmt: dict) -> np.ndarray:
    """D1: canonical bit-by-bit decode (CodeLengths + stream + PackedSignMantissa only)."""
    N = fmt["num_elements"]
    v = _vf(fmt)
    out = np.zeros(N, WORD_DTYPE[v])
    if N == 0:
        return out
    s = fmt["encoded_exponent"]
    psm = fmt["packed_sign_mantissa"]
    rc = _load().df11o_decode_sequential(_ptr(s), s.size, _ptr(fmt["code_lengths"]), _ptr(psm), psm.size, N, v,
                                         _ptr(out))
    if rc != 0:
        raise FormatError("corrupt", f"sequential decode failed ({rc})")
    return out


def decode_sequential_blocks(fmt: dict, b0: int, b1: int, out: np.ndarray) -> None:
    """D1 over format blocks [b0, b1): the sequential decoder started at block b0's first code (stream
    bit 8nT*b0 + Gaps[b0 T], element BlockOutputPos[b0]) for the blocks' elements, written
    into `out` (the whole tensor's array).  Lets a caller spread one tensor over threads."""
    if b1 <= b0:
        return
    T, n = int(fmt["T"]), int(fmt["n"])
    bop = fmt["block_output_pos"]
    first, last = int(bop[b0]), int(bop[b1])
    start = 8 * n * T * b0 + _read_gap(fmt["gaps"], b0 * T)
    s, psm = fmt["encoded_exponent"], fmt["packed_sign_mantissa"]
    rc = _load().df11o_decode_sequential_range(_ptr(s), s.size, _ptr(fmt["code_lengths"]), _ptr(psm), psm.size,
                                               int(fmt["num_elements"]), start, first, last - first, _vf(fmt),
                                               _ptr(out))
    if rc != 0:
        raise FormatError("corrupt", f"sequential decode failed ({rc})")


def decode_alg1(fmt: dict, check_counts: bool = True) -> np.ndarray:
    """D2: Algorithm 1 emulated block by block, thread by thread."""
    N = fmt["num_elements"]
    v = _vf(fmt)
    out = np.zeros(N, WORD_DTYPE[v])
    if N == 0:
        return out
    s, g, psm = fmt["encoded_exponent"], fmt["gaps"], fmt["packed_sign_mantissa"]
    rc = _load().df11o_decode_alg1(
        _ptr(fmt["luts"]), fmt["lut_entry_bytes"], fmt["k"], int(fmt.get("lut_bits", 8)), _ptr(fmt["code_lengths"]),
        _ptr(s), s.size, _ptr(g), g.size, _ptr(fmt["block_output_pos"]),
        _ptr(psm), psm.size, fmt["B"], fmt["T"], fmt["n"], N, v,
        1 if check_counts else 0, _ptr(out))
    if rc != 0:
        raise FormatError("corrupt", f"Alg. 1 emulation failed ({rc})")
    return out


def decode_alg1_range(fmt: dict, b0: int, b1: int, out: np.ndarray) -> None:
    """D2 over format blocks [b0, b1) only, writing their outputs into `out` (the whole tensor's uint16
    array): the same Alg. 1 emulation as decode_alg1, on views that start at block b0 (BlockOutputPos
    values are absolute, so outputs land at their final positions).  Lets a caller spread the blocks
    of one tensor over threads (ctypes releases the GIL); requires 5*T*b0 to be a whole number of
    bytes (true for T = 256)."""
    T, n = int(fmt["T"]), int(fmt["n"])
    if b1 <= b0:
        return
    if (5 * T * b0) % 8:
        raise ValueError("block range start must fall on a byte of the gap stream")
    s = fmt["encoded_exponent"][b0 * T * n:]
    g = fmt["gaps"][(5 * T * b0) // 8:]
    bop = np.ascontiguousarray(fmt["block_output_pos"][b0:b1 + 1])
    psm = fmt["packed_sign_mantissa"]
    rc = _load().df11o_decode_alg1(
        _ptr(fmt["luts"]), fmt["lut_entry_bytes"], fmt["k"], int(fmt.get("lut_bits", 8)), _ptr(fmt["code_lengths"]),
        _ptr(s), s.size, _ptr(g), g.size, _ptr(bop),
        _ptr(psm), psm.size, b1 - b0, T, n, fmt["num_elements"], _vf(fmt), 1, _ptr(out))
    if rc != 0:
        raise FormatError("corrupt", f"Alg. 1 emulation failed ({rc})")


def decode_alg1_blocks(fmt: dict, blocks) -> dict:
    """D2 restricted to the given format blocks: returns {block b: (start, decoded words)} for
    sampled parity checks at full size.  Runs Alg. 1 on a view containing only those blocks."""
    res = {}
    for b in blocks:
        b = int(b)
        T, n = fmt["T"], fmt["n"]
        lo, hi = int(fmt["block_output_pos"][b]), int(fmt["block_output_pos"][b + 1])
        cb = T * n
        stream = np.zeros(cb + 16, np.uint8)
        src = fmt["encoded_exponent"][b * cb: b * cb + cb + 16]
        stream[: src.size] = src
        gap_vals = [_read_gap(fmt["gaps"], b * T + t) for t in range(T)]
        gaps = np.zeros(_roundup((5 * T + 7) // 8, 16) + 16, np.uint8)
        gv = np.array(gap_vals, np.uint8)
        _load().df11o_pack_gaps(_ptr(gv), T, _ptr(gaps))
        bop = np.array([0, hi - lo], np.uint32)
        R = residual_bits(_vf(fmt))
        n_sub = hi - lo
        psm = np.zeros(residual_array_bytes(n_sub, _vf(fmt)), np.uint8)
        src = fmt["packed_sign_mantissa"]
        if R >= 8:                # byte plane slice, then the (R - 8)-bit plane re-aligned to bit 0
            psm[:n_sub] = src[lo:hi]
            if R > 8:
                Lfull, Lsub = _roundup(int(fmt["num_elements"]), 16), _roundup(n_sub, 16)
                bits = np.unpackbits(src[Lfull:])[(R - 8) * lo: (R - 8) * hi]
                packed = np.packbits(bits)
                psm[Lsub: Lsub + packed.size] = packed
        else:                     # the block's residual bits [R lo, R hi), re-aligned to bit 0
            bits = np.unpackbits(src)[R * lo: R * hi]
            packed = np.packbits(bits)
            psm[: packed.size] = packed
        sub = dict(fmt, num_elements=hi - lo, B=1, encoded_exponent=stream, gaps=gaps,
                   block_output_pos=bop, packed_sign_mantissa=psm)
        res[b] = (lo, decode_alg1(sub, check_counts=False))
    return res


def _read_gap(gaps: np.ndarray, g: int) -> int:
    v = 0
    for j in range(5):
        bit = 5 * g + j
        v = (v << 1) | ((int(gaps[bit >> 3]) >> (7 - (bit & 7))) & 1)
    return v
