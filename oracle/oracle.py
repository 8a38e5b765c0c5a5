"""DF11 CPU oracle — orchestration of E1..E9 and the decoders D1/D2 over numpy arrays.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this module.  It shares no code with paper_2504_11651_b200/ and
neither imports the other.

The bulk loops live in plain C (df11_oracle.c, compiled to liboracle.so by build_oracle()); the
per-codebook steps live in huffman.py.  Citations "P:n" = PAPER.md line n; R-numbers = DESIGN.md §3.

Format produced ("DF11 format"):
    num_elements N, encoded_bits, T, n, B, k, lut_entry_bytes (1 narrow | 2 wide), max_code_len
    code_lengths          uint8[256]
    luts                  uint8[k*256*lut_entry_bytes]
    encoded_exponent      uint8[B*T*n + 16], MSB-first stream
    packed_sign_mantissa  uint8[roundup(N,16) + 16]
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
        lib.df11o_histogram.argtypes = [P, U64, P]
        lib.df11o_pack_bits.argtypes = [P, U64, P, P, P]
        lib.df11o_pack_bits.restype = U64
        lib.df11o_gaps_bop.argtypes = [P, U64, P, U32, U32, U32, P, P]
        lib.df11o_gaps_bop.restype = I
        lib.df11o_pack_gaps.argtypes = [P, U64, P]
        lib.df11o_decode_sequential.argtypes = [P, U64, P, P, U64, P]
        lib.df11o_decode_sequential.restype = I
        lib.df11o_decode_alg1.argtypes = [P, U32, U32, P, P, U64, P, U64, P, P, U32, U32, U32, U64, I, P]
        lib.df11o_decode_alg1.restype = I
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _roundup(x: int, m: int) -> int:
    return (x + m - 1) // m * m


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


def encode(w: np.ndarray, T: int = 256, n: int = 8, lut_mode: str = "auto", codebook_hist=None) -> dict:
    """E1..E8 for one tensor.  Codebook scope (R5): the tensor's own histogram, or `codebook_hist`
    (e.g. the summed histogram of a group sharing "a Huffman tree based on the distribution of
    exponents in model weights"); it must give every exponent of `w` a code."""
    w = np.ascontiguousarray(w, dtype=np.uint16).reshape(-1)
    N = int(w.size)
    if N >= 1 << 32:
        raise FormatError("too_large", "N >= 2^32 (BlockOutputPos is uint32, P:387)")
    lib = _load()
    exp, psm = split(w)
    hist = histogram(exp)
    cb_hist = hist if codebook_hist is None else np.asarray(codebook_hist)
    lengths = huffman.code_lengths([int(h) for h in cb_hist])
    if any(int(hist[s]) and not lengths[s] for s in range(256)):
        raise FormatError("invalid_argument", "codebook_hist gives an exponent of w no code")
    codes = huffman.canonical_codes(lengths)
    L = max(lengths)
    if L > 8 * n:
        raise FormatError("invalid_argument", "max code length exceeds the 8n-bit chunk")
    tables, _depth = huffman.hierarchical_luts(lengths, codes, b=8)
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
    psm_padded = np.zeros(_roundup(N, 16) + 16, np.uint8)
    psm_padded[:N] = psm
    return dict(
        num_elements=N, encoded_bits=encoded_bits, T=T, n=n, B=B, k=len(tables),
        lut_entry_bytes=2 if wide else 1, max_code_len=L,
        code_lengths=code_len, luts=luts, encoded_exponent=stream,
        packed_sign_mantissa=psm_padded, gaps=gaps, block_output_pos=bop,
        # oracle-side extras for tests
        histogram=hist, codes=code_arr, gap_values=gap_values[: B * T],
    )


def compressed_bytes(fmt: dict) -> int:
    """Bytes of the DF11 representation that the method must store/read (excluding alignment pad):
    encoded stream + sign/mantissa + 5-bit gaps + 32-bit BlockOutputPos + LUTs + CodeLengths."""
    B, T = fmt["B"], fmt["T"]
    return ((fmt["encoded_bits"] + 7) // 8 + fmt["num_elements"] + (5 * B * T + 7) // 8
            + 4 * (B + 1) + len(fmt["luts"]) + 256)


# --------------------------------------------------------------------------- decoders
def decode_sequential(fmt: dict) -> np.ndarray:
    """D1: canonical bit-by-bit decode (CodeLengths + stream + PackedSignMantissa only)."""
    N = fmt["num_elements"]
    out = np.zeros(N, np.uint16)
    if N == 0:
        return out
    s = fmt["encoded_exponent"]
    rc = _load().df11o_decode_sequential(_ptr(s), s.size, _ptr(fmt["code_lengths"]),
                                         _ptr(fmt["packed_sign_mantissa"]), N, _ptr(out))
    if rc != 0:
        raise FormatError("corrupt", f"sequential decode failed ({rc})")
    return out


def decode_alg1(fmt: dict, check_counts: bool = True) -> np.ndarray:
    """D2: Algorithm 1 emulated block by block, thread by thread."""
    N = fmt["num_elements"]
    out = np.zeros(N, np.uint16)
    if N == 0:
        return out
    s, g = fmt["encoded_exponent"], fmt["gaps"]
    rc = _load().df11o_decode_alg1(
        _ptr(fmt["luts"]), fmt["lut_entry_bytes"], fmt["k"], _ptr(fmt["code_lengths"]),
        _ptr(s), s.size, _ptr(g), g.size, _ptr(fmt["block_output_pos"]),
        _ptr(fmt["packed_sign_mantissa"]), fmt["B"], fmt["T"], fmt["n"], N,
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
    rc = _load().df11o_decode_alg1(
        _ptr(fmt["luts"]), fmt["lut_entry_bytes"], fmt["k"], _ptr(fmt["code_lengths"]),
        _ptr(s), s.size, _ptr(g), g.size, _ptr(bop),
        _ptr(fmt["packed_sign_mantissa"]), b1 - b0, T, n, fmt["num_elements"], 1, _ptr(out))
    if rc != 0:
        raise FormatError("corrupt", f"Alg. 1 emulation failed ({rc})")


def decode_alg1_blocks(fmt: dict, blocks) -> dict:
    """D2 restricted to the given format blocks: returns {block b: (start, uint16 values)} for
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
        psm = np.zeros(_roundup(hi - lo, 16) + 16, np.uint8)
        psm[: hi - lo] = fmt["packed_sign_mantissa"][lo:hi]
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
