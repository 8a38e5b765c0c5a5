// fast_helpers.cuh — device helpers shared by the persistent sm_100a decode kernels (decode_fast.cu,
// decode_sp.cu): format-tile constants, FMA-pipe integer helpers, the 96-bit bit buffer, TMA bulk
// copies on mbarriers, the paper's hierarchical LUT walk and the BF16 compose.
#pragma once
#include "decode_common.cuh"

namespace df11 {
namespace {

constexpr uint32_t kT = 256;               // format threads per block
constexpr uint32_t kN = 8;                 // bytes per format thread
constexpr uint32_t kCpl = 2;               // chunks per lane
constexpr uint32_t kLanes = kT / kCpl;     // 128 threads per group (one tile)
constexpr uint32_t kChunkBytes = kT * kN + 16;   // a tile's EncodedExponent + spill
constexpr uint32_t kGapBytes = kT * 5 / 8 + 16;  // a tile's 5-bit gaps (+ 1 byte read past)
constexpr uint32_t kStageBytes = kChunkBytes + kGapBytes;

extern __shared__ __align__(16) uint32_t smem_w[];

__device__ __forceinline__ uint8_t *smem_b() { return reinterpret_cast<uint8_t *>(smem_w); }
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// FMA-pipe integer helpers.  The B200 ALU pipe (SHF/LOP3/PRMT/SEL/ISETP) issues a warp instruction
// every 2 cycles per SMSP, as does the FMA pipe (IMAD*): bit-field extraction is moved onto the FMA
// pipe with multiplies by powers of two that the compiler cannot strength-reduce (runtime operands).
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t madlo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
// st.shared.u8 [addr + k] = v, predicated on pos < lim (no branch).
template <int k>
__device__ __forceinline__ void sts8_if(uint32_t addr, uint32_t v, uint32_t pos, uint32_t lim) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %2, %3;\n\t@p st.shared.u8 [%0+%4], %1;\n\t}"
                 ::"r"(addr), "r"(v), "r"(pos), "r"(lim), "n"(k) : "memory");
}

// 96-bit MSB-first bit buffer (a:b:c) shifted left by `s` (only the low 5 bits of s are used).
__device__ __forceinline__ void shift96(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t s) {
    a = __funnelshift_l(b, a, s);
    b = __funnelshift_l(c, b, s);
    c = __funnelshift_l(0u, c, s);
}
// Shift by 0..63 bits (escape path).
__device__ __forceinline__ void shift96_long(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t s) {
    const bool w = s >= 32;                                   // select, then funnel by s & 31
    a = w ? b : a;
    b = w ? c : b;
    c = w ? 0u : c;
    shift96(a, b, c, s);
}
// PTX shifts clamp the shift amount: any amount >= 32 (incl. "negative" unsigned) yields 0.
__device__ __forceinline__ uint32_t shl_c(uint32_t x, uint32_t n) {
    uint32_t d;
    asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(n));
    return d;
}
__device__ __forceinline__ uint32_t shr_c(uint32_t x, uint32_t n) {
    uint32_t d;
    asm("shr.b32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(n));
    return d;
}
// OR word w into the buffer at bit position v (0 = top, v < 96); bits below the valid region are
// zero.  Branch-free: every out-of-range term shifts by >= 32 and vanishes.
__device__ __forceinline__ void insert96(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t v, uint32_t w) {
    a |= shr_c(w, v);
    b |= shl_c(w, 32u - v) | shr_c(w, v - 32u);
    c |= shl_c(w, 64u - v) | shr_c(w, v - 64u);
}

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\tLAB_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra LAB_WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// Prefetch [src, src + bytes) into L2 (one TMA instruction, no registers, no SMEM).
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Stage format block b of tensor ts (EncodedExponent chunk + spill, and its gaps) into `stage`.
__device__ __forceinline__ void issue_tile(const df11_device_tensor &ts, uint32_t b, uint32_t stage, uint32_t bar) {
    mbar_expect_tx(bar, kChunkBytes + kGapBytes);
    tma_g2s(stage, ts.encoded_exponent + (size_t)b * (kT * kN), kChunkBytes, bar);
    tma_g2s(stage + kChunkBytes, ts.gaps + (size_t)b * (kT * 5 / 8), kGapBytes, bar);
}
// The same for the format T = 128, n = 16 (a format block of the same 2 048 stream bytes, half the
// gaps: 80 bytes, + 16 read past).
__device__ __forceinline__ void issue_tile16(const df11_device_tensor &ts, uint32_t b, uint32_t stage, uint32_t bar) {
    mbar_expect_tx(bar, kChunkBytes + 128 * 5 / 8 + 16);
    tma_g2s(stage, ts.encoded_exponent + (size_t)b * (kT * kN), kChunkBytes, bar);
    tma_g2s(stage + kChunkBytes, ts.gaps + (size_t)b * (128 * 5 / 8), 128 * 5 / 8 + 16, bar);
}

// Level i (0-based) of a b-bit LUT walk reads window bits [b*i, b*(i+1)), zero-extended past bit 32
// (R28: a symbol's entries cover every value of the bits after its code); b = 8 reads byte i.
__device__ __forceinline__ uint32_t lut_level_idx(uint32_t w, uint32_t lb, uint32_t i) {
    return shr_c(shl_c(w, lb * i), 32u - lb);          // PTX shifts by >= 32 give 0
}

// Paper's hierarchical LUT walk over the format's b-bit tables in global memory; returns
// the exponent and its code length.  Bounded: <= ceil(32/b) levels, child < k, zero length -> 32.
// kB8: the paper's byte tables (b = 8, a compile-time constant: fewer registers at the call sites of
// the product kernel); otherwise b = ts.lut_bits.
template <bool kB8>
__device__ __noinline__ uint32_t lut_walk_global(uint32_t w, const df11_device_tensor &ts, uint32_t &len) {
    const uint8_t *__restrict__ luts = ts.luts;
    const uint32_t eb = ts.lut_entry_bytes, thr = eb == 1 ? 240u : 256u;
    const uint32_t lb = kB8 ? 8u : lut_bits_of(ts), levels = kB8 ? 4u : (32u + lb - 1u) / lb;
    uint32_t table = 0, e = 0;
#pragma unroll 1
    for (uint32_t i = 0; i < levels; i++) {
        const uint32_t off = (table << lb) + lut_level_idx(w, lb, i);
        e = eb == 1 ? (uint32_t)__ldg(luts + off)
                    : ((uint32_t)__ldg(luts + 2 * off) | ((uint32_t)__ldg(luts + 2 * off + 1) << 8));
        if (e < thr) break;
        table = eb == 1 ? 256u - e : e - 256u;
        if (table >= ts.k || i == levels - 1) { e = 0; break; }
    }
    e &= 0xFFu;
    len = __ldg(ts.code_lengths + e);
    if (len == 0) len = 32;
    return e;
}

// The same walk over the SMEM copy of the format tables (narrow or wide).
__device__ __forceinline__ uint32_t lut_walk_smem(uint32_t w, uint32_t lut, uint32_t clen, uint32_t eb,
                                                  uint32_t k, uint32_t lb, uint32_t &len) {
    const uint32_t thr = eb == 1 ? 240u : 256u, levels = (32u + lb - 1u) / lb;
    uint32_t e = 0, table = 0;
#pragma unroll 1
    for (uint32_t i = 0; i < levels; i++) {
        const uint32_t idx = (table << lb) + lut_level_idx(w, lb, i);
        if (eb == 1) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(e) : "r"(lut + idx));
        else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(e) : "r"(lut + 2 * idx));
        if (e < thr) break;
        table = eb == 1 ? 256u - e : e - 256u;
        if (table >= k || i == levels - 1) { e = 0; break; }
    }
    e &= 0xFFu;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(len) : "r"(clen + e));
    if (len == 0) len = 32;
    return e;
}

__device__ __forceinline__ void group_bar(uint32_t g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kLanes) : "memory");
}

// Two BF16 from 2 exponents (bytes 0,1 of E) and 2 sign/mantissa bytes (bytes 0,1 of S) — or bytes
// 2,3 with hi = true: W = [S0, sign(S0)x8, S1, sign(S1)x8] (PRMT sign replicate), X = [E0,0,E1,0];
// result = (W & 0x807F807F) + (X << 7)  =  (sign << 15) | (E << 7) | mantissa per half.
template <bool hi>
__device__ __forceinline__ uint32_t compose2(uint32_t E, uint32_t S) {
    const uint32_t W = prmt(S, 0u, hi ? 0xB3A2u : 0x9180u);
    const uint32_t X = prmt(E, 0u, hi ? 0x4342u : 0x4140u);
    return (W & 0x807F807Fu) + (X << 7);
}

// Four BF16 from 4 exponents E and 4 sign/mantissa bytes S, as byte planes: the high byte of each
// BF16 is sign | E >> 1, the low byte (E & 1) << 7 | mantissa; PRMT interleaves them.
// Phase-1 update "if ((acc & M) == 0) { acc += e; e1 = e; }" as one predicate-setting LOP3 and two
// predicated instructions.
template <uint32_t M>
__device__ __forceinline__ void p1_apply(uint32_t &acc, uint32_t &e1, uint32_t e) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %0, %3;\n\tsetp.eq.u32 p, t, 0;\n\t"
        "@p add.u32 %0, %0, %2;\n\t@p mov.b32 %1, %2;\n\t}"
        : "+r"(acc), "+r"(e1) : "r"(e), "n"(M));
}
// (m ? c : a) bitwise, one LOP3 (truth table 0xB8 for a=0xF0, b=0xCC, c=0xAA)
template <uint32_t m>
__device__ __forceinline__ uint32_t bitsel(uint32_t a, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(d) : "r"(a), "n"(m), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t mullo(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
// E >> 1 and E << 7 as IMAD.HI / IMAD by constant-bank multipliers k_half = 2^31, k_128 = 2^7 (FMA
// pipe), the byte-plane selects as one LOP3 each and the interleave as two PRMT (ALU pipe).
__device__ __forceinline__ void compose4(uint32_t E, uint32_t S, uint32_t &lo2, uint32_t &hi2, uint32_t k_half,
                                         uint32_t k_128) {
#ifdef DF11_OLD_COMPOSE
    const uint32_t H = (S & 0x80808080u) | ((E >> 1) & 0x7F7F7F7Fu);
    const uint32_t L = ((E << 7) & 0x80808080u) | (S & 0x7F7F7F7Fu);
#else
    const uint32_t H = bitsel<0x80808080u>(mulhi(E, k_half), S);
    const uint32_t L = bitsel<0x7F7F7F7Fu>(mullo(E, k_128), S);
#endif
    lo2 = prmt(L, H, 0x5140u);
    hi2 = prmt(L, H, 0x7362u);
}


}  // namespace
}  // namespace df11
