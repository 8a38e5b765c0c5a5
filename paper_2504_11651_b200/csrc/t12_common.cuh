// t12_common.cuh — pieces of the product decode kernel shared with its A/B variants: the 12-bit
// multi-code decode table T12 (layout, lookup, CTA-wide build from the format's LUTs and CodeLengths),
// the slot packing of decoded exponents, the compaction and the BF16 compose.
#pragma once
#include "fast_helpers.cuh"

namespace df11 {
namespace {

constexpr uint32_t kR = 12;                 // root bits of T12
constexpr uint32_t kRows = 1u << kR;
constexpr uint32_t kCodes = 4;              // codes per entry
constexpr uint32_t kT12Bytes = (kRows + 16) * 8;   // entries at r + (r >> 8) < kRows + 15 (+ pad)
constexpr uint32_t kLutSmem = 8192;         // format LUT bytes staged in SMEM (larger: walked in global)
// Chain progress x = 2^16 - (chain length in bits) + consumed bits: x += hi adds the consumed bits in the
// low bits (the count sits in bits 27..31 and never reaches bit 16), so the chain is active while bit 16
// is clear.
constexpr uint32_t kXEnd = 1u << 16;
constexpr uint32_t kXMask = 2 * kXEnd - 1;

// T12 row r lives at entry r + (r >> 8): chains near their end look up rows whose low bits are the
// one-bit padding (see the kernels), which would otherwise all fall into one bank pair (measured 10.5
// wavefronts per LDS.64 in the decode loop); adding the row's top 4 bits spreads them.  The map is
// injective on [0, 4096) (block h of 256 rows moves to [257h, 257h + 256)); entries up to 4110.
__host__ __device__ __forceinline__ uint32_t t12_slot(uint32_t r) { return r + (r >> 8); }
__device__ __forceinline__ uint32_t t12_addr(uint32_t a, uint32_t base, uint32_t k_row, uint32_t k_top,
                                             uint32_t k_ent) {
    return madlo(madhi(a, k_top, mulhi(a, k_row)), k_ent, base);   // ((a >> 20) + (a >> 28)) * 8 + base
}
__device__ __forceinline__ uint32_t rot8(uint32_t e) { return ((e >> 1) | (e << 7)) & 0xFFu; }
__device__ __forceinline__ uint32_t unrot8(uint32_t r) { return ((r << 1) | (r >> 7)) & 0xFFu; }
// Symbol as stored in T12 / the slots: BF16 exponents rotated (the merge's bit-select trick); the other
// value formats' exponents pre-shifted to where the merge needs them inside their byte (FP16 and FP8
// E5M2: e << 2, FP8 E4M3: e << 3; still < 256 and distinct, so CodeLengths by stored symbol works).
template <uint32_t kVF>
__device__ __forceinline__ uint32_t to_stored(uint32_t e) {
    if constexpr (kVF == DF11_VF_BF16) return rot8(e);
    else if constexpr (kVF == DF11_VF_FP8_E4M3) return (e & 15u) << 3;
    else return (e & 31u) << 2;
}
template <uint32_t kVF>
__device__ __forceinline__ uint32_t from_stored(uint32_t r) {
    if constexpr (kVF == DF11_VF_BF16) return unrot8(r);
    else if constexpr (kVF == DF11_VF_FP8_E4M3) return (r >> 3) & 15u;
    else return (r >> 2) & 31u;
}

__device__ __forceinline__ void st8(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
template <int k>
__device__ __forceinline__ void st8k(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u8 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(k) : "memory");
}
__device__ __forceinline__ uint32_t ld8(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void lds64(uint32_t addr, uint32_t &lo, uint32_t &hi) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(addr));
}
// ld.shared.v2.u32 only if p (lo / hi keep their values otherwise)
__device__ __forceinline__ void lds64_if(uint32_t addr, uint32_t &lo, uint32_t &hi, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q ld.shared.v2.u32 {%0, %1}, [%2];\n\t}"
                 : "+r"(lo), "+r"(hi) : "r"(addr), "r"((uint32_t)p));
}
__device__ __forceinline__ void lds128(uint32_t addr, uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Output slot of one chain: decoded (rotated) exponents are appended to a lane-column slot (word k at
// wp0 + 128 k) through a pending word.  State: acc = the pending word (valid low bits only), tb = bits
// appended so far, wp = address of the pending word.
struct Slot {
    uint32_t acc, tb, wp;
};
__device__ __forceinline__ void slot_init(Slot &s, uint32_t wp0) {
    s.acc = 0;
    s.tb = 0;
    s.wp = wp0;
}
#ifndef DF11_PACK_ALU
// Append the n <= 4 bytes of lo (8n = hi >> 24).  The pending word is stored every time (later appends
// complete and rewrite it).  (sp:m0) = lo * 2^fb on the FMA pipe gives the appended bytes in place
// and the bytes that spill into the next word; crossing a word boundary flips bit 5 of tb.
__device__ __forceinline__ void pack(Slot &s, uint32_t lo, uint32_t hi, uint32_t k_s24) {
    uint64_t v;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(v) : "r"(lo), "r"(__funnelshift_l(0u, 1u, s.tb)));   // lo * 2^(tb mod 32)
    const uint32_t m = (uint32_t)v | s.acc, sp = (uint32_t)(v >> 32);
    sts32(s.wp, m);
    const uint32_t t2 = madhi(hi, k_s24, s.tb);            // tb + 8n
    const uint32_t f32 = (t2 ^ s.tb) & 32u;                // 32: the word is complete
    s.acc = __funnelshift_rc(m, sp, f32);                  // sp if complete, else m
    s.wp = madlo(f32, 4u, s.wp);                           // + 128 if complete
    s.tb = t2;
}
#else
// ALU form (round 1): shifts, OR and selects.
__device__ __forceinline__ void pack(Slot &s, uint32_t lo, uint32_t hi, uint32_t k_s24) {
    const uint32_t fb = s.tb & 31u;
    const uint32_t m = s.acc | (lo << fb);
    const uint32_t sp = __funnelshift_l(lo, 0u, fb);        // bytes that spill into the next word
    sts32(s.wp, m);
    const uint32_t t2 = madhi(hi, k_s24, s.tb);
    const bool full = ((t2 ^ s.tb) & 32u) != 0;
    s.wp = full ? s.wp + 128u : s.wp;
    s.acc = full ? sp : m;
    s.tb = t2;
}
#endif
// Bytes appended so far; the pending word is flushed by slot_flush.
__device__ __forceinline__ uint32_t slot_bytes(const Slot &s) { return s.tb >> 3; }
__device__ __forceinline__ void slot_flush(const Slot &s) { sts32(s.wp, s.acc); }

// 96-bit bit buffer shifts that pull in one-bits (the chain-end sentinel, see the kernel)
__device__ __forceinline__ void shift96_ones(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t s) {
    a = __funnelshift_l(b, a, s);
    b = __funnelshift_l(c, b, s);
    c = __funnelshift_l(0xFFFFFFFFu, c, s);
}
__device__ __forceinline__ void shift96_long_ones(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t s) {
    const bool w = s >= 32;
    a = w ? b : a;
    b = w ? c : b;
    c = w ? 0xFFFFFFFFu : c;
    shift96_ones(a, b, c, s);
}
__device__ __forceinline__ void sts32_if(uint32_t addr, uint32_t v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
                 ::"r"(addr), "r"(v), "r"((uint32_t)p) : "memory");
}

// Copy n (<= 32) bytes held in w[0..7] (little-endian byte stream) to SMEM byte address d.  Phase A:
// the whole words of the destination (the last may carry garbage past the end: the next chain's phase B
// rewrites those bytes).  Phase B (after a __syncwarp): the first, partial word.
__device__ __forceinline__ void compact_words(uint32_t d, const uint32_t (&w)[8], uint32_t n) {
    const uint32_t r = d & 3u, db = d - r, sh = r * 8u;
    const uint32_t nw = (r + n + 3u) >> 2;                 // <= 9
#pragma unroll
    for (int k = 0; k < 9; k++) {
        const uint32_t v = k == 0 ? w[0] : __funnelshift_l(w[k - 1], k < 8 ? w[k] : 0u, sh);
        sts32_if(db + 4u * k, v, (uint32_t)k < nw && (k > 0 || r == 0));
    }
}
// compact_words for runs of up to 64 bytes held in w[0..15] (one chain of a 16-byte chunk)
__device__ __forceinline__ void compact_words16(uint32_t d, const uint32_t (&w)[16], uint32_t n) {
    const uint32_t r = d & 3u, db = d - r, sh = r * 8u;
    const uint32_t nw = (r + n + 3u) >> 2;                 // <= 17
#pragma unroll
    for (int k = 0; k < 17; k++) {
        const uint32_t v = k == 0 ? w[0] : __funnelshift_l(w[k - 1], k < 16 ? w[k] : 0u, sh);
        sts32_if(db + 4u * k, v, (uint32_t)k < nw && (k > 0 || r == 0));
    }
}
// 160-bit buffer (a:b:c:d:e) shifts for one chain over a 16-byte chunk (n = 16), pulling in one-bits
__device__ __forceinline__ void shift160_ones(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d, uint32_t &e,
                                              uint32_t s) {
    a = __funnelshift_l(b, a, s);
    b = __funnelshift_l(c, b, s);
    c = __funnelshift_l(d, c, s);
    d = __funnelshift_l(e, d, s);
    e = __funnelshift_l(0xFFFFFFFFu, e, s);
}
__device__ __forceinline__ void shift160_long_ones(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d, uint32_t &e,
                                                   uint32_t s) {
    const bool w = s >= 32;
    a = w ? b : a;
    b = w ? c : b;
    c = w ? d : c;
    d = w ? e : d;
    e = w ? 0xFFFFFFFFu : e;
    shift160_ones(a, b, c, d, e, s);
}
__device__ __forceinline__ void compact_head(uint32_t d, uint32_t w0, uint32_t n) {
    const uint32_t r = d & 3u, db = d - r;
    if (r == 0) return;
    const uint32_t v0 = w0 << (r * 8u);
#pragma unroll
    for (uint32_t i = 1; i < 4; i++)
        if (i >= r && i < r + n) st8(db + i, v0 >> (8u * i));
}

// Four BF16 from 4 rotated exponents R and 4 sign/mantissa bytes S (byte planes):
// high byte = sign | (R & 0x7F), low byte = (R & 0x80) | mantissa; PRMT interleaves them.
__device__ __forceinline__ void compose4r(uint32_t R, uint32_t S, uint32_t &lo2, uint32_t &hi2) {
    const uint32_t H = bitsel<0x80808080u>(R, S);
    const uint32_t L = bitsel<0x7F7F7F7Fu>(R, S);
    lo2 = prmt(L, H, 0x5140u);
    hi2 = prmt(L, H, 0x7362u);
}
__device__ __forceinline__ uint16_t compose_r(uint32_t r, uint32_t psm) {
    return (uint16_t)(((psm & 0x80u) << 8) | ((r & 0x7Fu) << 8) | (r & 0x80u) | (psm & 0x7Fu));
}


// Build T12 for tensor ts (CTA-wide, kThreads threads; contains __syncthreads).  T12 entry of row r
// (the next 12 stream bits): lo = up to 4 complete codes' rotated exponents, hi = consumed bits |
// 8 * count << 24.  The format LUTs are staged at lut (if they fit kLutSmem) and
// CodeLengths at len / rlen (indexed by exponent / by rotated exponent; absent codes: 32 in rlen).
// fc: 8 KB of scratch for the first-code table.  Returns whether the all-ones row is an escape (some
// code is longer than 12 bits); `safe` = some code is 1 bit long.  Symbols are stored as
// to_stored<kVF>; b-bit tables (lut_bits != 8, kB8 = false) are walked row by row.
template <uint32_t kThreads, uint32_t kVF, bool kB8>
__device__ __forceinline__ bool build_t12(const df11_device_tensor &ts, uint8_t *sb, uint32_t sbase,
                                          uint32_t off_t, uint32_t off_lut, uint32_t off_len, uint32_t off_rlen,
                                          uint32_t off_fc, uint32_t tid, bool &safe, bool &lut_in_smem) {
    // the format tables are staged in SMEM when they fit (b = 8: the paper's byte tables, b a compile-time
    // constant; other b: b-bit tables, App. I.2, walked with a runtime b); otherwise walked in global
    const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k, lb = kB8 ? 8u : lut_bits_of(ts);
    const uint32_t lut_bytes = (kk << lb) * eb_bytes;
    lut_in_smem = lut_bytes <= kLutSmem;
    if (lut_in_smem) {
        // 16-byte loads (k * 2^b * entry bytes is a multiple of 16 for b >= 4), then the tail bytes
        const uint32_t n16 = (reinterpret_cast<uintptr_t>(ts.luts) & 15) == 0 ? lut_bytes / 16 : 0;
        for (uint32_t i = tid; i < n16; i += kThreads)
            reinterpret_cast<uint4 *>(sb + off_lut)[i] = __ldg(reinterpret_cast<const uint4 *>(ts.luts) + i);
        for (uint32_t i = 16 * n16 + tid; i < lut_bytes; i += kThreads) sb[off_lut + i] = __ldg(ts.luts + i);
    }
    uint32_t len_t = 0;
    if (tid < 256u) {
        len_t = __ldg(ts.code_lengths + tid);
        sb[off_len + tid] = (uint8_t)len_t;
        // CodeLengths by stored symbol; only exponent fields of the format are symbols (their stored
        // values are distinct: no two threads write one entry)
        if (kVF == DF11_VF_BF16 || tid < (kVF == DF11_VF_FP8_E4M3 ? 16u : 32u))
            sb[off_rlen + to_stored<kVF>(tid)] = (uint8_t)(len_t ? len_t : 32u);
    }
    // a 1-bit codeword allows 64 codes per chain: such tensors take the count + direct path
    safe = __syncthreads_or(len_t == 1) != 0;

    // first code of every kR-bit prefix (rotated exponent | length << 8; 0 = longer than kR bits); an
    // entry then chains up to kCodes of these: the code starting s bits into the row is the first
    // code of the zero-padded prefix row << s if it fits in kR - s bits
    uint16_t *fc = reinterpret_cast<uint16_t *>(sb + off_fc);
    // lookups at row << s hit indices with s zero low bits: XOR-swizzle the bank bits with bits 6..10
    // so that they spread over the banks instead of piling into one
    auto fci = [](uint32_t i) { return i ^ (((i >> 6) & 31u) << 1); };
    bool row_esc_last = false;
    if (kB8 && kRows == 4 * kThreads && lut_in_smem) {
        // 12-bit prefix r: its first 8 bits index the root LUT; a code of 9..12 bits is
        // resolved by the second-level LUT from the last 4 bits (zero-padded).  Four rows per thread,
        // unrolled for ILP; then up to 4 chained first-code lookups per row.
        const uint32_t thr = eb_bytes == 1 ? 240u : 256u;
        auto lut = [&](uint32_t idx) -> uint32_t {
            return eb_bytes == 1 ? (uint32_t)sb[off_lut + idx]
                                 : (uint32_t)reinterpret_cast<const uint16_t *>(sb + off_lut)[idx];
        };
        uint32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t r = tid + u * kThreads;
            uint32_t e = lut(r >> 4), ok = 1;
            if (e >= thr) {
                const uint32_t j = eb_bytes == 1 ? 256u - e : e - 256u;
                ok = j < kk;
                e = ok ? lut(j * 256u + ((r & 15u) << 4)) : 0u;
                ok = ok && e < thr;
            }
            const uint32_t len = ok ? (uint32_t)sb[off_len + (e & 0xFFu)] : 0u;
            v[u] = (len != 0 && len <= kR) ? (to_stored<kVF>(e & 0xFFu) | (len << 8)) : 0u;
            fc[fci(r)] = (uint16_t)v[u];
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t r = tid + u * kThreads;
            uint32_t w = v[u], st = 0, syms = 0, c2 = 0;
#pragma unroll
            for (int k2 = 0; k2 < (int)kCodes; k2++) {
                const uint32_t len = w >> 8;
                if (len == 0 || len > kR - st) break;
                syms |= (w & 0xFFu) << (8 * c2);
                st += len;
                c2++;
                if (st < kR) w = fc[fci((r << st) & (kRows - 1u))];
                else w = 0;
            }
            *reinterpret_cast<uint2 *>(sb + off_t + t12_slot(r) * 8u) = make_uint2(syms, st | (c2 << 27));
            if (r == kRows - 1) row_esc_last = c2 == 0;
        }
    } else {
        // b-bit tables other than b = 8, or tables too large for SMEM: one walk of the format LUTs per row
        for (uint32_t row = tid; row < kRows; row += kThreads) {
            uint32_t len;
            const uint32_t sym = lut_in_smem ? lut_walk_smem(row << (32 - kR), sbase + off_lut, sbase + off_len,
                                                             eb_bytes, kk, lb, len)
                                             : lut_walk_global<kB8>(row << (32 - kR), ts, len);
            fc[fci(row)] = len <= kR ? (uint16_t)(to_stored<kVF>(sym) | (len << 8)) : (uint16_t)0;
        }
        __syncthreads();
        for (uint32_t row = tid; row < kRows; row += kThreads) {
            uint32_t st = 0, syms = 0, c2 = 0;
            while (st < kR && c2 < kCodes) {
                const uint32_t v = fc[fci((row << st) & (kRows - 1u))], len = v >> 8;
                if (len == 0 || len > kR - st) break;
                st += len;
                syms |= (v & 0xFFu) << (8 * c2);
                c2++;
            }
            *reinterpret_cast<uint2 *>(sb + off_t + t12_slot(row) * 8u) = make_uint2(syms, st | (c2 << 27));
            if (row == kRows - 1) row_esc_last = c2 == 0;
        }
    }
    // if kR one-bits hold no complete code (true for canonical codes longer than kR bits), one-bits
    // after a chain's last bit stall it exactly there
    return __syncthreads_or(row_esc_last) != 0;
}

}  // namespace
}  // namespace df11
