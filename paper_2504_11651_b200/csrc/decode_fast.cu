// decode_fast.cu — persistent sm_100a DF11 decode kernel (format T = 256, n = 8; narrow or wide LUTs).
//
// Same result as Algorithm 1 — every thread decodes the codewords that start in its
// 8-byte chunk, a block-level exclusive scan turns per-thread counts into output positions
// (P:148-150), phase 2 re-decodes into an SRAM buffer and BF16 leaves with coalesced stores —
// re-designed for B200:
//
//  * Persistent CTAs, one per SM, 4 groups of 256 threads; group g of CTA c walks the format blocks
//    ("tiles") of a contiguous range.  Each group owns a 16 KB exponent buffer and its own named
//    barrier (one per tile), so groups drift apart and hide each other's latency.
//  * Derived decode tables are built in SMEM once per (CTA, tensor) from the format's hierarchical
//    LUTs.  For every R-bit prefix (R = 9):
//      T1 = consumed | count << 8 | startmask << 23        (phase 1; every complete code in R bits)
//      T2 = s0 | s1 << 8 | s2 << 16 | consumed << 24 | count << 29   (phase 2; up to 3 exponents)
//    T1/T2 are replicated 32x with lane-private banks (word = prefix*32 + lane): conflict-free LDS.
//    A prefix whose first code is longer than R bits (~0.1 % of codes on LLM-like weights) is an
//    "escape" row: its entry advances nothing, the thread stalls on it and a warp-uniform check every
//    4 steps resolves it through a second-level table (next 9 bits -> symbol, length) built for up to
//    8 escape rows, or, for longer codes, through the paper's LUT walk.
//  * Phase 1 keeps (bit offset | count << 8) in ONE register and adds the T1 entry to it.
//  * The decode window is the top word of a 96-bit bit buffer shifted by the consumed bits; field
//    extraction uses IMAD.HI so the ALU and FMA pipes are equally loaded.
//  * The thread's 8-byte chunk + 4 spill bytes live in 3 registers; the decode window is a funnel
//    shift, so EncodedExponent is read from HBM exactly once.
//  * One barrier per tile: the scan.  Each warp then merges its own contiguous output range (its 32
//    threads' outputs are adjacent): 16 elements per lane-step, LDS.128 exponents + LDG.128
//    sign/mantissa (prefetched before phase 2) -> PRMT sign-replicate compose -> 2x 128-bit stores.
#include "decode_common.cuh"

namespace df11 {
namespace {

constexpr int kT = 256;                    // format threads per block == group size
constexpr int kN = 8;                      // bytes per thread
constexpr int kGroups = 4;
constexpr int kCta = kT * kGroups;         // 1024 threads
constexpr int kR = 9;                      // root bits of the derived tables
constexpr uint32_t kRows = 1u << kR;
constexpr uint32_t kTabWords = kRows * 32; // 32 lane replicas
constexpr uint32_t kExpBuf = 8 * kN * kT + 64;

// SMEM layout (bytes)
constexpr uint32_t kOffT1 = 0;
constexpr uint32_t kOffT2 = kOffT1 + kTabWords * 4;
constexpr uint32_t kEscRows = 8;                              // escape rows with a second-level table
constexpr uint32_t kR2 = 9;                                   // bits resolved by the second level
constexpr uint32_t kOffL2 = kOffT2 + kTabWords * 4;           // uint16 [kEscRows][1 << kR2]: sym | len << 8
constexpr uint32_t kLutSmem = 8192;                           // format LUTs copied when they fit
constexpr uint32_t kOffLut = kOffL2 + kEscRows * (1u << kR2) * 2;   // uint8/uint16 [k][256]
constexpr uint32_t kOffLen = kOffLut + kLutSmem;              // CodeLengths[256]
constexpr uint32_t kOffWsum = kOffLen + 256;                  // [groups][2 parities][8] uint32
constexpr uint32_t kOffExp = kOffWsum + kGroups * 2 * 8 * 4;  // [groups][kExpBuf]
constexpr uint32_t kChunkBytes = kT * kN + 16;                // a tile's EncodedExponent + spill
constexpr uint32_t kGapBytes = kT * 5 / 8 + 16;               // a tile's 5-bit gaps (+ 1 byte read past)
constexpr uint32_t kStageBytes = kChunkBytes + kGapBytes;     // one TMA stage
constexpr uint32_t kOffStage = kOffExp + kGroups * kExpBuf;   // [groups][2][kStageBytes]
constexpr uint32_t kOffMbar = kOffStage + kGroups * 2 * kStageBytes;   // [groups][2] uint64
constexpr uint32_t kSmemBytes = kOffMbar + kGroups * 2 * 8;
static_assert(kStageBytes % 16 == 0 && kOffStage % 16 == 0 && kOffMbar % 8 == 0, "TMA alignment");
static_assert(kSmemBytes <= 232448, "SMEM budget");
static_assert(kOffExp % 16 == 0 && kExpBuf % 16 == 0, "alignment");

extern __shared__ __align__(16) uint32_t smem_w[];

__device__ __forceinline__ uint8_t *smem_b() { return reinterpret_cast<uint8_t *>(smem_w); }

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// Paper's hierarchical LUT walk over the format tables in global memory; returns the
// exponent and its code length.  Bounded: <= 4 levels, child < k, zero length -> 32.
__device__ __noinline__ uint32_t lut_walk(uint32_t w, const df11_device_tensor &ts, uint32_t &len) {
    const uint8_t *__restrict__ luts = ts.luts;
    const uint32_t eb = ts.lut_entry_bytes, thr = eb == 1 ? 240u : 256u;
    uint32_t table = 0, e = 0;
#pragma unroll 1
    for (int i = 0; i < 4; i++) {
        const uint32_t off = table * 256u + ((w >> (24 - 8 * i)) & 0xFFu);
        e = eb == 1 ? (uint32_t)__ldg(luts + off)
                    : ((uint32_t)__ldg(luts + 2 * off) | ((uint32_t)__ldg(luts + 2 * off + 1) << 8));
        if (e < thr) break;
        table = eb == 1 ? 256u - e : e - 256u;
        if (table >= ts.k || i == 3) { e = 0; break; }
    }
    e &= 0xFFu;
    len = __ldg(ts.code_lengths + e);
    if (len == 0) len = 32;
    return e;
}

// Same walk over the SMEM copy of the format tables (used when k*256*entry_bytes <= kLutSmem).
__device__ __forceinline__ uint32_t lut_walk_smem(uint32_t w, const uint8_t *lut, const uint8_t *clen,
                                                  uint32_t eb, uint32_t k, uint32_t &len) {
    const uint32_t thr = eb == 1 ? 240u : 256u;
    uint32_t e = eb == 1 ? lut[w >> 24] : reinterpret_cast<const uint16_t *>(lut)[w >> 24];
#pragma unroll 1
    for (int sh = 16; e >= thr; sh -= 8) {
        const uint32_t table = eb == 1 ? 256u - e : e - 256u;
        if (table >= k || sh < 0) { e = 0; break; }
        const uint32_t idx = table * 256u + ((w >> sh) & 0xFFu);
        e = eb == 1 ? lut[idx] : reinterpret_cast<const uint16_t *>(lut)[idx];
    }
    e &= 0xFFu;
    len = clen[e];
    if (len == 0) len = 32;
    return e;
}

__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kT) : "memory");
}

// 32-bit MSB-first window at bit `off` (0 <= off < 64) of the 96-bit chunk (w0:w1:w2).  Only bits
// 0..5 of `off` are used, so callers may pass a packed counter.
__device__ __forceinline__ uint32_t window(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t off) {
    const bool lo = (off & 32u) == 0;
    return __funnelshift_l(lo ? w1 : w2, lo ? w0 : w1, off);
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

// FMA-pipe integer helpers.  The B200 ALU pipe (SHF/LOP3/PRMT/SEL/ISETP) issues a warp instruction
// every 2 cycles per SMSP, as does the FMA pipe (IMAD*): bit-field extraction is moved onto the FMA
// pipe with multiplies by powers of two that the compiler cannot strength-reduce (runtime operands).
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {     // (a * b) >> 32
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c) {   // ((a*b) >> 32) + c
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t madlo(uint32_t a, uint32_t b, uint32_t c) {   // a*b + c
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
// 96-bit MSB-first bit buffer (a:b:c) shifted left by `s` (0..31; only the low 5 bits are used).
__device__ __forceinline__ void shift96(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t s) {
    a = __funnelshift_l(b, a, s);
    b = __funnelshift_l(c, b, s);
    c = __funnelshift_l(0u, c, s);
}

// Row `w >> (32-R)` of a lane-private replicated table: address = lane_base + row * 128.
__device__ __forceinline__ uint32_t lds_row(uint32_t lane_base, uint32_t w) {
    uint32_t v;
    asm volatile("{\n\t.reg .u32 t;\n\tshr.u32 t, %1, %3;\n\tmad.lo.u32 t, t, 128, %2;\n\tld.shared.u32 %0, [t];\n\t}"
                 : "=r"(v) : "r"(w), "r"(lane_base), "n"(32 - kR));
    return v;
}

// st.shared.u8 [addr + k] = v, predicated on pos < lim (no branch).
template <int k>
__device__ __forceinline__ void sts8_if(uint32_t addr, uint32_t v, uint32_t pos, uint32_t lim) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %2, %3;\n\t@p st.shared.u8 [%0+%4], %1;\n\t}"
                 ::"r"(addr), "r"(v), "r"(pos), "r"(lim), "n"(k) : "memory");
}

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
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
// Stage format block b of tensor ts (its EncodedExponent chunk + spill, and its gaps) into `stage`.
__device__ __forceinline__ void issue_tile(const df11_device_tensor &ts, uint32_t b, uint32_t stage, uint32_t bar) {
    mbar_expect_tx(bar, kChunkBytes + kGapBytes);
    tma_g2s(stage, ts.encoded_exponent + (size_t)b * (kT * kN), kChunkBytes, bar);
    tma_g2s(stage + kChunkBytes, ts.gaps + (size_t)b * (kT * 5 / 8), kGapBytes, bar);
}

__global__ void __launch_bounds__(kCta, 1) fast_kernel(const __grid_constant__ Batch bt) {
    const uint32_t tid = threadIdx.x;
    const int g = (int)(tid / kT);
    const uint32_t t = tid % kT;
    const uint32_t lane = tid & 31, wig = t >> 5;
    const uint32_t FULL = 0xFFFFFFFFu;
    const uint32_t one = blockDim.x >> 10;                       // == 1, opaque to the compiler
    const uint32_t K_ROW = one << kR, K_128 = one << 7, K_S24 = one << 8, K_S8 = one << 24,
                   K_S16 = one << 16, K_S29 = one << 3;
    uint8_t *sb = smem_b();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_w);
    // lane-private table addresses: row r of table X is at X + r*128 + lane*4
    const uint32_t t1_lane = sbase + kOffT1 + lane * 4u;
    const uint32_t t2_lane = sbase + kOffT2 + lane * 4u;
    const uint32_t ebuf_off = kOffExp + (uint32_t)g * kExpBuf;             // byte offset into smem
    uint32_t *wsum = smem_w + kOffWsum / 4 + (uint32_t)g * 16;            // [2][8]

    const uint32_t total = bt.total_tiles;
    const uint32_t c_begin = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t c_end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    if (c_begin >= c_end) return;

    const uint32_t stage0 = sbase + kOffStage + (uint32_t)g * 2 * kStageBytes;
    const uint32_t mbar0 = sbase + kOffMbar + (uint32_t)g * 16;
    if (t == 0) {
        mbar_init(mbar0, 1);
        mbar_init(mbar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t q = 0;                    // tiles consumed by this group so far (stage = q & 1)

    uint32_t parity = 0;
    int ti_idx = tensor_of_tile(bt, c_begin);
    for (uint32_t seg_begin = c_begin; seg_begin < c_end; ti_idx++) {
        const df11_device_tensor &ts = bt.t[ti_idx];
        const uint32_t seg_end = min(c_end, bt.tile_start[ti_idx + 1]);
        const uint32_t base_tile = bt.tile_start[ti_idx];
        if (seg_end <= seg_begin) continue;

        // ---- derived tables for this tensor (CTA-wide)
        __syncthreads();
        const uint32_t lut_bytes = ts.k * 256u * ts.lut_entry_bytes;
        const bool lut_in_smem = lut_bytes <= kLutSmem;
        if (lut_in_smem)
            for (uint32_t i = tid; i < lut_bytes; i += kCta) sb[kOffLut + i] = __ldg(ts.luts + i);
        for (uint32_t i = tid; i < 256u; i += kCta) sb[kOffLen + i] = __ldg(ts.code_lengths + i);
        uint32_t *esc_mask = smem_w + kOffExp / 4;                 // scratch: the exponent buffers are idle
        uint32_t *esc_row = esc_mask + kRows / 32;
        if (tid < kRows / 32) esc_mask[tid] = 0;
        __syncthreads();
        const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k;
        const bool narrow_smem = lut_in_smem && eb_bytes == 1;
        // the paper's LUT walk for one code at the top of window w
        auto walk = [&](uint32_t w, uint32_t &len) -> uint32_t {
            if (narrow_smem) {                                  // root, then child tables via 256 - v
                const uint32_t lb = sbase + kOffLut;
                uint32_t e, sh = 24, table = 0;
#pragma unroll 1
                for (int i = 0; i < 4; i++, sh -= 8) {
                    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(e) : "r"(lb + table * 256u + ((w >> sh) & 0xFFu)));
                    if (e < 240u) break;
                    table = 256u - e;
                    if (table >= kk || i == 3) { e = 0; break; }
                }
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(len) : "r"(sbase + kOffLen + e));
                if (len == 0) len = 32;
                return e;
            }
            if (lut_in_smem) return lut_walk_smem(w, sb + kOffLut, sb + kOffLen, eb_bytes, kk, len);
            return lut_walk(w, ts, len);
        };
        uint32_t row_e1 = 0, row_e2 = 0;
        bool row_esc = false;
        if (tid < kRows) {
            const uint32_t idx = tid, W = idx << (32 - kR);
            uint32_t s = 0, cnt = 0, mask = 0, cons = 0, syms = 0, c2 = 0, cons2 = 0;
            while (s < (uint32_t)kR) {
                uint32_t len;
                const uint32_t sym = walk(W << s, len);
                if (len > (uint32_t)kR - s) break;
                mask |= 1u << s;
                cnt++;
                s += len;
                cons = s;
                if (c2 < 3) { syms |= sym << (8 * c2); c2++; cons2 = s; }
            }
            row_esc = cnt == 0;
            row_e1 = cons | (cnt << 8) | (mask << 23);
            row_e2 = syms | (cons2 << 24) | (c2 << 29);
            if (row_esc) atomicOr(esc_mask + idx / 32, 1u << (idx % 32));
        }
        __syncthreads();
        if (row_esc) {                                             // id = 1 + rank among escape rows
            uint32_t id = 1 + __popc(esc_mask[tid / 32] & ((1u << (tid % 32)) - 1u));
            for (uint32_t q2 = 0; q2 < tid / 32; q2++) id += __popc(esc_mask[q2]);
            if (id > kEscRows) id = 0;                             // no second-level table: walk
            else esc_row[id - 1] = tid;
            row_e1 = id << 23;                                     // advances nothing: the thread stalls
            row_e2 = id;
        }
        if (tid < kRows) {
            uint4 *d1 = reinterpret_cast<uint4 *>(smem_w + kOffT1 / 4 + tid * 32);
            uint4 *d2 = reinterpret_cast<uint4 *>(smem_w + kOffT2 / 4 + tid * 32);
#pragma unroll
            for (int q2 = 0; q2 < 8; q2++) {
                d1[q2] = make_uint4(row_e1, row_e1, row_e1, row_e1);
                d2[q2] = make_uint4(row_e2, row_e2, row_e2, row_e2);
            }
        }
        __syncthreads();
        {   // second-level tables: row id-1, next kR2 bits -> sym | len << 8 (0 if longer than kR + kR2)
            uint32_t n_esc = 0;
            for (uint32_t q2 = 0; q2 < kRows / 32; q2++) n_esc += __popc(esc_mask[q2]);
            n_esc = min(n_esc, kEscRows);
            uint16_t *l2 = reinterpret_cast<uint16_t *>(sb + kOffL2);
            for (uint32_t i = tid; i < n_esc << kR2; i += kCta) {
                const uint32_t row = esc_row[i >> kR2], j = i & ((1u << kR2) - 1u);
                uint32_t len;
                const uint32_t sym = walk((row << (32 - kR)) | (j << (32 - kR - kR2)), len);
                l2[i] = len <= (uint32_t)(kR + kR2) ? (uint16_t)(sym | (len << 8)) : (uint16_t)0;
            }
        }
        __syncthreads();

        // resolve one code longer than R bits at the top of `a` (escape row id from the table entry)
        auto escape = [&](uint32_t a_, uint32_t id, uint32_t &len) -> uint32_t {
            if (id != 0) {
                uint32_t v;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v)
                             : "r"(sbase + kOffL2 + (((id - 1) << kR2) + ((a_ >> (32 - kR - kR2)) & ((1u << kR2) - 1u))) * 2));
                if (v >> 8) { len = v >> 8; return v & 0xFFu; }
            }
            return walk(a_, len);
        };
        const uint32_t N = (uint32_t)ts.num_elements;
        const bool vec_out = ((reinterpret_cast<uintptr_t>(ts.out) & 15) == 0);
        const uint4 *__restrict__ psm4 = reinterpret_cast<const uint4 *>(ts.packed_sign_mantissa);
        uint16_t *__restrict__ out = ts.out;

        uint32_t tile = seg_begin + g;
        if (t == 0) {                                                          // producer: first two tiles
            if (tile < seg_end) issue_tile(ts, tile - base_tile, stage0 + (q & 1) * kStageBytes, mbar0 + (q & 1) * 8);
            if (tile + kGroups < seg_end)
                issue_tile(ts, tile + kGroups - base_tile, stage0 + ((q + 1) & 1) * kStageBytes, mbar0 + ((q + 1) & 1) * 8);
        }
        uint32_t nlo = 0, nhi = 0;
        if (tile < seg_end) {
            nlo = __ldg(ts.block_output_pos + tile - base_tile);
            nhi = __ldg(ts.block_output_pos + tile - base_tile + 1);
        }
        for (; tile < seg_end; tile += kGroups, q++) {
            const uint32_t b = tile - base_tile;
            const uint32_t clo = nlo, chi = nhi;
            const bool has_next = tile + kGroups < seg_end;
            if (has_next) {                                                    // prefetch next BlockOutputPos
                nlo = __ldg(ts.block_output_pos + b + kGroups);
                nhi = __ldg(ts.block_output_pos + b + kGroups + 1);
            }
            const uint32_t st = stage0 + (q & 1) * kStageBytes;
            mbar_wait(mbar0 + (q & 1) * 8, (q >> 1) & 1u);
            uint32_t gap, raw0, raw1, raw2;
            {
                uint32_t h0, h1;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(raw0), "=r"(raw1) : "r"(st + t * kN));
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(raw2) : "r"(st + t * kN + 8));
                const uint32_t gb0 = st + kChunkBytes + ((t * 5) >> 3);
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(h0) : "r"(gb0));
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(h1) : "r"(gb0 + 1));
                gap = (((h0 << 8) | h1) >> (11u - ((t * 5) & 7u))) & 31u;
            }
            const uint32_t lo = min(clo, N);
            const uint32_t hi = min(max(min(chi, N), lo), lo + (uint32_t)(8 * kN * kT));
            const uint32_t f = lo & ~15u;                                      // 16-element frame

            // ---- phase 1: bit buffer (a:b:c) starts at the gap; acc = offset | count << 8 (+ junk >= bit 23)
            uint32_t a = bswap32(raw0), bb = bswap32(raw1), c = bswap32(raw2);
            shift96(a, bb, c, gap);
            uint32_t acc = gap, e1 = 1;
            for (;;) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t e = lds32(madlo(mulhi(a, K_ROW), K_128, t1_lane));
                    if ((acc & 0xC0u) == 0) {                                  // offset < 64: still ours
                        acc += e;
                        e1 = e;
                    }
                    shift96(a, bb, c, e);                                      // e & 31 = consumed bits
                }
                const bool live = (acc & 0xC0u) == 0, esc = live && (e1 & 0x7FFFFFu) == 0;
                const uint32_t flags = __reduce_or_sync(FULL, (live ? 1u : 0u) | (esc ? 2u : 0u));
                if (!(flags & 1u)) break;
                if (flags & 2u) {
                    if (esc) {                                                 // code longer than R bits
                        uint32_t len;
                        escape(a, e1 >> 23, len);
                        e1 = 0;                                                // exactly one code: no fixup
                        acc += len + (1u << 8);
                        shift96(a, bb, c, len & 31u);
                        if (len == 32) { a = bb; bb = c; c = 0; }
                    }
                }
            }
            uint32_t cnt = (acc >> 8) & 0x7Fu;
            if ((e1 & 0x7FFFFFu) != 0) {   // last T1 group may hold complete codes starting at bit >= 64
                const uint32_t last = (acc & 0xFFu) - (e1 & 0xFu);             // < 64
                cnt -= __popc((e1 >> 23) >> min(64u - last, 31u));
            }

            // ---- block exclusive scan of the counts: warp shuffles + 8 warp totals (1 barrier)
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(FULL, incl, d);
                if (lane >= (uint32_t)d) incl += v;
            }
            uint32_t *ws = wsum + parity * 8;
            if (lane == 31) ws[wig] = incl;
            group_bar(g);                          // every thread has read this tile's stage
            parity ^= 1u;
            if (t == 0 && tile + 2 * kGroups < seg_end)
                issue_tile(ts, b + 2 * kGroups, st, mbar0 + (q & 1) * 8);
            uint32_t wpre = 0;
            {
                const uint4 a = *reinterpret_cast<const uint4 *>(ws);
                const uint4 c = *reinterpret_cast<const uint4 *>(ws + 4);
                const uint32_t v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
                for (uint32_t q = 0; q < 7; q++) wpre += q < wig ? v[q] : 0u;
            }
            const uint32_t wtot = __shfl_sync(FULL, incl, 31);
            // this warp's output range [ra, rb) (absolute elements), clipped to the tile
            const uint32_t ra = min(lo + wpre, hi), rb = min(lo + wpre + wtot, hi);
            // full 16-element groups [ga, gb) take the vector path; the <= 15 + 15 edge elements
            // [ra, ha) and [tb, rb) are shared with the neighbouring warps and go one per lane
            const uint32_t ga = vec_out ? (ra + 15) >> 4 : 0, gb = vec_out ? max(rb >> 4, ga) : 0;
            const uint32_t ha = vec_out ? min(ga << 4, rb) : rb, tb = vec_out ? max(gb << 4, ha) : rb;
            uint4 smA = make_uint4(0, 0, 0, 0), smB = make_uint4(0, 0, 0, 0);
            if (ga + lane < gb) smA = __ldg(psm4 + ga + lane);                 // prefetch for the merge
            if (ga + lane + 32 < gb) smB = __ldg(psm4 + ga + lane + 32);
            const uint32_t es = lane < 16 ? ra + lane : tb + (lane - 16);      // this lane's edge element
            const bool edge = vec_out && (lane < 16 ? es < ha : es < rb);
            uint32_t sm1 = 0;
            if (edge) sm1 = __ldg(ts.packed_sign_mantissa + es);

            // ---- phase 2: re-decode with T2 (<= 3 exponents per lookup) into the SMEM buffer
            const uint32_t wp0 = sbase + ebuf_off + (lo - f) + wpre + incl - cnt;
            const uint32_t wend = wp0 + cnt;
            const uint32_t wend1 = wend - 1, wend2 = wend - 2;
            uint32_t wp = wp0, e2 = 1;
            a = bswap32(raw0); bb = bswap32(raw1); c = bswap32(raw2);
            shift96(a, bb, c, gap);
            for (;;) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    // finished lanes keep advancing harmlessly: every store is predicated on wp
                    e2 = lds32(madlo(mulhi(a, K_ROW), K_128, t2_lane));
                    sts8_if<0>(wp, e2, wp, wend);
                    sts8_if<1>(wp, mulhi(e2, K_S8), wp, wend1);
                    sts8_if<2>(wp, mulhi(e2, K_S16), wp, wend2);
                    wp = madhi(e2, K_S29, wp);                                 // wp += count
                    shift96(a, bb, c, mulhi(e2, K_S24));                       // (e2 >> 24) & 31 = consumed
                }
                const bool live = wp < wend, esc = live && e2 < (1u << 24);
                const uint32_t flags = __reduce_or_sync(FULL, (live ? 1u : 0u) | (esc ? 2u : 0u));
                if (!(flags & 1u)) break;
                if (flags & 2u) {
                    if (esc) {
                        uint32_t len;
                        const uint32_t sym = escape(a, e2 & 0xFFu, len);
                        asm volatile("st.shared.u8 [%0], %1;" ::"r"(wp), "r"(sym) : "memory");
                        wp++;
                        shift96(a, bb, c, len & 31u);
                        if (len == 32) { a = bb; bb = c; c = 0; }
                    }
                }
            }
            __syncwarp();

            // ---- per-warp merge of [ra, rb): compose BF16 and store
            const uint8_t *ebf = sb + ebuf_off;                                // ebf[e - f] = exponent of element e
            if (edge) out[es] = compose(ebf[es - f], sm1);
            for (uint32_t gi = ga + lane, it = 0; gi < gb; gi += 32, it++) {
                const uint32_t e0 = gi << 4;
                const uint4 sm = it == 0 ? smA : (it == 1 ? smB : __ldg(psm4 + gi));
                const uint4 ex = *reinterpret_cast<const uint4 *>(ebf + (e0 - f));
                uint4 o0, o1;
                o0.x = compose2<false>(ex.x, sm.x);
                o0.y = compose2<true>(ex.x, sm.x);
                o0.z = compose2<false>(ex.y, sm.y);
                o0.w = compose2<true>(ex.y, sm.y);
                o1.x = compose2<false>(ex.z, sm.z);
                o1.y = compose2<true>(ex.z, sm.z);
                o1.z = compose2<false>(ex.w, sm.w);
                o1.w = compose2<true>(ex.w, sm.w);
                uint4 *dst = reinterpret_cast<uint4 *>(out + e0);
                dst[0] = o0;
                dst[1] = o1;
            }
            if (!vec_out)                                                      // unaligned output: scalar
                for (uint32_t e = ra + lane; e < rb; e += 32)
                    out[e] = compose(ebf[e - f], __ldg(ts.packed_sign_mantissa + e));
        }
        seg_begin = seg_end;
    }
}

int g_attr_set[64];

}  // namespace

bool fast_supports(const df11_device_tensor &t) {
    return t.T == (uint32_t)kT && t.n == (uint32_t)kN &&
           (reinterpret_cast<uintptr_t>(t.encoded_exponent) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(t.gaps) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(t.packed_sign_mantissa) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(t.out) & 1) == 0;
}

cudaError_t launch_fast(const Batch &bt, int device, cudaStream_t stream, uint64_t *launches) {
    if (bt.total_tiles == 0) return cudaSuccess;
    int num_sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    if (device >= 0 && device < 64 && !g_attr_set[device]) {
        e = cudaFuncSetAttribute(fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        if (e != cudaSuccess) return e;
        g_attr_set[device] = 1;
    }
    const uint32_t want = (bt.total_tiles + kGroups - 1) / kGroups;
    const uint32_t grid = min((uint32_t)num_sms, want);
    fast_kernel<<<grid, kCta, kSmemBytes, stream>>>(bt);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace df11
