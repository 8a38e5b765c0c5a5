// decode_sp.cu — single-pass variant of the persistent sm_100a DF11 decode kernel.
//
// Same result and tile schedule as decode_fast.cu, but each chunk is decoded ONCE:
//
//  * Phase 1 (count) and phase 2 (re-decode) of Algorithm 1 are fused.  Every lane decodes
//    its two chunks as two interleaved chains with the 3-symbol table T2 and writes the exponents into
//    a private SMEM slot (48 bytes per chain), unpredicated.  A chain's bit offset is tracked as
//    x = Σ(consumed + 32·count) so that offset = gap + x − 32·written needs no per-step masking; at the
//    warp checks a chain whose offset passed its chunk end is frozen on an all-zero "null" table row.
//    The few codes decoded past the end before the freeze are dropped afterwards (walk back over the
//    slot with CodeLengths).
//  * After the group scan (BlockOutputPos + prefix of counts) each warp compacts its lanes'
//    slots in place into its own SMEM region at the final 16-byte frame offset (word stores with a
//    funnel shift; partial edge words byte by byte), then merges exactly as decode_fast.cu does.
//  * Tensors whose Huffman code has a 1-bit codeword (a chain could hold up to 64 codes) take a
//    count-only pass plus direct HBM writes instead (rare: near-constant tensors).
//
// Compared with two decode passes this removes the T1 table (64 KB of SMEM), its build, and the
// per-step conditional update of phase 1; it adds the compaction.
#include "fast_helpers.cuh"

#include <type_traits>

namespace df11 {
namespace {

constexpr int kSpFirst = 4;                 // decode steps before the first warp check
constexpr int kSpEach = 2;                  // decode steps between later warp checks
constexpr uint32_t kSpGroups = 8;
constexpr uint32_t kSpCta = kLanes * kSpGroups;
constexpr uint32_t kSpWarps = kLanes / 32;
constexpr uint32_t kSpR = 9;                // root bits of T2
constexpr uint32_t kSpRows = 1u << kSpR;
constexpr uint32_t kSpTabBytes = (kSpRows + 1) * 128;   // 32 lane replicas per row + the null row
constexpr uint32_t kSpEscRows = 8;
constexpr uint32_t kSpR2 = 9;
constexpr uint32_t kSpLutSmem = 8192;
constexpr uint32_t kSub = 48;               // slot bytes per chain: <= 32 codes + overshoot + 3
constexpr uint32_t kSlot = 2 * kSub + 4;    // per lane (chain A, chain B); 25 words: lanes hit distinct banks
constexpr uint32_t kWarpReg = 16 + 32 * kSlot;   // per-warp region: frame pad + 32 slots

constexpr uint32_t kSpOffT2 = 0;
constexpr uint32_t kSpOffL2 = kSpOffT2 + kSpTabBytes;                   // uint16 [esc rows][1 << R2]
constexpr uint32_t kSpOffLut = kSpOffL2 + kSpEscRows * (1u << kSpR2) * 2;
constexpr uint32_t kSpOffLen = kSpOffLut + kSpLutSmem;
constexpr uint32_t kSpOffWsum = kSpOffLen + 256;                        // [groups][2][warps]
constexpr uint32_t kSpOffReg = kSpOffWsum + kSpGroups * 2 * kSpWarps * 4;   // [groups][warps][kWarpReg]
constexpr uint32_t kSpOffStage = kSpOffReg + kSpGroups * kSpWarps * kWarpReg;
constexpr uint32_t kSpOffMbar = kSpOffStage + kSpGroups * kStageBytes;
constexpr uint32_t kSpSmem = kSpOffMbar + kSpGroups * 8;
static_assert(kSpOffReg % 16 == 0 && kWarpReg % 16 == 0 && kSpOffStage % 16 == 0 && kSpOffMbar % 8 == 0,
              "alignment");
static_assert(kSpSmem <= 232448, "SMEM budget");

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
__device__ __forceinline__ void lds128(uint32_t addr, uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
}
// 96-bit bit buffer shifts that pull in one-bits (the chain-end sentinel, see sp_kernel)
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

// Copy n (<= 47) bytes held in w[0..11] (little-endian byte stream) to SMEM byte address d.
// Phase A: the whole words of the destination (the last may carry garbage past the end: the next
// chain's phase B rewrites those bytes).  Phase B (after a __syncwarp): the first, partial word.
__device__ __forceinline__ void compact_words(uint32_t d, const uint32_t (&w)[12], uint32_t n) {
    const uint32_t r = d & 3u, db = d - r, sh = r * 8u;
    const uint32_t nw = (r + n + 3u) >> 2;
#pragma unroll
    for (int k = 0; k < 12; k++) {
        const uint32_t v = k == 0 ? w[0] : __funnelshift_l(w[k - 1], w[k], sh);
        sts32_if(db + 4u * k, v, (uint32_t)k < nw && (k > 0 || r == 0));
    }
}
__device__ __forceinline__ void compact_head(uint32_t d, uint32_t w0, uint32_t n) {
    const uint32_t r = d & 3u, db = d - r;
    if (r == 0) return;
    const uint32_t v0 = w0 << (r * 8u);
#pragma unroll
    for (uint32_t i = 1; i < 4; i++)
        if (i >= r && i < r + n) st8(db + i, v0 >> (8u * i));
}

__global__ void __launch_bounds__(kSpCta, 1) sp_kernel(const __grid_constant__ Batch bt) {
    const uint32_t tid = threadIdx.x;
    const uint32_t g = tid / kLanes;
    const uint32_t t = tid % kLanes;
    const uint32_t lane = tid & 31, wig = t >> 5;
    const uint32_t FULL = 0xFFFFFFFFu;
#define K_ROW bt.kpow[0]
#define K_128 bt.kpow[1]
#define K_S24 bt.kpow[2]
#define K_S8 bt.kpow[3]
#define K_S16 bt.kpow[4]
#define K_HALF bt.kpow[6]
#define K_SH7 bt.kpow[7]
    uint8_t *sb = smem_b();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_w);
    const uint32_t t2_lane = sbase + kSpOffT2 + lane * 4u;
    const uint32_t null_lane = sbase + kSpOffT2 + kSpRows * 128u + lane * 4u;
    const uint32_t wreg = kSpOffReg + (g * kSpWarps + wig) * kWarpReg;   // this warp's region (byte offset)
    uint32_t *wsum = smem_w + kSpOffWsum / 4 + g * 2 * kSpWarps;
    const uint32_t stage = sbase + kSpOffStage + g * kStageBytes;
    const uint32_t mbar = sbase + kSpOffMbar + g * 8;
    const uint32_t slotA = sbase + wreg + 16u + lane * kSlot, slotB = slotA + kSub;

    const uint32_t total = bt.total_tiles;
    const uint32_t c_begin = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t c_end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    if (c_begin >= c_end) return;
    if (t == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) smem_w[(kSpOffT2 + kSpRows * 128u) / 4 + tid] = 0;   // null row: advances nothing
    uint32_t q = 0, parity = 0;

    int ti_idx = tensor_of_tile(bt, c_begin);
    for (uint32_t seg_begin = c_begin; seg_begin < c_end; ti_idx++) {
        const df11_device_tensor &ts = bt.t[ti_idx];
        const uint32_t seg_end = min(c_end, bt.tile_start[ti_idx + 1]);
        const uint32_t base_tile = bt.tile_start[ti_idx] - bt.tile_off[ti_idx];
        if (seg_end <= seg_begin) continue;

        // =============================== T2 for this tensor (CTA-wide)
        __syncthreads();
        const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k;
        const uint32_t lut_bytes = kk * 256u * eb_bytes;
        const bool lut_in_smem = lut_bytes <= kSpLutSmem;
        if (lut_in_smem)
            for (uint32_t i = tid; i < lut_bytes; i += kSpCta) sb[kSpOffLut + i] = __ldg(ts.luts + i);
        for (uint32_t i = tid; i < 256u; i += kSpCta) sb[kSpOffLen + i] = __ldg(ts.code_lengths + i);
        uint32_t *esc_mask = smem_w + kSpOffReg / 4;                 // scratch: the regions are idle
        uint32_t *esc_row = esc_mask + kSpRows / 32;
        if (tid < kSpRows / 32) esc_mask[tid] = 0;
        __syncthreads();
        auto walk = [&](uint32_t w, uint32_t &len) -> uint32_t {
            if (lut_in_smem) return lut_walk_smem(w, sbase + kSpOffLut, sbase + kSpOffLen, eb_bytes, kk, len);
            return lut_walk_global(w, ts, len);
        };
        uint32_t row_e2 = 0;
        bool row_esc = false;
        if (tid < kSpRows) {
            const uint32_t W = tid << (32 - kSpR);
            uint32_t s = 0, syms = 0, c2 = 0, cons2 = 0;
            while (s < kSpR && c2 < 3) {
                uint32_t len;
                const uint32_t sym = walk(W << s, len);
                if (len > kSpR - s) break;
                s += len;
                syms |= sym << (8 * c2);
                c2++;
                cons2 = s;
            }
            row_esc = c2 == 0;
            row_e2 = syms | (cons2 << 24) | (c2 << 29);
            if (row_esc) atomicOr(esc_mask + tid / 32, 1u << (tid % 32));
        }
        __syncthreads();
        if (row_esc) {
            uint32_t id = 1 + __popc(esc_mask[tid / 32] & ((1u << (tid % 32)) - 1u));
            for (uint32_t q2 = 0; q2 < tid / 32; q2++) id += __popc(esc_mask[q2]);
            if (id > kSpEscRows) id = 0;
            else esc_row[id - 1] = tid;
            row_e2 = id;
        }
        if (tid < kSpRows) {
            uint4 *d2 = reinterpret_cast<uint4 *>(smem_w + kSpOffT2 / 4 + tid * 32);
#pragma unroll
            for (int q2 = 0; q2 < 8; q2++) d2[q2] = make_uint4(row_e2, row_e2, row_e2, row_e2);
        }
        // a 1-bit codeword allows 64 codes per chain: such tensors take the count + direct path
        const bool safe = __syncthreads_or(tid < 256u && sb[kSpOffLen + tid] == 1) != 0;
        // if R one-bits hold no complete code (row 1...1 is an escape row: true for canonical codes
        // longer than R bits), one-bits after a chain's last bit stall it exactly there
        const bool long_codes = __syncthreads_or(tid == kSpRows - 1 && row_esc) != 0;
        {
            uint32_t n_esc = 0;
            for (uint32_t q2 = 0; q2 < kSpRows / 32; q2++) n_esc += __popc(esc_mask[q2]);
            n_esc = min(n_esc, kSpEscRows);
            uint16_t *l2 = reinterpret_cast<uint16_t *>(sb + kSpOffL2);
            for (uint32_t i = tid; i < (n_esc << kSpR2); i += kSpCta) {
                const uint32_t row = esc_row[i >> kSpR2], j = i & ((1u << kSpR2) - 1u);
                uint32_t len;
                const uint32_t sym = walk((row << (32 - kSpR)) | (j << (32 - kSpR - kSpR2)), len);
                l2[i] = len <= kSpR + kSpR2 ? (uint16_t)(sym | (len << 8)) : (uint16_t)0;
            }
        }
        __syncthreads();

        auto escape = [&](uint32_t a_, uint32_t id, uint32_t &len) -> uint32_t {
            if (id != 0) {
                uint32_t v;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v)
                             : "r"(sbase + kSpOffL2 + (((id - 1) << kSpR2) + ((a_ >> (32 - kSpR - kSpR2)) & ((1u << kSpR2) - 1u))) * 2));
                if (v >> 8) { len = v >> 8; return v & 0xFFu; }
            }
            return walk(a_, len);
        };
        auto escape_packed = [&](uint32_t a_, uint32_t id) -> uint32_t {
            uint32_t v = 0;
            if (id != 0)
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v)
                             : "r"(sbase + kSpOffL2 + (((id - 1) << kSpR2) + ((a_ >> (32 - kSpR - kSpR2)) & ((1u << kSpR2) - 1u))) * 2));
            if ((v >> 8) == 0) {
                uint32_t len;
                const uint32_t sym = walk(a_, len);
                v = sym | (len << 8);
            }
            return v;
        };
        const uint32_t N = (uint32_t)ts.num_elements;
        const bool vec_out = ((reinterpret_cast<uintptr_t>(ts.out) & 15) == 0);
        const uint4 *__restrict__ psm4 = reinterpret_cast<const uint4 *>(ts.packed_sign_mantissa);
        uint16_t *__restrict__ out = ts.out;
        const uint32_t lenb = sbase + kSpOffLen;

        // =============================== tiles of this group
        uint32_t tile = seg_begin + g;
        if (t == 0 && tile < seg_end) issue_tile(ts, tile - base_tile, stage, mbar);
        uint32_t nlo = 0, nhi = 0;
        if (tile < seg_end) {
            nlo = __ldg(ts.block_output_pos + tile - base_tile);
            nhi = __ldg(ts.block_output_pos + tile - base_tile + 1);
        }
        auto prefetch_sm = [&](uint32_t plo, uint32_t phi) {
            const uint32_t a0 = min(plo, N) & ~15u, a1 = (min(max(phi, plo), N) + 15u) & ~15u;
            if (a1 > a0) prefetch_l2(ts.packed_sign_mantissa + a0, a1 - a0);
        };
        if (t == 0 && tile < seg_end) prefetch_sm(nlo, nhi);
        for (; tile < seg_end; tile += kSpGroups, q++) {
            const uint32_t b = tile - base_tile;
            const uint32_t clo = nlo, chi = nhi;
            const bool has_next = tile + kSpGroups < seg_end;
            if (has_next) {
                nlo = __ldg(ts.block_output_pos + b + kSpGroups);
                nhi = __ldg(ts.block_output_pos + b + kSpGroups + 1);
            }
            mbar_wait(mbar, q & 1u);
            uint32_t r0, r1, r2, r3, r4, gapA, gapB, gapC;
            {
                lds128(stage + t * 16, r0, r1, r2, r3);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r4) : "r"(stage + t * 16 + 16));
                const uint32_t gb0 = stage + kChunkBytes + ((t * 10) >> 3);
                // gaps of chunks 2t, 2t+1 and 2t+2 (the next tile's first for t = 127: the stage holds
                // 16 bytes of gaps past the tile) start at bit 10t
                const uint32_t h0 = ld8(gb0), h1 = ld8(gb0 + 1), h2 = ld8(gb0 + 2), h3 = ld8(gb0 + 3);
                const uint32_t g32 = (h0 << 24) | (h1 << 16) | (h2 << 8) | h3;
                const uint32_t g15 = (g32 >> (17u - ((t * 10) & 7u))) & 32767u;
                gapA = g15 >> 10;
                gapB = (g15 >> 5) & 31u;
                gapC = g15 & 31u;
            }
            const uint32_t lo = min(clo, N);
            const uint32_t hi = min(max(min(chi, N), lo), lo + 8 * kN * kT);
            const uint32_t W0 = bswap32(r0), W1 = bswap32(r1), W2 = bswap32(r2), W3 = bswap32(r3),
                           W4 = bswap32(r4);

            uint32_t cntA, cntB;
            if (!safe) {
                // ---- single decode pass into the private slots (chains A: [gapA, 64), B: [64+gapB, 128))
                // exact chain ends when the next chunk's gap marks a code start (every tile but the
                // one holding the tensor's last code): A = [gapA, 64 + gapB), B = [64 + gapB, 128 + gapC),
                // enforced by one-bits after the end; otherwise [.., 64) / [.., 128) + walk back
                const bool exact = long_codes && hi < N;
                const uint32_t endA = exact ? 64u + gapB : 64u, endB = exact ? 128u + gapC : 128u;
                uint32_t aA = W0, bA = W1, cA = exact ? W2 | (0xFFFFFFFFu >> gapB) : W2;
                uint32_t aB = W2, bB = W3, cB = exact ? W4 | (0xFFFFFFFFu >> gapC) : W4;
                shift96_ones(aA, bA, cA, gapA);
                shift96_ones(aB, bB, cB, gapB);
                uint32_t wA = slotA, wB = slotB, xA = 0, xB = 0, tA = t2_lane, tB = t2_lane;
                uint32_t eA = 1u << 24, eB = 1u << 24;
                auto step = [&]() {
                    eA = lds32(madlo(mulhi(aA, K_ROW), K_128, tA));
                    eB = lds32(madlo(mulhi(aB, K_ROW), K_128, tB));
                    st8k<0>(wA, eA);
                    st8k<1>(wA, mulhi(eA, K_S8));
                    st8k<2>(wA, mulhi(eA, K_S16));
                    st8k<0>(wB, eB);
                    st8k<1>(wB, mulhi(eB, K_S8));
                    st8k<2>(wB, mulhi(eB, K_S16));
                    wA += eA >> 29;                                            // count
                    wB += eB >> 29;
                    const uint32_t vA = mulhi(eA, K_S24), vB = mulhi(eB, K_S24);   // consumed + 32*count
                    xA += vA;
                    xB += vB;
                    shift96_ones(aA, bA, cA, vA);
                    shift96_ones(aB, bB, cB, vB);
                };
#pragma unroll
                for (int u = 0; u < kSpFirst; u++) step();
                for (;;) {
                    const uint32_t offA = gapA + xA - 32u * (wA - slotA);
                    const uint32_t offB = 64u + gapB + xB - 32u * (wB - slotB);
                    const bool actA = offA < endA, actB = offB < endB;
                    if (!__any_sync(FULL, actA || actB)) break;
                    if (!actA) { tA = null_lane; aA = 0; }                     // freeze on the null row
                    if (!actB) { tB = null_lane; aB = 0; }
                    const bool escA = actA && eA < (1u << 24), escB = actB && eB < (1u << 24);
                    if (__any_sync(FULL, escA || escB)) {
                        const uint32_t vA = escA ? escape_packed(aA, eA & 0xFFu) : 0u;
                        const uint32_t vB = escB ? escape_packed(aB, eB & 0xFFu) : 0u;
                        if (escA) {
                            st8(wA, vA);
                            wA++;
                            xA += (vA >> 8) + 32u;
                            shift96_long_ones(aA, bA, cA, vA >> 8);
                        }
                        if (escB) {
                            st8(wB, vB);
                            wB++;
                            xB += (vB >> 8) + 32u;
                            shift96_long_ones(aB, bB, cB, vB >> 8);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kSpEach; u++) step();
                }
                // drop the codes decoded past each chain's end (they start at or after it)
                uint32_t offA = gapA + xA - 32u * (wA - slotA);
                while (!exact && wA > slotA) {
                    const uint32_t l = ld8(lenb + ld8(wA - 1));
                    if (offA - l < 64u) break;
                    offA -= l;
                    wA--;
                }
                uint32_t offB = 64u + gapB + xB - 32u * (wB - slotB);
                while (!exact && wB > slotB) {
                    const uint32_t l = ld8(lenb + ld8(wB - 1));
                    if (offB - l < 128u) break;
                    offB -= l;
                    wB--;
                }
                cntA = wA - slotA;
                cntB = wB - slotB;
            } else {
                // ---- count-only pass, one code at a time (1-bit codewords)
                auto count_chain = [&](uint32_t a, uint32_t bb, uint32_t c, uint32_t off, uint32_t lim) {
                    uint32_t n = 0;
                    while (off < lim) {
                        const uint32_t e = lds32(madlo(mulhi(a, K_ROW), K_128, t2_lane));
                        uint32_t len;
                        if (e >= (1u << 24)) len = ld8(lenb + (e & 0xFFu));
                        else escape(a, e & 0xFFu, len);
                        n++;
                        off += len;
                        shift96_long(a, bb, c, len);
                    }
                    return n;
                };
                uint32_t a = W0, bb = W1, c = W2;
                shift96(a, bb, c, gapA);
                cntA = count_chain(a, bb, c, gapA, 64u);
                a = W2; bb = W3; c = W4;
                shift96(a, bb, c, gapB);
                cntB = count_chain(a, bb, c, 64u + gapB, 128u);
            }
            const uint32_t cnt = cntA + cntB;

            // ---- exclusive scan of the counts over the tile: warp shuffles + 4 warp totals
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(FULL, incl, d);
                if (lane >= (uint32_t)d) incl += v;
            }
            uint32_t *ws = wsum + parity * kSpWarps;
            if (lane == 31) ws[wig] = incl;
            group_bar(g);                          // also: every thread has read this tile's stage
            parity ^= 1u;
            if (t == 0 && has_next) {
                issue_tile(ts, b + kSpGroups, stage, mbar);
                prefetch_sm(nlo, nhi);
            }
            uint32_t wpre = 0;
            {
                const uint4 v = *reinterpret_cast<const uint4 *>(ws);
                wpre = (wig > 0 ? v.x : 0u) + (wig > 1 ? v.y : 0u) + (wig > 2 ? v.z : 0u);
            }
            const uint32_t wtot = __shfl_sync(FULL, incl, 31);
            const uint32_t lpos = incl - cnt;                                  // first output in the warp
            const uint32_t wbeg = lo + wpre;                                   // the warp's first output

            if (safe) {
                // direct mode: compose and store to HBM per code
                uint32_t a = W0, bb = W1, c = W2;
                shift96(a, bb, c, gapA);
                uint32_t p = wbeg + lpos;
                const uint32_t pend = min(p + cnt, hi);
#pragma unroll 1
                for (int sub = 0; sub < 2; sub++) {
                    uint32_t off = sub ? 64u + gapB : gapA;
                    if (sub) { a = W2; bb = W3; c = W4; shift96(a, bb, c, gapB); }
                    const uint32_t lim_off = sub ? 128u : 64u;
                    while (p < pend && off < lim_off) {
                        uint32_t len;
                        const uint32_t e = lds32(madlo(mulhi(a, K_ROW), K_128, t2_lane));
                        uint32_t syms, n, consumed;
                        if (e >= (1u << 24)) { syms = e; n = e >> 29; consumed = (e >> 24) & 31u; }
                        else { syms = escape(a, e & 0xFFu, len); n = 1; consumed = len; }
                        uint32_t start = off;
                        for (uint32_t i = 0; i < n && p < pend && start < lim_off; i++, p++) {
                            const uint32_t sym = (syms >> (8 * i)) & 0xFFu;
                            out[p] = compose(sym, __ldg(ts.packed_sign_mantissa + p));
                            start += n == 1 ? consumed : ld8(lenb + sym);
                        }
                        off += consumed;
                        shift96_long(a, bb, c, consumed);
                    }
                }
                continue;
            }

            // ---- this warp's output range and its sign/mantissa prefetch
            const uint32_t F = wbeg & ~15u;                                    // region byte of e: e - F
            const uint32_t ra = min(wbeg, hi), rb = min(wbeg + wtot, hi);
            const uint32_t ga = vec_out ? (ra + 15) >> 4 : 0, gb = vec_out ? max(rb >> 4, ga) : 0;
            const uint32_t ha = vec_out ? min(ga << 4, rb) : rb, tb = vec_out ? max(gb << 4, ha) : rb;
            uint4 smA = make_uint4(0, 0, 0, 0), smB = make_uint4(0, 0, 0, 0);
            if (ga + lane < gb) smA = __ldg(psm4 + ga + lane);
            if (ga + lane + 32 < gb) smB = __ldg(psm4 + ga + lane + 32);
            const uint32_t es = lane < 16 ? ra + lane : tb + (lane - 16);
            const bool edge = vec_out && (lane < 16 ? es < ha : es < rb);
            uint32_t sm1 = 0;
            if (edge) sm1 = __ldg(ts.packed_sign_mantissa + es);

            // ---- compaction of the slots into [F, ...) of the warp region (in place: load all first)
            {
                uint32_t wa[12], wb[12];
#pragma unroll
                for (int k = 0; k < 12; k++) {
                    wa[k] = lds32(slotA + 4u * k);
                    wb[k] = lds32(slotB + 4u * k);
                }
                __syncwarp();
                const uint32_t dA = sbase + wreg + (wbeg - F) + lpos, dB = dA + cntA;
                compact_words(dA, wa, cntA);
                compact_words(dB, wb, cntB);
                __syncwarp();
                compact_head(dA, wa[0], cntA);
                compact_head(dB, wb[0], cntB);
            }
            __syncwarp();

            // ---- per-warp merge of [ra, rb): compose BF16 and store
            const uint8_t *ebf = sb + wreg;                                    // ebf[e - F]
            if (edge) out[es] = compose(ebf[es - F], sm1);
            for (uint32_t gi = ga + lane, it = 0; gi < gb; gi += 32, it++) {
                const uint32_t e0 = gi << 4;
                const uint4 sm = it == 0 ? smA : (it == 1 ? smB : __ldg(psm4 + gi));
                const uint4 ex = *reinterpret_cast<const uint4 *>(ebf + (e0 - F));
                uint4 o0, o1;
                compose4(ex.x, sm.x, o0.x, o0.y, K_HALF, K_SH7);
                compose4(ex.y, sm.y, o0.z, o0.w, K_HALF, K_SH7);
                compose4(ex.z, sm.z, o1.x, o1.y, K_HALF, K_SH7);
                compose4(ex.w, sm.w, o1.z, o1.w, K_HALF, K_SH7);
                uint4 *dst = reinterpret_cast<uint4 *>(out + e0);
                dst[0] = o0;
                dst[1] = o1;
            }
            if (!vec_out)                                                      // unaligned output: scalar
                for (uint32_t e = ra + lane; e < rb; e += 32)
                    out[e] = compose(ebf[e - F], __ldg(ts.packed_sign_mantissa + e));
        }
        seg_begin = seg_end;
    }
#undef K_ROW
#undef K_128
#undef K_S24
#undef K_S8
#undef K_S16
#undef K_HALF
#undef K_SH7
}

int g_sp_attr_set[64];

}  // namespace

cudaError_t launch_sp(const Batch &bt, int device, cudaStream_t stream, uint64_t *launches) {
    if (bt.total_tiles == 0) return cudaSuccess;
    int num_sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    if (device >= 0 && device < 64 && !g_sp_attr_set[device]) {
        e = cudaFuncSetAttribute(sp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpSmem);
        if (e != cudaSuccess) return e;
        g_sp_attr_set[device] = 1;
    }
    const uint32_t grid = bt.grid ? bt.grid : min((uint32_t)num_sms, (bt.total_tiles + kSpGroups - 1) / kSpGroups);
    sp_kernel<<<grid, kSpCta, kSpSmem, stream>>>(bt);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace df11
