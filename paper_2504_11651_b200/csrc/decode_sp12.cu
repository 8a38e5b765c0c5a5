// decode_sp12.cu — the product kernel: single-pass persistent sm_100a DF11 decode with a 12-bit
// multi-code table.
//
// Persistent 1024-thread CTAs of 8 groups; a group owns one format block ("tile") at a time, each
// lane decodes two chunks as two interleaved chains into private SMEM slots, a group scan gives the
// output positions (Alg. 1), the slots are compacted per warp and merged with
// PackedSignMantissa into coalesced BF16 stores.  (The earlier two-pass and 9-bit kernels it
// replaced are kept under scripts/variants/ for A/B history; they are not part of libdf11.so.)
//
//  * T12: 4096 entries of 8 bytes indexed by the next 12 bits of the stream.  An entry holds up to 4
//    complete codes: lo = their exponents (one byte each), hi = consumed bits | 8*count << 24.  12 bits
//    decode 3.8 codes per lookup on LLM-like exponents vs 2.8 for a 9-bit, 3-code table, and codes
//    longer than 12 bits (resolved by the paper's LUT walk) are 8x rarer.  The table is not
//    lane-replicated (32 KB); its LDS.64 bank conflicts are the price of 1.35x fewer lookups.  Row r is
//    stored at index r + (r >> 8): chains near their end look up rows whose low bits are the one-bit
//    padding (below), which would otherwise all fall into one bank pair (measured 10.5 wavefronts per
//    LDS.64 in the decode loop; adding the row's top 4 bits spreads them).
//  * Exponents are stored rotated right by one bit, r = (e >> 1) | (e & 1) << 7: the BF16 high byte is
//    then sign | (r & 0x7F) and the low byte (r & 0x80) | mantissa, two bit-selects per 4
//    elements in the merge instead of a shift, a multiply and two bit-selects.
//  * One step per chain: row = a >> 20, one LDS.64, x += hi, the 96-bit bit-buffer shift by hi & 31
//    (funnel shifts use the low 5 bits), and the exponents are appended to the chain's slot through a
//    pending word: m = acc | lo << fb is stored with ONE 32-bit STS, and the word pointer advances when
//    the word is full.  Slots are lane-column-major (word k of lane l at k*128 + 4l), so every slot
//    access of a warp hits 32 distinct banks.  x += hi accumulates the consumed bits in its low 16 bits
//    (the count sits above).
//  * The merge stores one 8-element unit (16 bytes) per lane and STG.128, so a warp instruction writes
//    512 contiguous bytes (4 L1 wavefronts; two 16-byte halves per lane 32 bytes apart took 8).
//  * A tile's PackedSignMantissa range is staged in SMEM by one TMA bulk copy (FP16: two, one per
//    residual plane); the first tile's copies are issued before the table build; per-CTA tile ranges
//    come from df11_plan_cta_ranges (api.cu).
//  * Programmatic dependent launch: a decode that follows a decode on the same stream builds its table
//    and decodes its first tile on the SMs the previous one leaves in its tail, and waits for it
//    (griddepcontrol.wait) before each tile's first global write (df11.h states the stream semantics).
#include <type_traits>

#include "t12_common.cuh"

namespace df11 {
namespace {

#ifndef SP12_FIRST
#define SP12_FIRST 6
#endif
constexpr int kFirst = SP12_FIRST;          // decode steps before the first warp check
#ifndef SP12_GROUPS
#define SP12_GROUPS 8
#endif
constexpr uint32_t kGroups12 = SP12_GROUPS;
constexpr uint32_t kCta12 = kLanes * kGroups12;
constexpr uint32_t kWarps12 = kLanes / 32;
// slot words per chain: a chain holds <= 32 codes (<= 64 bits of code starts, codes >= 2 bits: 1-bit
// codes take the direct path); without exact ends it may overshoot its end by <= 3 codes (one lookup
// past it in the loop; the unrolled steps consume >= 52 bits only in >= 5 lookups): <= 35 bytes, so the
// pending word never passes word 8.
constexpr uint32_t kSubW = 10;
constexpr uint32_t kWarpReg12 = 16 + 2 * kSubW * 128;   // frame pad + lane-column slots of 2 chains

constexpr uint32_t kOffT = 0;                                       // T12 (t12_common.cuh)
constexpr uint32_t kOffLut = kOffT + kT12Bytes;
constexpr uint32_t kOffLen = kOffLut + kLutSmem;                    // CodeLengths[e]
constexpr uint32_t kOffRLen = kOffLen + 256;                        // CodeLengths[stored symbol]
constexpr uint32_t kOffGrp = kOffRLen + 256;                        // [groups][kGrpBytes]
// PackedSignMantissa bytes of one tile staged in SMEM: BF16 ~6.3 KB per tile on LLM weights; FP16
// (byte plane + 3-bit plane, NEXT-4) ~8.7 KB: it takes the SMEM left over (tiles above the cap read their
// residuals through L1/L2 instead)
constexpr uint32_t sm_cap(uint32_t vf) { return vf == DF11_VF_FP16 ? 11200u : 7168u; }
// FP16 (R25): the tile's byte plane is staged at [0, kFp16HiOff) of the buffer, its 3-bit plane after it
constexpr uint32_t kFp16HiOff = 8000u;
// one block per group, so that every per-group / per-warp address is one base register plus an
// immediate offset
template <uint32_t kVF>
struct Lay12 {
    static constexpr uint32_t kSmCap = sm_cap(kVF);
    static constexpr uint32_t kGStage = 0;                          // stream chunk + gaps (TMA)
    static constexpr uint32_t kGSm = kGStage + kStageBytes;         // PackedSignMantissa (TMA)
    static constexpr uint32_t kGReg = kGSm + kSmCap;                // [warps][kWarpReg12] slots / regions
    static constexpr uint32_t kGWsum = kGReg + kWarps12 * kWarpReg12;   // [2][warps] warp totals
    static constexpr uint32_t kGCnt = kGWsum + 2 * kWarps12 * 4;    // warps done with the merge
    static constexpr uint32_t kGMbar = kGCnt + 16;                  // [stage, sign/mantissa] mbarriers
    static constexpr uint32_t kGrpBytes = kGMbar + 16;
    static constexpr uint32_t kSmem = kOffGrp + kGroups12 * kGrpBytes;
    static_assert(kOffGrp % 16 == 0 && kGSm % 16 == 0 && kGReg % 16 == 0 && kWarpReg12 % 16 == 0 &&
                      kGWsum % 16 == 0 && kGMbar % 8 == 0 && kGrpBytes % 16 == 0,
                  "alignment");
    static_assert(kWarps12 * kWarpReg12 >= 8192, "first-code table scratch fits group 0's warp regions");
    static_assert(kSmem <= 232448, "SMEM budget");
};

// ---- merge helpers of the value formats other than BF16 (NEXT-4, R25): a unit is 16 output bytes
// (8 FP16 / 16 FP8 words) and its residuals are R * (unit words) / 8 bytes at SMEM byte address o.
// Eight FP16 words from 8 stored exponents (bytes of x0, x1: e << 2), their 8 low residual bytes
// (byte plane, s0 / s1) and their 3-bit high fields (sign, m9, m8) as 3 whole bytes at SMEM address h
// (R25).  Per 4 words: the 3-bit fields spread to bytes (W), W * 0x21 puts the sign at bit 7 next to
// m9 m8 at bits 1..0, the exponent byte is ORed in, and one PRMT interleaves high and low bytes.
__device__ __forceinline__ uint4 unit_fp16(uint32_t x0, uint32_t x1, uint32_t s0, uint32_t s1, uint32_t h) {
    const uint32_t base = h & ~3u, r = h & 3u;
    const uint32_t L0 = lds32(base);
    uint32_t L1 = 0;
    if (r >= 2) L1 = lds32(base + 4);                  // 3 bytes from byte 2 or 3 reach the next word
    const uint32_t H = prmt(L0, L1, 0x0123u + r * 0x1111u);   // the 24 bits MSB-first in H's bits 31..8
    const uint32_t W0 = (H >> 29) | ((H >> 18) & 0x700u) | ((H >> 7) & 0x70000u) | ((H << 4) & 0x7000000u);
    const uint32_t W1 = ((H >> 17) & 7u) | ((H >> 6) & 0x700u) | ((H << 5) & 0x70000u) | ((H << 16) & 0x7000000u);
    const uint32_t Y0 = ((W0 * 0x21u) & 0x83838383u) | x0, Y1 = ((W1 * 0x21u) & 0x83838383u) | x1;
    uint4 o;
    o.x = prmt(s0, Y0, 0x5140u);
    o.y = prmt(s0, Y0, 0x7362u);
    o.z = prmt(s1, Y1, 0x5140u);
    o.w = prmt(s1, Y1, 0x7362u);
    return o;
}
// Four FP8 E4M3 bytes from 4 exponents E and the nibbles of residual bytes (b_lo, b_hi) of word r
// (element 2j in the high nibble of byte j): s << 7 | e << 3 | m.
template <uint32_t kSel>
__device__ __forceinline__ uint32_t quad_e4m3(uint32_t r, uint32_t E) {
    const uint32_t P = prmt(r, 0u, kSel);                // [b, b, b', b']
    const uint32_t N = bitsel<0xFF00FF00u>(P >> 4, P);   // low nibble of byte j = residual of element j
    return ((N << 4) & 0x80808080u) | (N & 0x07070707u) | E;          // E: stored e << 3
}
// Four FP8 E5M2 bytes from 4 exponents E and 12 residual bits u (element 0 in bits 11..9): s << 7 |
// e << 2 | m.
__device__ __forceinline__ uint32_t quad_e5m2(uint32_t u, uint32_t E) {
    const uint32_t W = ((u >> 9) & 7u) | (((u >> 6) & 7u) << 8) | (((u >> 3) & 7u) << 16) | ((u & 7u) << 24);
    return ((W << 5) & 0x80808080u) | (W & 0x03030303u) | E;          // E: stored e << 2
}
// Residual of one element from the SMEM staging: R bits at bit position `bit` of the buffer at `buf`.
template <uint32_t kR_>
__device__ __forceinline__ uint32_t res_smem(uint32_t buf, uint32_t bit) {
    const uint32_t p = buf + (bit >> 3), end = (bit & 7u) + kR_;   // bytes read: only those it spans
    uint32_t v = ld8(p) << 16;
    if (end > 8) v |= ld8(p + 1) << 8;
    if (end > 16) v |= ld8(p + 2);
    return (v >> (24u - end)) & ((1u << kR_) - 1u);
}

// kNB = 8: the paper's format (T = 256, n = 8); a lane decodes two 8-byte chunks as two chains.
// kNB = 16: T = 128, n = 16 (NEXT-4: half the gap bits); a format block has the same 2 048 stream
// bytes and a lane decodes its one 16-byte chunk as one chain in a 160-bit buffer.
// kVF: value format (DF11_VF_*, NEXT-4).  Decode, scan and compaction are the same for every format
// (the symbols are exponent fields); the merge composes the format's words.  kB8: the format's LUTs
// are the paper's byte tables (b = 8); otherwise b-bit tables (App. I.2), walked in global memory.
template <uint32_t kNB, uint32_t kVF, bool kB8>
__global__ void __launch_bounds__(kCta12, 1) sp12_kernel(const __grid_constant__ Batch bt) {
    using L = Lay12<kVF>;
    constexpr VF kF = vf_of(kVF);
    constexpr uint32_t kRb = kF.R;                        // residual bits per element
    constexpr uint32_t kU = 16 / kF.word_bytes;           // words per 16-byte output unit
    using OutT = typename std::conditional<kF.word_bytes == 2, uint16_t, uint8_t>::type;
    const uint32_t tid = threadIdx.x;
    const uint32_t g = tid / kLanes;
    const uint32_t t = tid % kLanes;
    const uint32_t lane = tid & 31, wig = t >> 5;
    const uint32_t FULL = 0xFFFFFFFFu;
#define K_ROW bt.kpow[0]   // 2^12: a >> 20
#define K_TOP bt.kpow[1]   // 2^4: a >> 28 (the row's top 4 bits: bank swizzle)
#define K_S24 bt.kpow[2]   // 2^8: >> 24
#define K_ENT bt.kpow[3]   // 8: entry bytes
    uint8_t *sb = smem_b();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_w);
    const uint32_t tab = sbase + kOffT;
    const uint32_t gbase = sbase + kOffGrp + g * L::kGrpBytes;           // this group's block
    const uint32_t wreg = gbase + L::kGReg + wig * kWarpReg12;           // this warp's region
    const uint32_t stage = gbase + L::kGStage;
    const uint32_t mbar = gbase + L::kGMbar;
    const uint32_t smbar = mbar + 8;                        // the tile's PackedSignMantissa has landed
    const uint32_t smb = gbase + L::kGSm;
    const uint32_t mcnt = gbase + L::kGCnt;
    const uint32_t slotA = wreg + 16u + lane * 4u, slotB = slotA + kSubW * 128u;
    const uint32_t rlenb = sbase + kOffRLen;

#ifndef SP12_NO_PDL
    // programmatic dependent launch: the next decode in the stream may start its prologue (the table
    // build and the decode of its first tiles, which read only its own inputs) on SMs this grid leaves;
    // it waits for this grid before its first global write (griddepcontrol.wait after each tile's scan
    // barrier; -DSP12_PDL_EARLY: after the table build instead)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    const uint32_t total = bt.total_tiles;
    const uint32_t c_begin = bt.cta_ranges ? bt.cta_start[blockIdx.x]
                                           : (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t c_end = bt.cta_ranges ? bt.cta_start[blockIdx.x + 1]
                                         : (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    if (c_begin >= c_end) return;
    if (t == 0) {
        mbar_init(mbar, 1);
        mbar_init(smbar, 1);
        sts32(mcnt, 0);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t q = 0, parity = 0, qs = 0;

    int ti_idx = tensor_of_tile(bt, c_begin);
    for (uint32_t seg_begin = c_begin; seg_begin < c_end; ti_idx++) {
        const df11_device_tensor &ts = bt.t[ti_idx];
        const uint32_t seg_end = min(c_end, bt.tile_start[ti_idx + 1]);
        const uint32_t base_tile = bt.tile_start[ti_idx] - bt.tile_off[ti_idx];
        if (seg_end <= seg_begin) continue;

        // =============================== T12 for this tensor (CTA-wide)
        __syncthreads();
        // each group's first tile: its BlockOutputPos reads and stream copies go out first, so that
        // their latency overlaps the table build
        uint32_t tile = seg_begin + g;
        uint32_t nlo = 0, nhi = 0;
        if (tile < seg_end) {
            nlo = __ldg(ts.block_output_pos + tile - base_tile);
            nhi = __ldg(ts.block_output_pos + tile - base_tile + 1);
            if (t == 0) {
                if constexpr (kNB == 8) issue_tile(ts, tile - base_tile, stage, mbar);
                else issue_tile16(ts, tile - base_tile, stage, mbar);
            }
        }
        bool safe, lut_in_smem;
        const bool long_codes = build_t12<kCta12, kVF, kB8>(ts, sb, sbase, kOffT, kOffLut, kOffLen, kOffRLen,
                                                       kOffGrp + L::kGReg, tid, safe, lut_in_smem);
#if !defined(SP12_NO_PDL) && defined(SP12_PDL_EARLY)
        asm volatile("griddepcontrol.wait;" ::: "memory");   // the previous grid is complete and visible
#endif
        const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k;

        const uint32_t N = (uint32_t)ts.num_elements;
        const bool vec_out = ((reinterpret_cast<uintptr_t>(ts.out) & 15) == 0);
        const uint2 *__restrict__ psm2 = reinterpret_cast<const uint2 *>(ts.packed_sign_mantissa);
        OutT *__restrict__ out = static_cast<OutT *>(ts.out);
        // PackedSignMantissa of a tile, [a0, a1) = its output range widened to 16 bytes, is staged in
        // SMEM by one TMA bulk copy (issued by the last warp to finish the previous tile's merge) when
        // it fits kSmCap; otherwise it is prefetched into L2 and read with LDG in the merge.
        const bool psm_al = (reinterpret_cast<uintptr_t>(ts.packed_sign_mantissa) & 15) == 0;   // bulk copies
        const bool sm_tma = vec_out && !safe && psm_al;
        // [a0, a1): bytes of the residuals of outputs [l & ~15, (h + 15) & ~15), widened to 16 bytes.
        // FP16 (R25): [a0, a1) is the byte-plane range; its 3-bit plane range is [hib + q0, hib + q1)
        // with q0 = (3 a0 / 8) & ~15, q1 = roundup(3 a1 / 8, 16), staged at smb + kFp16HiOff.
        const uint32_t hib = (N + 15u) & ~15u;
        auto sm_range = [&](uint32_t plo, uint32_t phi, uint32_t &a0, uint32_t &a1) {
            const uint32_t l = min(plo, N), h = min(max(min(phi, N), l), l + 8 * kN * kT);
            if constexpr (kVF == DF11_VF_FP16) {
                a0 = l & ~15u;
                a1 = (h + 15u) & ~15u;
                const uint32_t q0 = (a0 / 8u * 3u) & ~15u, q1 = (a1 / 8u * 3u + 15u) & ~15u;
                return sm_tma && a1 > a0 && a1 - a0 <= kFp16HiOff && q1 - q0 <= L::kSmCap - kFp16HiOff;
            } else {
                a0 = ((l & ~15u) / 8u * kRb) & ~15u;
                a1 = (((h + 15u) & ~15u) / 8u * kRb + 15u) & ~15u;
                return sm_tma && a1 > a0 && a1 - a0 <= L::kSmCap;
            }
        };
        auto stage_sm = [&](uint32_t plo, uint32_t phi) {
            uint32_t a0, a1;
            const bool fits = sm_range(plo, phi, a0, a1);
            if constexpr (kVF == DF11_VF_FP16) {
                const uint32_t q0 = (a0 / 8u * 3u) & ~15u, q1 = (a1 / 8u * 3u + 15u) & ~15u;
                if (fits) {
                    mbar_expect_tx(smbar, (a1 - a0) + (q1 - q0));
                    tma_g2s(smb, ts.packed_sign_mantissa + a0, a1 - a0, smbar);
                    tma_g2s(smb + kFp16HiOff, ts.packed_sign_mantissa + hib + q0, q1 - q0, smbar);
                } else if (a1 > a0 && psm_al) {
                    prefetch_l2(ts.packed_sign_mantissa + a0, a1 - a0);
                    prefetch_l2(ts.packed_sign_mantissa + hib + q0, q1 - q0);
                }
            } else {
                if (fits) {
                    mbar_expect_tx(smbar, a1 - a0);
                    tma_g2s(smb, ts.packed_sign_mantissa + a0, a1 - a0, smbar);
                } else if (a1 > a0 && psm_al) {
                    prefetch_l2(ts.packed_sign_mantissa + a0, a1 - a0);
                }
            }
        };
        if (t == 0 && tile < seg_end) stage_sm(nlo, nhi);

        auto walk = [&](uint32_t w, uint32_t &len) -> uint32_t {
            if (lut_in_smem)
                return lut_walk_smem(w, sbase + kOffLut, sbase + kOffLen, eb_bytes, kk, kB8 ? 8u : lut_bits_of(ts), len);
            return lut_walk_global<kB8>(w, ts, len);
        };

        // =============================== tiles of this group
        for (; tile < seg_end; tile += kGroups12, q++) {
            const uint32_t b = tile - base_tile;
            const uint32_t clo = nlo, chi = nhi;
            const bool has_next = tile + kGroups12 < seg_end;
            if (has_next) {
                nlo = __ldg(ts.block_output_pos + b + kGroups12);
                nhi = __ldg(ts.block_output_pos + b + kGroups12 + 1);
            }
            mbar_wait(mbar, q & 1u);
            uint32_t r0, r1, r2, r3, r4, gapA, gapB, gapC;
            {
                lds128(stage + t * 16, r0, r1, r2, r3);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r4) : "r"(stage + t * 16 + 16));
                if constexpr (kNB == 8) {
                    const uint32_t gb0 = stage + kChunkBytes + ((t * 10) >> 3);
                    // gaps of chunks 2t, 2t+1 and 2t+2 (the next tile's first for t = 127: the stage
                    // holds 16 bytes of gaps past the tile) start at bit 10t
                    const uint32_t h0 = ld8(gb0), h1 = ld8(gb0 + 1), h2 = ld8(gb0 + 2), h3 = ld8(gb0 + 3);
                    const uint32_t g32 = (h0 << 24) | (h1 << 16) | (h2 << 8) | h3;
                    const uint32_t g15 = (g32 >> (17u - ((t * 10) & 7u))) & 32767u;
                    gapA = g15 >> 10;
                    gapB = (g15 >> 5) & 31u;
                    gapC = g15 & 31u;
                } else {
                    // gaps of chunks t and t+1 start at bit 5t (gapB: the end of this lane's chain)
                    const uint32_t gb0 = stage + kChunkBytes + ((t * 5) >> 3);
                    const uint32_t g24 = (ld8(gb0) << 16) | (ld8(gb0 + 1) << 8) | ld8(gb0 + 2);
                    const uint32_t g10 = (g24 >> (14u - ((t * 5) & 7u))) & 1023u;
                    gapA = g10 >> 5;
                    gapB = g10 & 31u;
                    gapC = 0;
                }
            }
            const uint32_t lo = min(clo, N);
            const uint32_t hi = min(max(min(chi, N), lo), lo + 8 * kN * kT);
            const uint32_t W0 = bswap32(r0), W1 = bswap32(r1), W2 = bswap32(r2), W3 = bswap32(r3),
                           W4 = bswap32(r4);

            uint32_t cntA, cntB;
            if constexpr (kNB == 8) {
                if (!safe) {
                    // ---- single decode pass into the private slots (chains A: [gapA, 64), B: [64+gapB, 128))
                    // exact chain ends when the next chunk's gap marks a code start (every tile but the
                    // one holding the tensor's last code): A = [gapA, 64 + gapB), B = [64 + gapB, 128 + gapC),
                    // enforced by one-bits after the end; otherwise [.., 64) / [.., 128) + walk back
                    const bool exact = long_codes && hi < N;
                    const uint32_t limA = exact ? 64u + gapB - gapA : 64u - gapA;
                    const uint32_t limB = exact ? 64u + gapC - gapB : 64u - gapB;
                    uint32_t aA = W0, bA = W1, cA = exact ? W2 | (0xFFFFFFFFu >> gapB) : W2;
                    uint32_t aB = W2, bB = W3, cB = exact ? W4 | (0xFFFFFFFFu >> gapC) : W4;
                    shift96_ones(aA, bA, cA, gapA);
                    shift96_ones(aB, bB, cB, gapB);
                    uint32_t xA = kXEnd - limA, xB = kXEnd - limB;   // see kXEnd
                    Slot oA, oB;
                    slot_init(oA, slotA);
                    slot_init(oB, slotB);
                    uint32_t hA = 1, hB = 1;
                    auto step = [&]() {
                        uint32_t lA, lB;
                        lds64(t12_addr(aA, tab, K_ROW, K_TOP, K_ENT), lA, hA);
                        lds64(t12_addr(aB, tab, K_ROW, K_TOP, K_ENT), lB, hB);
                        pack(oA, lA, hA, K_S24);
                        pack(oB, lB, hB, K_S24);
                        xA += hA;
                        xB += hB;
                        shift96_ones(aA, bA, cA, hA);
                        shift96_ones(aB, bB, cB, hB);
                    };
    #pragma unroll
                    for (int u = 0; u < kFirst; u++) step();
                    for (;;) {
                        const bool actA = (xA & kXEnd) == 0, actB = (xB & kXEnd) == 0;
                        if (!__any_sync(FULL, actA || actB)) break;
                        // an escape row (a code longer than 12 bits) has hi == 0
                        const bool escA = actA && hA == 0, escB = actB && hB == 0;
                        if (__any_sync(FULL, escA || escB)) {
                            if (escA) {
                                uint32_t len;
                                const uint32_t r = to_stored<kVF>(walk(aA, len));
                                pack(oA, r & 0xFFu, 8u << 24, K_S24);
                                xA += len;
                                shift96_long_ones(aA, bA, cA, len);
                            }
                            if (escB) {
                                uint32_t len;
                                const uint32_t r = to_stored<kVF>(walk(aB, len));
                                pack(oB, r & 0xFFu, 8u << 24, K_S24);
                                xB += len;
                                shift96_long_ones(aB, bB, cB, len);
                            }
                        }
                        // one step; a chain past its end skips the lookup: lo = hi = 0 leave its state unchanged
                        uint32_t lA = 0, lB = 0;
                        hA = 0;
                        hB = 0;
                        lds64_if(t12_addr(aA, tab, K_ROW, K_TOP, K_ENT), lA, hA, actA);
                        lds64_if(t12_addr(aB, tab, K_ROW, K_TOP, K_ENT), lB, hB, actB);
                        pack(oA, lA, hA, K_S24);
                        pack(oB, lB, hB, K_S24);
                        xA += hA;
                        xB += hB;
                        shift96_ones(aA, bA, cA, hA);
                        shift96_ones(aB, bB, cB, hB);
                    }
                    slot_flush(oA);                                               // the last partial word
                    slot_flush(oB);
                    uint32_t nA = slot_bytes(oA);
                    uint32_t nB = slot_bytes(oB);
                    // drop the codes decoded past each chain's end (they start at or after it)
                    if (!exact) {
                        uint32_t offA = xA & kXMask;   // kXEnd - limA + consumed
                        while (nA > 0) {
                            const uint32_t j = nA - 1;
                            const uint32_t l = ld8(rlenb + ld8(slotA + (j >> 2) * 128u + (j & 3u)));
                            if (offA - l < kXEnd) break;
                            offA -= l;
                            nA--;
                        }
                        uint32_t offB = xB & kXMask;
                        while (nB > 0) {
                            const uint32_t j = nB - 1;
                            const uint32_t l = ld8(rlenb + ld8(slotB + (j >> 2) * 128u + (j & 3u)));
                            if (offB - l < kXEnd) break;
                            offB -= l;
                            nB--;
                        }
                    }
                    cntA = nA;
                    cntB = nB;
                } else {
                    // ---- count-only pass, one code at a time (1-bit codewords)
                    auto count_chain = [&](uint32_t a, uint32_t bb, uint32_t c, uint32_t off, uint32_t lim) {
                        uint32_t n = 0;
                        while (off < lim) {
                            uint32_t el, eh, len;
                            lds64(t12_addr(a, tab, K_ROW, K_TOP, K_ENT), el, eh);
                            if ((eh & 0xFFFFu) != 0) len = ld8(rlenb + (el & 0xFFu));
                            else walk(a, len);
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
            } else if (!safe) {
                // ---- one chain per lane: [gapA, 128 + gapB) exact, else [gapA, 128) + walk back
                const bool exact = long_codes && hi < N;
                const uint32_t limA = exact ? 128u + gapB - gapA : 128u - gapA;
                uint32_t a = W0, b1 = W1, c = W2, d = W3, e = exact ? W4 | (0xFFFFFFFFu >> gapB) : W4;
                shift160_ones(a, b1, c, d, e, gapA);
                uint32_t xA = kXEnd - limA;
                Slot oA;
                slot_init(oA, slotA);
                uint32_t hA = 1;
                auto step = [&]() {
                    uint32_t lA;
                    lds64(t12_addr(a, tab, K_ROW, K_TOP, K_ENT), lA, hA);
                    pack(oA, lA, hA, K_S24);
                    xA += hA;
                    shift160_ones(a, b1, c, d, e, hA);
                };
#pragma unroll
                for (int u = 0; u < 2 * kFirst; u++) step();
                for (;;) {
                    const bool actA = (xA & kXEnd) == 0;
                    if (!__any_sync(FULL, actA)) break;
                    const bool escA = actA && hA == 0;           // an escape row (a code > 12 bits)
                    if (__any_sync(FULL, escA)) {
                        if (escA) {
                            uint32_t len;
                            const uint32_t r = to_stored<kVF>(walk(a, len));
                            pack(oA, r & 0xFFu, 8u << 24, K_S24);
                            xA += len;
                            shift160_long_ones(a, b1, c, d, e, len);
                        }
                    }
                    uint32_t lA = 0;
                    hA = 0;
                    lds64_if(t12_addr(a, tab, K_ROW, K_TOP, K_ENT), lA, hA, actA);
                    pack(oA, lA, hA, K_S24);
                    xA += hA;
                    shift160_ones(a, b1, c, d, e, hA);
                }
                slot_flush(oA);
                uint32_t nA = slot_bytes(oA);
                if (!exact) {
                    uint32_t offA = xA & kXMask;   // kXEnd - limA + consumed
                    while (nA > 0) {
                        const uint32_t j = nA - 1;
                        const uint32_t l = ld8(rlenb + ld8(slotA + (j >> 2) * 128u + (j & 3u)));
                        if (offA - l < kXEnd) break;
                        offA -= l;
                        nA--;
                    }
                }
                cntA = nA;
                cntB = 0;
            } else {
                // ---- count-only pass, one code at a time (1-bit codewords)
                uint32_t a = W0, b1 = W1, c = W2, d = W3, e = W4, off = gapA;
                shift160_long_ones(a, b1, c, d, e, gapA);
                uint32_t n = 0;
                while (off < 128u) {
                    uint32_t el, eh, len;
                    lds64(t12_addr(a, tab, K_ROW, K_TOP, K_ENT), el, eh);
                    if ((eh & 0xFFFFu) != 0) len = ld8(rlenb + (el & 0xFFu));
                    else walk(a, len);
                    n++;
                    off += len;
                    shift160_long_ones(a, b1, c, d, e, len);
                }
                cntA = n;
                cntB = 0;
            }
            const uint32_t cnt = cntA + cntB;

            // ---- exclusive scan of the counts over the tile: warp shuffles + 4 warp totals
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(FULL, incl, d);
                if (lane >= (uint32_t)d) incl += v;
            }
            const uint32_t ws = gbase + L::kGWsum + parity * (kWarps12 * 4);
            if (lane == 31) sts32(ws + wig * 4, incl);
            group_bar(g);                          // also: every thread has read this tile's stage
#if !defined(SP12_NO_PDL) && !defined(SP12_PDL_EARLY) && !defined(SP12_PDL_NOWAIT)   // NOWAIT: negative test only
            asm volatile("griddepcontrol.wait;" ::: "memory");   // before this tile's first global write
#endif
            parity ^= 1u;
            if (t == 0 && has_next) {
                if constexpr (kNB == 8) issue_tile(ts, b + kGroups12, stage, mbar);
                else issue_tile16(ts, b + kGroups12, stage, mbar);
            }
            uint32_t wpre = 0;
            {
                uint4 v;
                lds128(ws, v.x, v.y, v.z, v.w);
                wpre = (wig > 0 ? v.x : 0u) + (wig > 1 ? v.y : 0u) + (wig > 2 ? v.z : 0u);
            }
            const uint32_t wtot = __shfl_sync(FULL, incl, 31);
            const uint32_t lpos = incl - cnt;                                  // first output in the warp
            const uint32_t wbeg = lo + wpre;                                   // the warp's first output

            if (safe) {
                // direct mode: compose and store to HBM per code
                uint32_t p = wbeg + lpos;
                const uint32_t pend = min(p + cnt, hi);
                if constexpr (kNB == 8) {
#pragma unroll 1
                    for (int sub = 0; sub < 2; sub++) {
                        uint32_t a, bb, c;
                        if (sub) { a = W2; bb = W3; c = W4; shift96(a, bb, c, gapB); }
                        else { a = W0; bb = W1; c = W2; shift96(a, bb, c, gapA); }
                        uint32_t off = sub ? 64u + gapB : gapA;
                        const uint32_t lim_off = sub ? 128u : 64u;
                        while (p < pend && off < lim_off) {
                            uint32_t el, eh, len, sym;
                            lds64(t12_addr(a, tab, K_ROW, K_TOP, K_ENT), el, eh);
                            if ((eh & 0xFFFFu) != 0) { sym = from_stored<kVF>(el & 0xFFu); len = ld8(rlenb + (el & 0xFFu)); }
                            else sym = walk(a, len);
                            out[p] = (OutT)compose_vf(kF, sym, load_residual(kF, ts.packed_sign_mantissa, p, N));
                            p++;
                            off += len;
                            shift96_long(a, bb, c, len);
                        }
                    }
                } else {
                    uint32_t a = W0, b1 = W1, c = W2, d = W3, e = W4, off = gapA;
                    shift160_long_ones(a, b1, c, d, e, gapA);
                    while (p < pend && off < 128u) {
                        uint32_t el, eh, len, sym;
                        lds64(t12_addr(a, tab, K_ROW, K_TOP, K_ENT), el, eh);
                        if ((eh & 0xFFFFu) != 0) { sym = from_stored<kVF>(el & 0xFFu); len = ld8(rlenb + (el & 0xFFu)); }
                        else sym = walk(a, len);
                        out[p] = (OutT)compose_vf(kF, sym, load_residual(kF, ts.packed_sign_mantissa, p, N));
                        p++;
                        off += len;
                        shift160_long_ones(a, b1, c, d, e, len);
                    }
                }
                continue;
            }

            // ---- this warp's output range
            const uint32_t F = wbeg & ~15u;                                    // region byte of e: e - F
            const uint32_t ra = min(wbeg, hi), rb = min(wbeg + wtot, hi);
            // kU-word units [ua, ub) (16 bytes: 8 BF16/FP16 or 16 FP8 words) leave with one STG.128 each;
            // head [ra, ha) and tail [tb, rb) (< kU words each) one element per lane
            const uint32_t ua = vec_out ? (ra + kU - 1) / kU : 0, ub = vec_out ? max(rb / kU, ua) : 0;
            const uint32_t ha = vec_out ? min(ua * kU, rb) : rb, tb = vec_out ? max(ub * kU, ha) : rb;
            const uint32_t es = lane < 16 ? ra + lane : tb + (lane - 16);
            const bool edge = vec_out && (lane < 16 ? es < ha : es < rb);

            // ---- compaction of the slots into [F, ...) of the warp region (in place: load all first)
            if constexpr (kNB == 8) {
                {
                    uint32_t wa[8], wb[8];
    #pragma unroll
                    for (int k = 0; k < 8; k++) {
                        wa[k] = lds32(slotA + 128u * k);
                        wb[k] = lds32(slotB + 128u * k);
                    }
                    __syncwarp();
                    const uint32_t dA = wreg + (wbeg - F) + lpos, dB = dA + cntA;
                    compact_words(dA, wa, cntA);
                    compact_words(dB, wb, cntB);
                    __syncwarp();
    #ifndef SP12_BYTE_HEADS
                    // first partial word of a chain: its low bytes already hold the previous chain's tail
                    // (that chain's last word, written above), so one read-modify-write completes it when
                    // every chain of the warp has >= 4 codes (then no word holds bytes of 3 chains)
                    if (!__any_sync(FULL, cntA < 4u || cntB < 4u)) {
                        const uint32_t rA = dA & 3u, rB = dB & 3u;
                        if (rA) {
                            const uint32_t o = lds32(dA - rA);
                            sts32(dA - rA, (o & ((1u << (8 * rA)) - 1u)) | (wa[0] << (8 * rA)));
                        }
                        if (rB) {
                            const uint32_t o = lds32(dB - rB);
                            sts32(dB - rB, (o & ((1u << (8 * rB)) - 1u)) | (wb[0] << (8 * rB)));
                        }
                    } else
    #endif
                    {
                        compact_head(dA, wa[0], cntA);
                        compact_head(dB, wb[0], cntB);
                    }
                }
                __syncwarp();
            } else {
                uint32_t wa[16];
#pragma unroll
                for (int k = 0; k < 16; k++) wa[k] = lds32(slotA + 128u * k);
                __syncwarp();
                const uint32_t dA = wreg + (wbeg - F) + lpos;
                compact_words16(dA, wa, cntA);
                __syncwarp();
                if (!__any_sync(FULL, cntA < 4u)) {
                    const uint32_t rA = dA & 3u;
                    if (rA) {
                        const uint32_t o = lds32(dA - rA);
                        sts32(dA - rA, (o & ((1u << (8 * rA)) - 1u)) | (wa[0] << (8 * rA)));
                    }
                } else {
                    compact_head(dA, wa[0], cntA);
                }
                __syncwarp();
            }

            // ---- per-warp merge of [ra, rb): compose the words and store
            uint32_t a0, a1;
            if (sm_range(lo, hi, a0, a1)) {
                mbar_wait(smbar, qs & 1u);                                     // PackedSignMantissa staged
                qs++;
                // lane l stores units u0 + 32k: every STG.128 of the warp covers 512 contiguous bytes.
                // A warp range has <= 64 * 32 outputs (<= 257 units, <= 9 per lane); the unit stride is
                // an immediate offset of the loads and stores.
                if constexpr (kVF == DF11_VF_BF16) {
                    if (edge) out[es] = compose_r(ld8(wreg + (es - F)), ld8(smb + (es - a0)));
                    // warp-uniform trip count: every lane stores (ub - ua) / 32 units, lanes below
                    // (ub - ua) % 32 one more
                    const uint32_t nun = ub - ua, nfull = nun >> 5;
                    const uint32_t e0 = (ua + lane) << 3;
                    uint32_t sa = smb + (e0 - a0), xa = wreg + (e0 - F);
                    uint4 *op = reinterpret_cast<uint4 *>(out + e0);
                    auto unit = [&](uint32_t k) {
                        uint32_t s0, s1, x0, x1;
                        lds64(sa + 256u * k, s0, s1);
                        lds64(xa + 256u * k, x0, x1);
                        uint4 o;
                        compose4r(x0, s0, o.x, o.y);
                        compose4r(x1, s1, o.z, o.w);
                        op[32 * k] = o;
                    };
                    uint32_t k = 0;
                    for (; k + 4 <= nfull; k += 4) {
                        unit(k);
                        unit(k + 1);
                        unit(k + 2);
                        unit(k + 3);
                    }
                    for (; k < nfull; k++) unit(k);
                    if (lane < (nun & 31u)) unit(nfull);
                } else {
                    if constexpr (kVF == DF11_VF_FP16) {
                        // byte plane of output e at smb + e - a0; its 3 high bits at bit 3 e - 8 q0 of
                        // the staged 3-bit plane (R25)
                        const uint32_t q0 = (a0 / 8u * 3u) & ~15u;
                        if (edge)
                            out[es] = (OutT)compose_vf(kF, from_stored<kVF>(ld8(wreg + (es - F))),
                                                       (res_smem<3>(smb + kFp16HiOff, 3u * es - 8u * q0) << 8) |
                                                           ld8(smb + (es - a0)));
                        // warp-uniform trip count with the unit stride as immediate offsets (as for BF16):
                        // lane l composes units ua + l + 32k (FP8 lost 0.4-1.9 % with this form)
                        const uint32_t nun = ub - ua, nfull = nun >> 5;
                        const uint32_t e0b = (ua + lane) * kU;
                        const uint32_t sb0 = smb + (e0b - a0), hb0 = smb + kFp16HiOff + (e0b / 8u * 3u - q0);
                        const uint32_t xb = wreg + (e0b - F);
                        uint4 *opb = reinterpret_cast<uint4 *>(out + e0b);
                        auto unit = [&](uint32_t k) {       // units 32 apart: 256 words, 96 bytes of high bits
                            uint32_t x0, x1, s0, s1;
                            lds64(xb + 256u * k, x0, x1);
                            lds64(sb0 + 256u * k, s0, s1);
                            opb[32 * k] = unit_fp16(x0, x1, s0, s1, hb0 + 96u * k);
                        };
                        uint32_t k = 0;
                        for (; k + 4 <= nfull; k += 4) {
                            unit(k);
                            unit(k + 1);
                            unit(k + 2);
                            unit(k + 3);
                        }
                        for (; k < nfull; k++) unit(k);
                        if (lane < (nun & 31u)) unit(nfull);
                    } else {
                        // FP8: residual bits of output e at bit kRb * e - 8 * a0
                        if (edge)
                            out[es] = (OutT)compose_vf(kF, from_stored<kVF>(ld8(wreg + (es - F))),
                                                       res_smem<kRb>(smb, es * kRb - 8u * a0));
                        for (uint32_t u = ua + lane; u < ub; u += 32) {
                            const uint32_t e0 = u * kU;
                            const uint32_t o = smb + (e0 / 8u * kRb - a0), xa = wreg + (e0 - F);
                            uint4 v;
                            uint32_t x0, x1, x2, x3;
                            lds128(xa, x0, x1, x2, x3);
                            if constexpr (kVF == DF11_VF_FP8_E4M3) {
                                uint32_t r0, r1;
                                lds64(o, r0, r1);                               // 16 nibbles
                                v.x = quad_e4m3<0x1100u>(r0, x0);
                                v.y = quad_e4m3<0x3322u>(r0, x1);
                                v.z = quad_e4m3<0x1100u>(r1, x2);
                                v.w = quad_e4m3<0x3322u>(r1, x3);
                            } else {                                            // E5M2: 48 bits at o (even)
                                const uint32_t base = o & ~3u, sh = (o & 3u) * 8u;
                                const uint32_t B0 = bswap32(lds32(base)), B1 = bswap32(lds32(base + 4));
                                const uint32_t H0 = __funnelshift_l(B1, B0, sh), H1 = B1 << sh;
                                v.x = quad_e5m2(H0 >> 20, x0);
                                v.y = quad_e5m2((H0 >> 8) & 0xFFFu, x1);
                                v.z = quad_e5m2(__funnelshift_l(H1, H0, 24) >> 20, x2);
                                v.w = quad_e5m2((H1 >> 16) & 0xFFFu, x3);
                            }
                            *reinterpret_cast<uint4 *>(out + e0) = v;
                        }
                    }
                }
#ifndef SP12_SM_BARRIER
                // the last warp done with this tile's buffer stages the group's next tile into it.
                // Ordering: each warp's reads of the buffer are complete before its
                // lane 0 passes __syncwarp; the warp's fence + relaxed atomic increment publish that, the
                // last incrementer's fence orders all four warps' reads before its proxy fence, and
                // fence.proxy.async orders those generic-proxy reads before the async-proxy TMA write.
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    uint32_t done;
                    asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(done) : "r"(mcnt) : "memory");
                    if (done == kWarps12 - 1) {
                        sts32(mcnt, 0);
                        __threadfence_block();
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        if (has_next) stage_sm(nlo, nhi);
                    }
                }
#else
                // A/B reference for the race evidence: a group barrier instead of the atomic hand-off
                group_bar(g);
                if (t == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (has_next) stage_sm(nlo, nhi);
                }
#endif
            } else {
                if constexpr (kVF == DF11_VF_BF16) {
                    if (edge) out[es] = compose_r(ld8(wreg + (es - F)), __ldg(ts.packed_sign_mantissa + es));
                    for (uint32_t u = ua + lane; u < ub; u += 32) {
                        const uint32_t e0 = u << 3;
                        const uint2 sm = __ldg(psm2 + u);
                        uint32_t x0, x1;
                        lds64(wreg + (e0 - F), x0, x1);
                        uint4 o0;
                        compose4r(x0, sm.x, o0.x, o0.y);
                        compose4r(x1, sm.y, o0.z, o0.w);
                        *reinterpret_cast<uint4 *>(out + e0) = o0;
                    }
                    if (!vec_out)                                              // unaligned output: scalar
                        for (uint32_t e = ra + lane; e < rb; e += 32)
                            out[e] = compose_r(ld8(wreg + (e - F)), __ldg(ts.packed_sign_mantissa + e));
                } else {
                    // residuals of a tile above the SMEM cap (or an unaligned output): per element
                    for (uint32_t e = ra + lane; e < rb; e += 32)
                        out[e] = (OutT)compose_vf(kF, from_stored<kVF>(ld8(wreg + (e - F))),
                                                  load_residual(kF, ts.packed_sign_mantissa, e, N));
                }
                if (t == 0 && has_next) stage_sm(nlo, nhi);
                __syncwarp();                  // the region's reads are done before the next tile's slots
            }
        }
        seg_begin = seg_end;
    }
#undef K_ROW
#undef K_TOP
#undef K_ENT
#undef K_S24
}

uint32_t g_sp12_attr_set[64];   // bit (b8 ? 0 : 8) + (n16 ? 4 : 0) + vf: smem attribute set

template <uint32_t kNB, uint32_t kVF, bool kB8>
cudaError_t launch_one(const Batch &bt, int device, uint32_t grid, cudaStream_t stream) {
    constexpr uint32_t bit = 1u << ((kB8 ? 0 : 8) + (kNB == 16 ? 4 : 0) + kVF);
    if (device >= 0 && device < 64 && !(g_sp12_attr_set[device] & bit)) {
        cudaError_t e = cudaFuncSetAttribute(sp12_kernel<kNB, kVF, kB8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)Lay12<kVF>::kSmem);
        if (e != cudaSuccess) return e;
        g_sp12_attr_set[device] |= bit;
    }
#ifndef SP12_NO_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kCta12);
    cfg.dynamicSmemBytes = Lay12<kVF>::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sp12_kernel<kNB, kVF, kB8>, bt);
#else
    sp12_kernel<kNB, kVF, kB8><<<grid, kCta12, Lay12<kVF>::kSmem, stream>>>(bt);
    return cudaGetLastError();
#endif
}

template <bool kB8>
cudaError_t launch_vf(const Batch &bt, int device, uint32_t grid, cudaStream_t stream, uint32_t key) {
    switch (key) {
        case 0: return launch_one<8, DF11_VF_BF16, kB8>(bt, device, grid, stream);
        case 1: return launch_one<8, DF11_VF_FP16, kB8>(bt, device, grid, stream);
        case 2: return launch_one<8, DF11_VF_FP8_E4M3, kB8>(bt, device, grid, stream);
        case 3: return launch_one<8, DF11_VF_FP8_E5M2, kB8>(bt, device, grid, stream);
        case 4: return launch_one<16, DF11_VF_BF16, kB8>(bt, device, grid, stream);
        case 5: return launch_one<16, DF11_VF_FP16, kB8>(bt, device, grid, stream);
        case 6: return launch_one<16, DF11_VF_FP8_E4M3, kB8>(bt, device, grid, stream);
        default: return launch_one<16, DF11_VF_FP8_E5M2, kB8>(bt, device, grid, stream);
    }
}

}  // namespace

uint32_t fast_grid(uint32_t total_tiles, int num_sms) {
    return min((uint32_t)num_sms, (total_tiles + kGroups12 - 1) / kGroups12);
}

// Tensors the product kernel decodes: the paper's format parameters (T = 256, n = 8) or
// T = 128, n = 16 (NEXT-4), any value format and LUT width b (FP16 up to ~3.1 G elements: 32-bit residual
// offsets), and the alignment its bulk copies need (stream, gaps and PackedSignMantissa 16-byte aligned,
// output aligned to its word size);
// df11_decompress_block_ex sends every other tensor to the Algorithm 1 kernel.
bool fast_supports(const df11_device_tensor &t) {
    // residual byte offsets are 32-bit in the kernel: R * roundup(N, 16) / 8 (+ padding) must fit
    const uint64_t res_bytes = (uint64_t)vf_of(t.value_format).R * ((t.num_elements + 15) & ~15ull) / 8 + 64;
    return ((t.T == kT && t.n == kN) || (t.T == 128 && t.n == 16)) && res_bytes < (1ull << 32) &&
           (reinterpret_cast<uintptr_t>(t.encoded_exponent) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(t.gaps) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(t.packed_sign_mantissa) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(t.out) & (vf_of(t.value_format).word_bytes - 1)) == 0;
}

// Launch for a batch whose tensors share n (8 with T = 256, or 16 with T = 128), the value format and
// whether their LUTs are the paper's byte tables.
cudaError_t launch_sp12(const Batch &bt, int device, cudaStream_t stream, uint64_t *launches) {
    if (bt.total_tiles == 0) return cudaSuccess;
    int num_sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const bool n16 = bt.t[0].n == 16;
    const uint32_t vf = bt.t[0].value_format;
    const uint32_t grid = bt.grid ? bt.grid
                                  : min((uint32_t)num_sms, (bt.total_tiles + kGroups12 - 1) / kGroups12);
    const uint32_t key = vf + (n16 ? 4u : 0u);
    e = lut_bits_of(bt.t[0]) == 8 ? launch_vf<true>(bt, device, grid, stream, key)
                                  : launch_vf<false>(bt, device, grid, stream, key);
    if (e == cudaSuccess && launches) (*launches)++;
    return e;
}

}  // namespace df11
