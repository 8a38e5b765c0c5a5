// decode_fast.cu — persistent sm_100a DF11 decode kernel (format T = 256, n = 8; narrow or wide LUTs).
//
// Same result as Algorithm 1: the codewords that start in each 8-byte chunk are
// counted (phase 1), a block-level exclusive scan turns counts into output positions, the
// chunks are re-decoded into an SRAM exponent buffer (phase 2) and BF16 leaves with coalesced stores
// (P:150).  Re-designed for B200:
//
//  * Persistent CTAs (one per SM, 1024 threads) = 8 groups of 128 threads; group g of CTA c walks the
//    format blocks ("tiles") of a contiguous range.  A thread decodes TWO adjacent chunks of its tile
//    as one 128-bit stream starting at the first chunk's gap (the second gap is implied), which
//    halves per-thread bookkeeping and evens out the per-lane work (warp lockstep).
//  * Derived decode tables are built in SMEM once per (CTA, tensor) from the format's hierarchical
//    LUTs.  For every R-bit prefix (R = 9):
//      T1 = consumed | count << 8 | startmask << 23        (phase 1; every complete code in R bits)
//      T2 = s0 | s1 << 8 | s2 << 16 | consumed << 24 | count << 29   (phase 2; up to 3 exponents)
//    T1/T2 are replicated 32x with lane-private banks (word = prefix*32 + lane): conflict-free LDS.
//    A prefix whose first code is longer than R bits (~0.1 % of codes on LLM-like weights) is an
//    "escape" row: its entry advances nothing, the thread stalls on it and a warp-uniform check every
//    4 steps resolves it through a second-level table (next 9 bits -> symbol, length) built for up to
//    8 escape rows, or, for longer codes, through the paper's LUT walk.
//  * The decode window is the top word of a 96-bit bit buffer shifted by the consumed bits and
//    refilled at the warp checks; field extraction uses IMAD.HI so the ALU and FMA pipes share the
//    work.  Phase 1 keeps (bit offset | count << 8) in one register and adds the T1 entry to it.
//  * EncodedExponent chunks and gaps of the next tile are staged by TMA (cp.async.bulk + mbarrier)
//    while the current tile decodes; EncodedExponent is read from HBM exactly once.
//  * One named barrier per tile (the scan).  Each warp then merges its own contiguous output range:
//    16 elements per lane-step, LDS.128 exponents + LDG.128 sign/mantissa (prefetched before phase
//    2) -> PRMT sign-replicate compose -> 2x 128-bit stores.  Tiles whose outputs exceed the SMEM
//    buffer (extremely compressible tensors) are written directly to HBM instead.
#include "fast_helpers.cuh"

namespace df11 {
namespace {

#ifndef DF11_STEPS_FIRST
#define DF11_STEPS_FIRST 4
#endif
#ifndef DF11_STEPS_EACH
#define DF11_STEPS_EACH 2
#endif
constexpr int kStepsFirst = DF11_STEPS_FIRST;   // decode steps before the first warp check
constexpr int kStepsEach = DF11_STEPS_EACH;     // decode steps between later warp checks
#ifndef DF11_GROUPS
#define DF11_GROUPS 8
#endif
constexpr uint32_t kGroups = DF11_GROUPS;    // tile groups (of kLanes threads) per CTA
constexpr uint32_t kCta = kLanes * kGroups;  // 1024 threads by default
constexpr uint32_t kWarps = kLanes / 32;   // 4 warps per group
constexpr uint32_t kBits = 8 * kN * kCpl;  // 128 bits decoded per lane
constexpr uint32_t kR = 9;                 // root bits of the derived tables
constexpr uint32_t kRows = 1u << kR;
constexpr uint32_t kTabWords = kRows * 32; // 32 lane replicas
constexpr uint32_t kEscRows = 8;           // escape rows with a second-level table
constexpr uint32_t kR2 = 9;                // bits resolved by the second level
constexpr uint32_t kLutSmem = 8192;        // format LUTs copied when they fit
constexpr uint32_t kExpBuf = 8304;         // per-group exponent buffer (bytes)
constexpr uint32_t kCap = kExpBuf - 32;    // max outputs per tile through SMEM (else direct mode)

// SMEM layout (bytes)
constexpr uint32_t kOffT1 = 0;
constexpr uint32_t kOffT2 = kOffT1 + kTabWords * 4;
constexpr uint32_t kOffL2 = kOffT2 + kTabWords * 4;                 // uint16 [kEscRows][1 << kR2]
constexpr uint32_t kOffLut = kOffL2 + kEscRows * (1u << kR2) * 2;    // uint8/uint16 [k][256]
constexpr uint32_t kOffLen = kOffLut + kLutSmem;                     // CodeLengths[256]
constexpr uint32_t kOffWsum = kOffLen + 256;                         // [groups][2][kWarps] uint32
constexpr uint32_t kOffExp = kOffWsum + kGroups * 2 * kWarps * 4;    // [groups][kExpBuf]
constexpr uint32_t kOffStage = kOffExp + kGroups * kExpBuf;          // [groups][kStageBytes]
constexpr uint32_t kOffMbar = kOffStage + kGroups * kStageBytes;     // [groups] uint64
constexpr uint32_t kSmemBytes = kOffMbar + kGroups * 8;
static_assert(kOffExp % 16 == 0 && kExpBuf % 16 == 0 && kStageBytes % 16 == 0 && kOffStage % 16 == 0 &&
              kOffMbar % 8 == 0, "alignment");
static_assert(kSmemBytes <= 232448, "SMEM budget");

__global__ void __launch_bounds__(kCta, 1) fast_kernel(const __grid_constant__ Batch bt) {
    const uint32_t tid = threadIdx.x;
    const uint32_t g = tid / kLanes;
    const uint32_t t = tid % kLanes;
    const uint32_t lane = tid & 31, wig = t >> 5;
    const uint32_t FULL = 0xFFFFFFFFu;
    // IMAD multipliers from the constant bank (see Batch::kpow)
#define K_ROW bt.kpow[0]
#define K_128 bt.kpow[1]
#define K_S24 bt.kpow[2]
#define K_S8 bt.kpow[3]
#define K_S16 bt.kpow[4]
#define K_S29 bt.kpow[5]
#define K_HALF bt.kpow[6]
#define K_SH7 bt.kpow[7]
    uint8_t *sb = smem_b();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_w);
    const uint32_t t1_lane = sbase + kOffT1 + lane * 4u;         // row r at + r*128
    const uint32_t t2_lane = sbase + kOffT2 + lane * 4u;
    const uint32_t ebuf_off = kOffExp + g * kExpBuf;
    uint32_t *wsum = smem_w + kOffWsum / 4 + g * 2 * kWarps;
    const uint32_t stage = sbase + kOffStage + g * kStageBytes;
    const uint32_t mbar = sbase + kOffMbar + g * 8;

    const uint32_t total = bt.total_tiles;
    const uint32_t c_begin = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t c_end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    if (c_begin >= c_end) return;
    if (t == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t q = 0;                    // tiles consumed by this group (mbarrier phase = q & 1)
    uint32_t parity = 0;               // wsum double buffer

    int ti_idx = tensor_of_tile(bt, c_begin);
    for (uint32_t seg_begin = c_begin; seg_begin < c_end; ti_idx++) {
        const df11_device_tensor &ts = bt.t[ti_idx];
        const uint32_t seg_end = min(c_end, bt.tile_start[ti_idx + 1]);
        const uint32_t base_tile = bt.tile_start[ti_idx] - bt.tile_off[ti_idx];   // b = tile - base_tile
        if (seg_end <= seg_begin) continue;

        // =============================== derived tables for this tensor (CTA-wide)
        __syncthreads();
        const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k;
        const uint32_t lut_bytes = kk * 256u * eb_bytes;
        const bool lut_in_smem = lut_bytes <= kLutSmem;
        if (lut_in_smem)
            for (uint32_t i = tid; i < lut_bytes; i += kCta) sb[kOffLut + i] = __ldg(ts.luts + i);
        for (uint32_t i = tid; i < 256u; i += kCta) sb[kOffLen + i] = __ldg(ts.code_lengths + i);
        uint32_t *esc_mask = smem_w + kOffExp / 4;                 // scratch: exponent buffers are idle
        uint32_t *esc_row = esc_mask + kRows / 32;
        if (tid < kRows / 32) esc_mask[tid] = 0;
        __syncthreads();
        auto walk = [&](uint32_t w, uint32_t &len) -> uint32_t {
            if (lut_in_smem) return lut_walk_smem(w, sbase + kOffLut, sbase + kOffLen, eb_bytes, kk, len);
            return lut_walk_global(w, ts, len);
        };
        uint32_t row_e1 = 0, row_e2 = 0;
        bool row_esc = false;
        if (tid < kRows) {
            const uint32_t W = tid << (32 - kR);
            uint32_t s = 0, cnt = 0, mask = 0, cons = 0, syms = 0, c2 = 0, cons2 = 0;
            while (s < kR) {
                uint32_t len;
                const uint32_t sym = walk(W << s, len);
                if (len > kR - s) break;
                mask |= 1u << s;
                cnt++;
                s += len;
                cons = s;
                if (c2 < 3) { syms |= sym << (8 * c2); c2++; cons2 = s; }
            }
            row_esc = cnt == 0;
            row_e1 = cons | (cnt << 8) | (mask << 23);
            row_e2 = syms | (cons2 << 24) | (c2 << 29);
            if (row_esc) atomicOr(esc_mask + tid / 32, 1u << (tid % 32));
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
            for (uint32_t i = tid; i < (n_esc << kR2); i += kCta) {
                const uint32_t row = esc_row[i >> kR2], j = i & ((1u << kR2) - 1u);
                uint32_t len;
                const uint32_t sym = walk((row << (32 - kR)) | (j << (32 - kR - kR2)), len);
                l2[i] = len <= kR + kR2 ? (uint16_t)(sym | (len << 8)) : (uint16_t)0;
            }
        }
        __syncthreads();

        // resolve one code longer than R bits at the top of window a_ (escape row id from the entry)
        auto escape = [&](uint32_t a_, uint32_t id, uint32_t &len) -> uint32_t {
            if (id != 0) {
                uint32_t v;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v)
                             : "r"(sbase + kOffL2 + (((id - 1) << kR2) + ((a_ >> (32 - kR - kR2)) & ((1u << kR2) - 1u))) * 2));
                if (v >> 8) { len = v >> 8; return v & 0xFFu; }
            }
            return walk(a_, len);
        };
        // packed form for the hot loops: sym | len << 8 (second-level table; the walk only on a miss)
        auto escape_packed = [&](uint32_t a_, uint32_t id) -> uint32_t {
            uint32_t v = 0;
            if (id != 0)
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v)
                             : "r"(sbase + kOffL2 + (((id - 1) << kR2) + ((a_ >> (32 - kR - kR2)) & ((1u << kR2) - 1u))) * 2));
            if ((v >> 8) == 0) {                                       // rare: code longer than kR + kR2
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

        // =============================== tiles of this group
        uint32_t tile = seg_begin + g;
        if (t == 0 && tile < seg_end) issue_tile(ts, tile - base_tile, stage, mbar);
        uint32_t nlo = 0, nhi = 0;
        if (tile < seg_end) {
            nlo = __ldg(ts.block_output_pos + tile - base_tile);
            nhi = __ldg(ts.block_output_pos + tile - base_tile + 1);
        }
        // sign/mantissa bytes of a tile -> L2 ahead of its merge (clipped, 16-byte granular)
        auto prefetch_sm = [&](uint32_t plo, uint32_t phi) {
            const uint32_t a0 = min(plo, N) & ~15u, a1 = (min(max(phi, plo), N) + 15u) & ~15u;
            if (a1 > a0) prefetch_l2(ts.packed_sign_mantissa + a0, a1 - a0);
        };
        if (t == 0 && tile < seg_end) prefetch_sm(nlo, nhi);
        for (; tile < seg_end; tile += kGroups, q++) {
            const uint32_t b = tile - base_tile;
            const uint32_t clo = nlo, chi = nhi;
            const bool has_next = tile + kGroups < seg_end;
            if (has_next) {                                                    // prefetch next BlockOutputPos
                nlo = __ldg(ts.block_output_pos + b + kGroups);
                nhi = __ldg(ts.block_output_pos + b + kGroups + 1);
            }
            mbar_wait(mbar, q & 1u);
            // this lane's 20 stream bytes (chunks 2t, 2t+1 + spill) and both chunks' gaps
            uint32_t r0, r1, r2, r3, r4, gapA, gapB;
            {
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(stage + t * 16));
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r4) : "r"(stage + t * 16 + 16));
                // 10 gap bits of chunks 2t, 2t+1 start at bit 10t: read the aligned 16-bit window
                uint32_t h0, h1, h2;
                const uint32_t gb0 = stage + kChunkBytes + ((t * 10) >> 3);
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(h0) : "r"(gb0));
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(h1) : "r"(gb0 + 1));
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(h2) : "r"(gb0 + 2));
                const uint32_t g24 = (h0 << 16) | (h1 << 8) | h2;                // bit 10t at bit 23-(10t&7)
                const uint32_t g10 = (g24 >> (14u - ((t * 10) & 7u))) & 1023u;
                gapA = g10 >> 5;
                gapB = g10 & 31u;
            }
            const uint32_t lo = min(clo, N);
            const uint32_t hi = min(max(min(chi, N), lo), lo + 8 * kN * kT);
            const uint32_t f = lo & ~15u;                                      // 16-element frame
            const bool direct = hi - lo > kCap;                                // group-uniform
            const uint32_t W0 = bswap32(r0), W1 = bswap32(r1), W2 = bswap32(r2), W3 = bswap32(r3),
                           W4 = bswap32(r4);

            // ---- phase 1: count the codes that start in chunk 2t ("A": bits [gapA, 64)) and in chunk
            // 2t+1 ("B": bits [64+gapB, 128)) as two independent chains interleaved step by step
            // (2x instruction-level parallelism); each fits a 96-bit bit buffer.
            uint32_t aA = W0, bA = W1, cA = W2, aB = W2, bB = W3, cB = W4;
            shift96(aA, bA, cA, gapA);
            shift96(aB, bB, cB, gapB);
            uint32_t accA = gapA, accB = 64u + gapB, eA1 = 1, eB1 = 1;          // acc = offset | count << 8
            // lockstep schedule: 4 steps, then a warp check (end / escapes) every 2 steps -- a chain
            // needs ~8.2 lookups and the warp waits for its slowest lane, so checking every 4 steps
            // wasted ~25 % of the steps
            auto p1_step = [&]() {
                const uint32_t eA = lds32(madlo(mulhi(aA, K_ROW), K_128, t1_lane));
                    const uint32_t eB = lds32(madlo(mulhi(aB, K_ROW), K_128, t1_lane));
                p1_apply<0xC0u>(accA, eA1, eA);                                // offset < 64
                p1_apply<0x80u>(accB, eB1, eB);                                // offset < 128
                shift96(aA, bA, cA, eA);                                       // e & 31 = consumed bits
                shift96(aB, bB, cB, eB);
            };
#pragma unroll
            for (int u = 0; u < kStepsFirst; u++) p1_step();
            for (;;) {
                const bool actA = (accA & 0xC0u) == 0, actB = (accB & 0x80u) == 0;
                if (!__any_sync(FULL, actA || actB)) break;
                const bool escA = actA && (eA1 & 0x7FFFFFu) == 0, escB = actB && (eB1 & 0x7FFFFFu) == 0;
                if (__any_sync(FULL, escA || escB)) {                          // codes longer than R bits
                    const uint32_t vA = escA ? escape_packed(aA, eA1 >> 23) : 0u;
                    const uint32_t vB = escB ? escape_packed(aB, eB1 >> 23) : 0u;
                    if (escA) {
                        eA1 = 0;                                               // exactly one code: no fixup
                        accA += (vA >> 8) + (1u << 8);
                        shift96_long(aA, bA, cA, vA >> 8);
                    }
                    if (escB) {
                        eB1 = 0;
                        accB += (vB >> 8) + (1u << 8);
                        shift96_long(aB, bB, cB, vB >> 8);
                    }
                }
#pragma unroll
                for (int u = 0; u < kStepsEach; u++) p1_step();
            }
            // each chain's last T1 group may hold complete codes starting past its end: not ours
            uint32_t cntA = (accA >> 8) & 0xFFu, cntB = (accB >> 8) & 0xFFu;
            if ((eA1 & 0x7FFFFFu) != 0) {
                const uint32_t last = (accA & 0xFFu) - (eA1 & 0xFu);
                cntA -= __popc((eA1 >> 23) >> min(64u - last, 31u));
            }
            if ((eB1 & 0x7FFFFFu) != 0) {
                const uint32_t last = (accB & 0xFFu) - (eB1 & 0xFu);
                cntB -= __popc((eB1 >> 23) >> min(kBits - last, 31u));
            }
            const uint32_t cnt = cntA + cntB;

            // ---- exclusive scan of the counts over the tile: warp shuffles + 4 warp totals
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(FULL, incl, d);
                if (lane >= (uint32_t)d) incl += v;
            }
            uint32_t *ws = wsum + parity * kWarps;
            if (lane == 31) ws[wig] = incl;
            group_bar(g);                          // also: every thread has read this tile's stage
            parity ^= 1u;
            if (t == 0 && has_next) {
                issue_tile(ts, b + kGroups, stage, mbar);
                prefetch_sm(nlo, nhi);                                         // next tile's sign/mantissa
            }
            uint32_t wpre = 0;
            {
                const uint4 v = *reinterpret_cast<const uint4 *>(ws);
                wpre = (wig > 0 ? v.x : 0u) + (wig > 1 ? v.y : 0u) + (wig > 2 ? v.z : 0u);
            }
            const uint32_t wtot = __shfl_sync(FULL, incl, 31);
            const uint32_t pos0 = wpre + incl - cnt;                           // this lane's first output
            // this warp's output range [ra, rb) (absolute elements), clipped to the tile
            const uint32_t ra = min(lo + wpre, hi), rb = min(lo + wpre + wtot, hi);
            // full 16-element groups [ga, gb) take the vector path; the <= 15 + 15 edge elements
            // [ra, ha) and [tb, rb) are shared with the neighbouring warps and go one per lane
            const bool vec = vec_out && !direct;
            const uint32_t ga = vec ? (ra + 15) >> 4 : 0, gb = vec ? max(rb >> 4, ga) : 0;
            const uint32_t ha = vec ? min(ga << 4, rb) : rb, tb = vec ? max(gb << 4, ha) : rb;
            uint4 smA = make_uint4(0, 0, 0, 0), smB = make_uint4(0, 0, 0, 0);
            if (ga + lane < gb) smA = __ldg(psm4 + ga + lane);                 // prefetch for the merge
            if (ga + lane + 32 < gb) smB = __ldg(psm4 + ga + lane + 32);
            const uint32_t es = lane < 16 ? ra + lane : tb + (lane - 16);      // this lane's edge element
            const bool edge = vec && (lane < 16 ? es < ha : es < rb);
            uint32_t sm1 = 0;
            if (edge) sm1 = __ldg(ts.packed_sign_mantissa + es);

            // ---- phase 2: re-decode with T2 (<= 3 exponents per lookup), chains A and B interleaved
            if (!direct) {
                const uint32_t wp0 = sbase + ebuf_off + (lo - f) + pos0;
                // A writes [wp0, wpAe), B writes [wpAe, wend); stores are predicated on the chain's end
                const uint32_t wpAe = wp0 + cntA, wend = wpAe + cntB;
                aA = W0; bA = W1; cA = W2; aB = W2; bB = W3; cB = W4;
                shift96(aA, bA, cA, gapA);
                shift96(aB, bB, cB, gapB);
                uint32_t wA = wp0, wB = wpAe, eA2 = 1, eB2 = 1;
                auto p2_step = [&]() {
                    eA2 = lds32(madlo(mulhi(aA, K_ROW), K_128, t2_lane));
                    eB2 = lds32(madlo(mulhi(aB, K_ROW), K_128, t2_lane));
                    sts8_if<0>(wA, eA2, wA, wpAe);
                    sts8_if<1>(wA, mulhi(eA2, K_S8), wA, wpAe - 1);
                    sts8_if<2>(wA, mulhi(eA2, K_S16), wA, wpAe - 2);
                    sts8_if<0>(wB, eB2, wB, wend);
                    sts8_if<1>(wB, mulhi(eB2, K_S8), wB, wend - 1);
                    sts8_if<2>(wB, mulhi(eB2, K_S16), wB, wend - 2);
                    wA += eA2 >> 29;                                           // count (LEA.HI)
                    wB += eB2 >> 29;
                    shift96(aA, bA, cA, mulhi(eA2, K_S24));                    // (e >> 24) & 31 = consumed
                    shift96(aB, bB, cB, mulhi(eB2, K_S24));
                };
#pragma unroll
                for (int u = 0; u < kStepsFirst; u++) p2_step();
                for (;;) {
                    const bool actA = wA < wpAe, actB = wB < wend;
                    if (!__any_sync(FULL, actA || actB)) break;
                    const bool escA = actA && eA2 < (1u << 24), escB = actB && eB2 < (1u << 24);
                    if (__any_sync(FULL, escA || escB)) {
                        const uint32_t vA = escA ? escape_packed(aA, eA2 & 0xFFu) : 0u;
                        const uint32_t vB = escB ? escape_packed(aB, eB2 & 0xFFu) : 0u;
                        if (escA) {
                            asm volatile("st.shared.u8 [%0], %1;" ::"r"(wA), "r"(vA) : "memory");
                            wA++;
                            shift96_long(aA, bA, cA, vA >> 8);
                        }
                        if (escB) {
                            asm volatile("st.shared.u8 [%0], %1;" ::"r"(wB), "r"(vB) : "memory");
                            wB++;
                            shift96_long(aB, bB, cB, vB >> 8);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kStepsEach; u++) p2_step();
                }
            } else {
                // direct mode (more than kCap outputs in this tile): compose and store to HBM per code
                uint32_t a = W0, bb = W1, c = W2;
                shift96(a, bb, c, gapA);
                uint32_t p = lo + pos0;
                const uint32_t pend = min(lo + pos0 + cnt, hi);
#pragma unroll 1
                for (int sub = 0; sub < 2; sub++) {
                    uint32_t off = sub ? 64u + gapB : gapA;
                    if (sub) { a = W2; bb = W3; c = W4; shift96(a, bb, c, gapB); }
                    const uint32_t lim_off = sub ? 128u : 64u;
                    while (p < pend && off < lim_off) {
                        uint32_t len;
                        const uint32_t e = lds32(madlo(mulhi(a, K_ROW), K_128, t2_lane));
                        uint32_t syms, n, consumed;
                        if (e >= (1u << 24)) { syms = e; n = e >> 29; consumed = (e >> 24) & 15u; }
                        else { syms = escape(a, e & 0xFFu, len); n = 1; consumed = len; }
                        // only the codes that start before the sub-stream end belong to it
                        uint32_t start = off;
                        for (uint32_t i = 0; i < n && p < pend && start < lim_off; i++, p++) {
                            out[p] = compose((syms >> (8 * i)) & 0xFFu, __ldg(ts.packed_sign_mantissa + p));
                            uint32_t l;
                            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(l) : "r"(sbase + kOffLen + ((syms >> (8 * i)) & 0xFFu)));
                            start += n == 1 ? consumed : l;
                        }
                        off += consumed;
                        shift96_long(a, bb, c, consumed);
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
                compose4(ex.x, sm.x, o0.x, o0.y, K_HALF, K_SH7);
                compose4(ex.y, sm.y, o0.z, o0.w, K_HALF, K_SH7);
                compose4(ex.z, sm.z, o1.x, o1.y, K_HALF, K_SH7);
                compose4(ex.w, sm.w, o1.z, o1.w, K_HALF, K_SH7);
                uint4 *dst = reinterpret_cast<uint4 *>(out + e0);
                dst[0] = o0;
                dst[1] = o1;
            }
            if (!vec_out && !direct)                                          // unaligned output: scalar
                for (uint32_t e = ra + lane; e < rb; e += 32)
                    out[e] = compose(ebf[e - f], __ldg(ts.packed_sign_mantissa + e));
        }
        seg_begin = seg_end;
    }
}

int g_attr_set[64];

}  // namespace

uint32_t fast_grid(uint32_t total_tiles, int num_sms) {
    return min((uint32_t)num_sms, (total_tiles + kGroups - 1) / kGroups);
}

bool fast_supports(const df11_device_tensor &t) {
    return t.T == kT && t.n == kN &&
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
    const uint32_t grid = bt.grid ? bt.grid : min((uint32_t)num_sms, (bt.total_tiles + kGroups - 1) / kGroups);
    fast_kernel<<<grid, kCta, kSmemBytes, stream>>>(bt);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace df11
