// decode_wt.cu — warp-per-format-block variant of the persistent sm_100a DF11 decode kernel
// (DESIGN.md §7).
//
// Same decode table, chains, slots, compaction and merge as decode_sp12.cu, but ONE warp owns a whole
// format block ("tile", T = 256 threads x n = 8 bytes): it walks the tile's 256 chunks as four
// quarters of 64 chunks (two chains per lane), and the output position of each quarter is the tile's
// BlockOutputPos plus the counts of the quarters before it, kept in a register.  No warp ever
// waits for another warp's counts, so there is no group barrier (Alg. 1's block-level scan, P:415-417,
// becomes a warp shuffle scan plus a running base).  Tiles are claimed dynamically from a per-CTA
// counter; the next tile's stream/gaps are copied by TMA into the warp's stage once the last quarter
// has read it, and its PackedSignMantissa range is prefetched into L2 (the merge reads it with LDG).
#include "t12_common.cuh"

namespace df11 {
namespace {

#ifndef WT_WARPS
#define WT_WARPS 32
#endif
constexpr uint32_t kW = WT_WARPS;                      // warps per CTA
constexpr uint32_t kCtaW = 32 * kW;
constexpr int kFirstW = 6;                             // decode steps before the first warp check
constexpr uint32_t kSubWW = 10;                        // slot words per chain: <= 36 codes incl. overshoot
constexpr uint32_t kRegW = 16 + 2 * kSubWW * 128;      // frame pad + lane-column slots of 2 chains
constexpr uint32_t kStageW = kChunkBytes + kGapBytes;  // a tile's stream (+16 spill) and gaps (+16)

constexpr uint32_t kOffTW = 0;
constexpr uint32_t kOffLutW = kOffTW + kT12Bytes;
constexpr uint32_t kOffLenW = kOffLutW + kLutSmem;
constexpr uint32_t kOffRLenW = kOffLenW + 256;
constexpr uint32_t kOffCtrW = kOffRLenW + 256;         // tile counter of the current segment
constexpr uint32_t kOffStgW = kOffCtrW + 16;           // [warps][kStageW]
constexpr uint32_t kOffRegW = kOffStgW + kW * kStageW; // [warps][kRegW]
constexpr uint32_t kOffMbarW = kOffRegW + kW * kRegW;  // [warps] stage mbarrier
constexpr uint32_t kSmemW = kOffMbarW + kW * 8;
static_assert(kOffStgW % 16 == 0 && kStageW % 16 == 0 && kOffRegW % 16 == 0 && kRegW % 16 == 0 &&
                  kOffMbarW % 8 == 0 && kOffCtrW % 16 == 0,
              "alignment");
static_assert(kSmemW <= 232448, "SMEM budget");
static_assert(kRegW >= 8192 / kW + 16, "first-code table scratch fits the warp regions");

__global__ void __launch_bounds__(kCtaW, 1) wt_kernel(const __grid_constant__ Batch bt) {
    const uint32_t tid = threadIdx.x;
    const uint32_t warp = tid >> 5, lane = tid & 31;
    const uint32_t FULL = 0xFFFFFFFFu;
#define K_ROW bt.kpow[0]   // 2^12: a >> 20
#define K_TOP bt.kpow[1]   // 2^4: a >> 28 (bank swizzle)
#define K_S24 bt.kpow[2]   // 2^8: >> 24
#define K_ENT bt.kpow[3]   // 8: entry bytes
    uint8_t *sb = smem_b();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_w);
    const uint32_t tab = sbase + kOffTW;
    const uint32_t wreg = sbase + kOffRegW + warp * kRegW;   // this warp's region
    const uint32_t stage = sbase + kOffStgW + warp * kStageW;
    const uint32_t mbar = sbase + kOffMbarW + warp * 8;
    uint32_t *ctr = smem_w + kOffCtrW / 4;
    const uint32_t slotA = wreg + 16u + lane * 4u, slotB = slotA + kSubWW * 128u;
    const uint32_t rlenb = sbase + kOffRLenW;

    const uint32_t total = bt.total_tiles;
    const uint32_t c_begin = bt.cta_ranges ? bt.cta_start[blockIdx.x]
                                           : (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t c_end = bt.cta_ranges ? bt.cta_start[blockIdx.x + 1]
                                         : (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    if (c_begin >= c_end) return;
    if (lane == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t q = 0;                                          // tiles staged into this warp's stage

    int ti_idx = tensor_of_tile(bt, c_begin);
    for (uint32_t seg_begin = c_begin; seg_begin < c_end; ti_idx++) {
        const df11_device_tensor &ts = bt.t[ti_idx];
        const uint32_t seg_end = min(c_end, bt.tile_start[ti_idx + 1]);
        const uint32_t base_tile = bt.tile_start[ti_idx] - bt.tile_off[ti_idx];
        if (seg_end <= seg_begin) continue;
        const uint32_t N = (uint32_t)ts.num_elements;
        const uint8_t *__restrict__ psm = ts.packed_sign_mantissa;

        // PackedSignMantissa [plo, phi), widened to 16 bytes, goes to L2 ahead of its merge
        auto prefetch_sm = [&](uint32_t plo, uint32_t phi) {
            const uint32_t a0 = plo & ~15u, a1 = (phi + 15u) & ~15u;
            if (a1 > a0) prefetch_l2(psm + a0, a1 - a0);
        };

        // =============================== T12 for this tensor (CTA-wide)
        __syncthreads();                                     // every warp is done with the last segment
        if (tid == 0) *ctr = seg_begin + kW;                 // tiles seg_begin + warp are claimed statically
        // each warp's first tile: its BlockOutputPos reads and stream copies overlap the table build
        uint32_t tile = seg_begin + warp;
        uint32_t nlo = 0, nhi = 0;
        if (tile < seg_end) {
            nlo = __ldg(ts.block_output_pos + tile - base_tile);
            nhi = __ldg(ts.block_output_pos + tile - base_tile + 1);
            if (lane == 0) issue_tile(ts, tile - base_tile, stage, mbar);
        }
        bool safe, lut_in_smem;
        const bool long_codes = build_t12<kCtaW>(ts, sb, sbase, kOffTW, kOffLutW, kOffLenW, kOffRLenW, kOffRegW,
                                                 tid, safe, lut_in_smem);
        const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k;
        const bool vec_out = ((reinterpret_cast<uintptr_t>(ts.out) & 15) == 0);
        const uint2 *__restrict__ psm2 = reinterpret_cast<const uint2 *>(psm);
        uint16_t *__restrict__ out = ts.out;
        auto walk = [&](uint32_t w, uint32_t &len) -> uint32_t {
            if (lut_in_smem) return lut_walk_smem(w, sbase + kOffLutW, sbase + kOffLenW, eb_bytes, kk, len);
            return lut_walk_global(w, ts, len);
        };

        // =============================== tiles of this warp
        while (tile < seg_end) {
            const uint32_t b = tile - base_tile;
            const uint32_t lo = min(nlo, N);
            const uint32_t hi = min(max(min(nhi, N), lo), lo + 8 * kN * kT);
            // exact chain ends when the next chunk's gap marks a code start (every tile but the one
            // holding the tensor's last code): one-bits after a chain's end stall it there
            const bool exact = long_codes && hi < N;
            uint32_t next = seg_end;
            mbar_wait(mbar, q & 1u);
            q++;
            uint32_t base = lo;                              // first output of the current quarter
#pragma unroll 1
            for (uint32_t r = 0; r < 4; r++) {
                // a quarter has at most 64 * 32 outputs: its PackedSignMantissa goes to L2 while it decodes
                if (lane == 0 && !safe) prefetch_sm(base, min(base + 64u * 32u, hi));
                // ---- the lane's chunks c = 64r + 2 lane (chain A) and c + 1 (chain B), 3 gaps
                const uint32_t cb = stage + (64u * r + 2u * lane) * kN;
                uint32_t r0, r1, r2, r3, r4;
                lds128(cb, r0, r1, r2, r3);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r4) : "r"(cb + 16));
                const uint32_t gb0 = stage + kChunkBytes + 40u * r + ((lane * 10u) >> 3);
                const uint32_t h0 = ld8(gb0), h1 = ld8(gb0 + 1), h2 = ld8(gb0 + 2), h3 = ld8(gb0 + 3);
                const uint32_t g32 = (h0 << 24) | (h1 << 16) | (h2 << 8) | h3;
                const uint32_t g15 = (g32 >> (17u - ((lane * 10u) & 7u))) & 32767u;
                const uint32_t gapA = g15 >> 10, gapB = (g15 >> 5) & 31u, gapC = g15 & 31u;
                const uint32_t W0 = bswap32(r0), W1 = bswap32(r1), W2 = bswap32(r2), W3 = bswap32(r3),
                               W4 = bswap32(r4);
                if (r == 3) {
                    // every lane holds its last words of the stage: claim the next tile and refill
                    __syncwarp();
                    uint32_t nt = 0;
                    if (lane == 0) nt = atomicAdd(ctr, 1u);
                    next = __shfl_sync(FULL, nt, 0);
                    if (next < seg_end) {
                        nlo = __ldg(ts.block_output_pos + next - base_tile);
                        nhi = __ldg(ts.block_output_pos + next - base_tile + 1);
                        if (lane == 0) issue_tile(ts, next - base_tile, stage, mbar);
                    }
                }

                uint32_t cntA, cntB;
                if (!safe) {
                    // ---- single decode pass into the private slots (chains A: [gapA, 64), B: [64+gapB,
                    // 128)); exact: A = [gapA, 64 + gapB), B = [64 + gapB, 128 + gapC)
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
                    for (int u = 0; u < kFirstW; u++) step();
                    for (;;) {
                        const bool actA = (xA & kXEnd) == 0, actB = (xB & kXEnd) == 0;
                        if (!__any_sync(FULL, actA || actB)) break;
                        // an escape row (a code longer than 12 bits) has hi == 0
                        const bool escA = actA && hA == 0, escB = actB && hB == 0;
                        if (__any_sync(FULL, escA || escB)) {
                            if (escA) {
                                uint32_t len;
                                const uint32_t rr = rot8(walk(aA, len));
                                pack(oA, rr & 0xFFu, 8u << 24, K_S24);
                                xA += len;
                                shift96_long_ones(aA, bA, cA, len);
                            }
                            if (escB) {
                                uint32_t len;
                                const uint32_t rr = rot8(walk(aB, len));
                                pack(oB, rr & 0xFFu, 8u << 24, K_S24);
                                xB += len;
                                shift96_long_ones(aB, bB, cB, len);
                            }
                        }
                        // one step; a chain past its end skips the lookup: lo = hi = 0 leave its state
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
                const uint32_t cnt = cntA + cntB;

                // ---- exclusive scan of the counts over the quarter: warp shuffles; the quarter's first
                // output is the tile's BlockOutputPos plus the earlier quarters' counts
                uint32_t incl = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t v = __shfl_up_sync(FULL, incl, d);
                    if (lane >= (uint32_t)d) incl += v;
                }
                const uint32_t wtot = __shfl_sync(FULL, incl, 31);
                const uint32_t lpos = incl - cnt;
                const uint32_t wbeg = base;
                base += wtot;

                if (safe) {
                    // direct mode: compose and store to HBM per code
                    uint32_t p = wbeg + lpos;
                    const uint32_t pend = min(p + cnt, hi);
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
                            if ((eh & 0xFFFFu) != 0) { sym = unrot8(el & 0xFFu); len = ld8(rlenb + (el & 0xFFu)); }
                            else sym = walk(a, len);
                            out[p] = compose(sym, __ldg(psm + p));
                            p++;
                            off += len;
                            shift96_long(a, bb, c, len);
                        }
                    }
                    continue;
                }

                // ---- this warp's output range [ra, rb) of the quarter: 8-element units [ua, ub) leave
                // with one STG.128 each, head [ra, ha) and tail [tb, rb) (< 8 each) one element per lane
                const uint32_t F = wbeg & ~15u;                                // region byte of e: e - F
                const uint32_t ra = min(wbeg, hi), rb = min(wbeg + wtot, hi);
                const uint32_t ua = vec_out ? (ra + 7) >> 3 : 0, ub = vec_out ? max(rb >> 3, ua) : 0;
                const uint32_t ha = vec_out ? min(ua << 3, rb) : rb, tb = vec_out ? max(ub << 3, ha) : rb;
                const uint32_t es = lane < 16 ? ra + lane : tb + (lane - 16);
                const bool edge = vec_out && (lane < 16 ? es < ha : es < rb);

                // ---- compaction of the slots into [F, ...) of the warp region (in place: load all first)
                {
                    uint32_t wa[8], wbv[8];
#pragma unroll
                    for (int k = 0; k < 8; k++) {
                        wa[k] = lds32(slotA + 128u * k);
                        wbv[k] = lds32(slotB + 128u * k);
                    }
                    __syncwarp();
                    const uint32_t dA = wreg + (wbeg - F) + lpos, dB = dA + cntA;
                    compact_words(dA, wa, cntA);
                    compact_words(dB, wbv, cntB);
                    __syncwarp();
                    // first partial word of a chain: its low bytes already hold the previous chain's
                    // tail, so one read-modify-write completes it when every chain of the warp has >= 4
                    // codes (then no word holds bytes of 3 chains)
                    if (!__any_sync(FULL, cntA < 4u || cntB < 4u)) {
                        const uint32_t rA = dA & 3u, rB = dB & 3u;
                        if (rA) {
                            const uint32_t o = lds32(dA - rA);
                            sts32(dA - rA, (o & ((1u << (8 * rA)) - 1u)) | (wa[0] << (8 * rA)));
                        }
                        if (rB) {
                            const uint32_t o = lds32(dB - rB);
                            sts32(dB - rB, (o & ((1u << (8 * rB)) - 1u)) | (wbv[0] << (8 * rB)));
                        }
                    } else {
                        compact_head(dA, wa[0], cntA);
                        compact_head(dB, wbv[0], cntB);
                    }
                }
                __syncwarp();

                // ---- merge of [ra, rb): compose BF16 with PackedSignMantissa (L2) and store
                // all of the lane's PackedSignMantissa loads go out first (a quarter has <= 257 units,
                // <= 9 per lane), then the compose + stores: one L2 round trip per quarter
                const uint32_t u0 = ua + lane;
                const uint32_t nu = ub > u0 ? (ub - u0 + 31u) >> 5 : 0u;
                uint2 sv[9];
#pragma unroll
                for (uint32_t k = 0; k < 9; k++)
                    if (k < nu) sv[k] = __ldg(psm2 + u0 + 32u * k);
                if (edge) out[es] = compose_r(ld8(wreg + (es - F)), __ldg(psm + es));
#pragma unroll
                for (uint32_t k = 0; k < 9; k++) {
                    if (k < nu) {
                        const uint32_t e0 = (u0 + 32u * k) << 3;
                        uint32_t x0, x1;
                        lds64(wreg + (e0 - F), x0, x1);
                        uint4 o0;
                        compose4r(x0, sv[k].x, o0.x, o0.y);
                        compose4r(x1, sv[k].y, o0.z, o0.w);
                        *reinterpret_cast<uint4 *>(out + e0) = o0;
                    }
                }
                if (!vec_out)                                                  // unaligned output: scalar
                    for (uint32_t e = ra + lane; e < rb; e += 32)
                        out[e] = compose_r(ld8(wreg + (e - F)), __ldg(psm + e));
                __syncwarp();                      // the region's reads are done before the next slots
            }
            tile = next;
        }
        seg_begin = seg_end;
    }
#undef K_ROW
#undef K_TOP
#undef K_ENT
#undef K_S24
}

int g_wt_attr_set[64];

}  // namespace

cudaError_t launch_wt(const Batch &bt, int device, cudaStream_t stream, uint64_t *launches) {
    if (bt.total_tiles == 0) return cudaSuccess;
    int num_sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    if (device >= 0 && device < 64 && !g_wt_attr_set[device]) {
        e = cudaFuncSetAttribute(wt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemW);
        if (e != cudaSuccess) return e;
        g_wt_attr_set[device] = 1;
    }
    const uint32_t grid = bt.grid ? bt.grid : min((uint32_t)num_sms, (bt.total_tiles + kW - 1) / kW);
    wt_kernel<<<grid, kCtaW, kSmemW, stream>>>(bt);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace df11
