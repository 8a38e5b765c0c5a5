// decode_ws.cu — A/B experiment, not part of libdf11.so (measured -3 %: DESIGN.md §7 "Experiments that did
// not pay"; to rebuild it, copy it back to csrc/ and dispatch to launch_ws in api.cu under DF11_WS=1).
// A warp-specialised form of the product
// kernel for BF16, T = 256, n = 8, byte tables.  Same per-tile work as sp12_kernel (decode_sp12.cu), split
// over two roles so that neither carries the other's live state:
//   decode warps (4 per group): stage wait -> chains into double-buffered private slots -> counts
//   merge warps  (4 per group): counts -> scan -> compaction of the slots -> merge with the TMA-staged
//                                sign/mantissa bytes -> 128-bit stores
// The roles hand tiles over through SMEM with mbarriers (FULL: slots + counts written; EMPTY: slots read).
// Four groups of 256 threads per CTA.  Tensors with a 1-bit code (the count + direct path) are not
// handled: the kernel traps (the launcher only selects it under the A/B knob).
#include "t12_common.cuh"
// Register redistribution knobs (round-2 follow-up, profiles/r02_ws_setmaxnreg_ab.log): -DWS_DEC_REGS=R /
// -DWS_MRG_REGS=R make the decode / merge warpgroups setmaxnreg to R on entry to their role and back to
// WS_BASE_REGS (the kernel's register target, 64 at 1 024 threads) before the roles rejoin; -DWS_GROUPS=3
// gives 768 threads.  ptxas only accepts setmaxnreg here with the LUT walk inlined (a CALL inside a
// setmaxnreg region fails register allocation).  Measured: 72 / 56 registers -1.4 %, 768 threads with
// 96 / 64 -6 % against the plain split (itself -3 % against the product kernel).
#ifndef WS_GROUPS
#define WS_GROUPS 4
#endif
#ifndef WS_BASE_REGS
#define WS_BASE_REGS 64
#endif

namespace df11 {
namespace {

constexpr uint32_t kGroupsWS = WS_GROUPS;
constexpr uint32_t kCtaWS = 2 * kLanes * kGroupsWS;           // 1024
constexpr uint32_t kSubWS = 10;                               // slot words per chain (see decode_sp12.cu)
constexpr uint32_t kSlotWarp = 2 * kSubWS * 128;              // slots of one decode warp's 64 chains
constexpr uint32_t kRegWarp = 16 + kSlotWarp;                 // a merge warp's output region
constexpr uint32_t kOffT = 0;
constexpr uint32_t kOffLut = kOffT + kT12Bytes;
constexpr uint32_t kOffLen = kOffLut + kLutSmem;
constexpr uint32_t kOffRLen = kOffLen + 256;
constexpr uint32_t kOffGrp = kOffRLen + 256;
constexpr uint32_t kSmCapWS = 7168;
constexpr uint32_t gStage = 0;
constexpr uint32_t gSm = gStage + kStageBytes;
constexpr uint32_t gSlots = gSm + kSmCapWS;                   // [2][4 warps][kSlotWarp]
constexpr uint32_t gCnt = gSlots + 2 * 4 * kSlotWarp;         // [2][128] (cntA, cntB)
constexpr uint32_t gReg = gCnt + 2 * 128 * 8;                 // [4][kRegWarp]
constexpr uint32_t gWsum = gReg + 4 * kRegWarp;               // [2][4] warp totals
constexpr uint32_t gMcnt = gWsum + 32;                        // merge warps done with the sm buffer
constexpr uint32_t gBar = gMcnt + 16;                         // stage, sm, full[2], empty[2]
constexpr uint32_t gBytes = gBar + 48;
constexpr uint32_t kSmemWS = kOffGrp + kGroupsWS * gBytes;
static_assert(gSm % 16 == 0 && gSlots % 16 == 0 && gCnt % 16 == 0 && gReg % 16 == 0 && kRegWarp % 16 == 0 &&
                  gWsum % 16 == 0 && gBar % 8 == 0 && gBytes % 16 == 0, "alignment");
static_assert(2 * 4 * kSlotWarp >= 8192, "first-code scratch fits group 0's slots");
static_assert(kSmemWS <= 232448, "SMEM budget");

__device__ __forceinline__ void named_bar(uint32_t id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kLanes) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

__global__ void __launch_bounds__(kCtaWS, 1) ws_kernel(const __grid_constant__ Batch bt) {
    constexpr uint32_t kVF = DF11_VF_BF16;
    const uint32_t tid = threadIdx.x;
    const uint32_t g = tid / (2 * kLanes);
    const uint32_t local = tid % (2 * kLanes);
    const bool decoder = local < kLanes;
    const uint32_t t = local % kLanes;                          // lane index within the role (0..127)
    const uint32_t lane = tid & 31, wig = t >> 5;
    const uint32_t FULL = 0xFFFFFFFFu;
#define K_ROW bt.kpow[0]
#define K_TOP bt.kpow[1]
#define K_S24 bt.kpow[2]
#define K_ENT bt.kpow[3]
    uint8_t *sb = smem_b();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_w);
    const uint32_t tab = sbase + kOffT;
    const uint32_t gbase = sbase + kOffGrp + g * gBytes;
    const uint32_t stage = gbase + gStage;
    const uint32_t mbar = gbase + gBar, smbar = mbar + 8, fullb = mbar + 16, emptyb = mbar + 32;
    const uint32_t smb = gbase + gSm;
    const uint32_t mcnt = gbase + gMcnt;
    const uint32_t rlenb = sbase + kOffRLen;

    const uint32_t total = bt.total_tiles;
    const uint32_t c_begin = bt.cta_ranges ? bt.cta_start[blockIdx.x]
                                           : (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t c_end = bt.cta_ranges ? bt.cta_start[blockIdx.x + 1]
                                         : (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    if (c_begin >= c_end) return;
    if (local == 0) {
        mbar_init(mbar, 1);
        mbar_init(smbar, 1);
        mbar_init(fullb, 4);
        mbar_init(fullb + 8, 4);
        mbar_init(emptyb, 4);
        mbar_init(emptyb + 8, 4);
        sts32(mcnt, 0);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t q = 0, parity = 0, qs = 0;                      // tiles of this group so far (both roles)

    int ti_idx = tensor_of_tile(bt, c_begin);
    for (uint32_t seg_begin = c_begin; seg_begin < c_end; ti_idx++) {
        const df11_device_tensor &ts = bt.t[ti_idx];
        const uint32_t seg_end = min(c_end, bt.tile_start[ti_idx + 1]);
        const uint32_t base_tile = bt.tile_start[ti_idx] - bt.tile_off[ti_idx];
        if (seg_end <= seg_begin) continue;
        __syncthreads();
        uint32_t tile = seg_begin + g;
        if (tile < seg_end && local == 0) issue_tile(ts, tile - base_tile, stage, mbar);
        bool safe, lut_in_smem;
        const bool long_codes = build_t12<kCtaWS, kVF, true>(ts, sb, sbase, kOffT, kOffLut, kOffLen, kOffRLen,
                                                            kOffGrp + gSlots, tid, safe, lut_in_smem);
        if (safe) __trap();                                   // 1-bit codes: not handled by this variant
        const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k;
        const uint32_t N = (uint32_t)ts.num_elements;
        const bool vec_out = ((reinterpret_cast<uintptr_t>(ts.out) & 15) == 0);
        const bool psm_al = (reinterpret_cast<uintptr_t>(ts.packed_sign_mantissa) & 15) == 0;
        const bool sm_tma = vec_out && psm_al;
        auto sm_range = [&](uint32_t plo, uint32_t phi, uint32_t &a0, uint32_t &a1) {
            const uint32_t l = min(plo, N), h = min(max(min(phi, N), l), l + 8 * kN * kT);
            a0 = l & ~15u;
            a1 = (h + 15u) & ~15u;
            return sm_tma && a1 > a0 && a1 - a0 <= kSmCapWS;
        };
        auto stage_sm = [&](uint32_t b) {
            const uint32_t plo = __ldg(ts.block_output_pos + b), phi = __ldg(ts.block_output_pos + b + 1);
            uint32_t a0, a1;
            if (sm_range(plo, phi, a0, a1)) {
                mbar_expect_tx(smbar, a1 - a0);
                tma_g2s(smb, ts.packed_sign_mantissa + a0, a1 - a0, smbar);
            }
        };
        if (!decoder && t == 0 && tile < seg_end) stage_sm(tile - base_tile);

        if (decoder) {
#ifdef WS_DEC_REGS
            asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(WS_DEC_REGS));
#endif
            // =============================== decode role
            auto walk = [&](uint32_t w, uint32_t &len) -> uint32_t {
                if (lut_in_smem) return lut_walk_smem(w, sbase + kOffLut, sbase + kOffLen, eb_bytes, kk, 8u, len);
                return lut_walk_global<true>(w, ts, len);
            };
            for (uint32_t qq = q; tile < seg_end; tile += kGroupsWS, qq++) {
                const uint32_t b = tile - base_tile;
                const uint32_t k = qq & 1u;
                const uint32_t hi = min(__ldg(ts.block_output_pos + b + 1), N);
                mbar_wait(mbar, qq & 1u);
                uint32_t r0, r1, r2, r3, r4, gapA, gapB, gapC;
                lds128(stage + t * 16, r0, r1, r2, r3);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r4) : "r"(stage + t * 16 + 16));
                {
                    const uint32_t gb0 = stage + kChunkBytes + ((t * 10) >> 3);
                    const uint32_t h0 = ld8(gb0), h1 = ld8(gb0 + 1), h2 = ld8(gb0 + 2), h3 = ld8(gb0 + 3);
                    const uint32_t g32 = (h0 << 24) | (h1 << 16) | (h2 << 8) | h3;
                    const uint32_t g15 = (g32 >> (17u - ((t * 10) & 7u))) & 32767u;
                    gapA = g15 >> 10;
                    gapB = (g15 >> 5) & 31u;
                    gapC = g15 & 31u;
                }
                named_bar(1 + 2 * g);                           // every decode lane has read the stage
                if (t == 0 && tile + kGroupsWS < seg_end) issue_tile(ts, b + kGroupsWS, stage, mbar);
                if (qq >= 2) mbar_wait(emptyb + 8 * k, ((qq >> 1) + 1) & 1u);   // slots k are free again
                const uint32_t slotA = gbase + gSlots + k * (4 * kSlotWarp) + wig * kSlotWarp + lane * 4u;
                const uint32_t slotB = slotA + kSubWS * 128u;
                const uint32_t W0 = bswap32(r0), W1 = bswap32(r1), W2 = bswap32(r2), W3 = bswap32(r3),
                               W4 = bswap32(r4);
                const bool exact = long_codes && hi < N;
                const uint32_t limA = exact ? 64u + gapB - gapA : 64u - gapA;
                const uint32_t limB = exact ? 64u + gapC - gapB : 64u - gapB;
                uint32_t aA = W0, bA = W1, cA = exact ? W2 | (0xFFFFFFFFu >> gapB) : W2;
                uint32_t aB = W2, bB = W3, cB = exact ? W4 | (0xFFFFFFFFu >> gapC) : W4;
                shift96_ones(aA, bA, cA, gapA);
                shift96_ones(aB, bB, cB, gapB);
                uint32_t xA = kXEnd - limA, xB = kXEnd - limB;
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
                for (int u = 0; u < 6; u++) step();
                for (;;) {
                    const bool actA = (xA & kXEnd) == 0, actB = (xB & kXEnd) == 0;
                    if (!__any_sync(FULL, actA || actB)) break;
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
                slot_flush(oA);
                slot_flush(oB);
                uint32_t nA = slot_bytes(oA), nB = slot_bytes(oB);
                if (!exact) {
                    uint32_t offA = xA & kXMask;
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
                sts64(gbase + gCnt + k * 1024u + t * 8u, nA, nB);
                __syncwarp();
                if (lane == 0) mbar_arrive(fullb + 8 * k);     // release: slots and counts of this warp
            }
#ifdef WS_DEC_REGS
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(WS_BASE_REGS));
#endif
        } else {
#ifdef WS_MRG_REGS
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(WS_MRG_REGS));
#endif
            // =============================== merge role
            uint32_t qq = q;
            for (; tile < seg_end; tile += kGroupsWS, qq++) {
                const uint32_t b = tile - base_tile;
                const uint32_t k = qq & 1u;
                const bool has_next = tile + kGroupsWS < seg_end;
                const uint32_t lo = min(__ldg(ts.block_output_pos + b), N);
                const uint32_t hi = min(max(min(__ldg(ts.block_output_pos + b + 1), N), lo), lo + 8 * kN * kT);
                mbar_wait(fullb + 8 * k, (qq >> 1) & 1u);
                uint32_t cntA, cntB;
                lds64(gbase + gCnt + k * 1024u + t * 8u, cntA, cntB);
                const uint32_t cnt = cntA + cntB;
                uint32_t incl = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t v = __shfl_up_sync(FULL, incl, d);
                    if (lane >= (uint32_t)d) incl += v;
                }
                const uint32_t ws = gbase + gWsum + parity * 16u;
                if (lane == 31) sts32(ws + wig * 4, incl);
                named_bar(2 + 2 * g);
                parity ^= 1u;
                uint32_t wpre;
                {
                    uint4 v;
                    lds128(ws, v.x, v.y, v.z, v.w);
                    wpre = (wig > 0 ? v.x : 0u) + (wig > 1 ? v.y : 0u) + (wig > 2 ? v.z : 0u);
                }
                const uint32_t wtot = __shfl_sync(FULL, incl, 31);
                const uint32_t lpos = incl - cnt;
                const uint32_t wbeg = lo + wpre;
                const uint32_t wreg = gbase + gReg + wig * kRegWarp;
                const uint32_t F = wbeg & ~15u;
                const uint32_t ra = min(wbeg, hi), rb = min(wbeg + wtot, hi);
                const uint32_t ua = vec_out ? (ra + 7) >> 3 : 0, ub = vec_out ? max(rb >> 3, ua) : 0;
                const uint32_t ha = vec_out ? min(ua << 3, rb) : rb, tb = vec_out ? max(ub << 3, ha) : rb;
                const uint32_t es = lane < 16 ? ra + lane : tb + (lane - 16);
                const bool edge = vec_out && (lane < 16 ? es < ha : es < rb);
                {
                    const uint32_t slotA = gbase + gSlots + k * (4 * kSlotWarp) + wig * kSlotWarp + lane * 4u;
                    const uint32_t slotB = slotA + kSubWS * 128u;
                    uint32_t wa[8], wb[8];
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        wa[j] = lds32(slotA + 128u * j);
                        wb[j] = lds32(slotB + 128u * j);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(emptyb + 8 * k);  // this warp's slots may be refilled
                    const uint32_t dA = wreg + (wbeg - F) + lpos, dB = dA + cntA;
                    compact_words(dA, wa, cntA);
                    compact_words(dB, wb, cntB);
                    __syncwarp();
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
                    } else {
                        compact_head(dA, wa[0], cntA);
                        compact_head(dB, wb[0], cntB);
                    }
                    __syncwarp();
                }
                uint16_t *__restrict__ out = static_cast<uint16_t *>(ts.out);
                uint32_t a0, a1;
                if (sm_range(lo, hi, a0, a1)) {
                    mbar_wait(smbar, qs & 1u);
                    qs++;
                    if (edge) out[es] = compose_r(ld8(wreg + (es - F)), ld8(smb + (es - a0)));
                    const uint32_t nun = ub - ua, nfull = nun >> 5;
                    const uint32_t e0 = (ua + lane) << 3;
                    const uint32_t sa = smb + (e0 - a0), xa = wreg + (e0 - F);
                    uint4 *op = reinterpret_cast<uint4 *>(out + e0);
                    auto unit = [&](uint32_t kk2) {
                        uint32_t s0, s1, x0, x1;
                        lds64(sa + 256u * kk2, s0, s1);
                        lds64(xa + 256u * kk2, x0, x1);
                        uint4 o;
                        compose4r(x0, s0, o.x, o.y);
                        compose4r(x1, s1, o.z, o.w);
                        op[32 * kk2] = o;
                    };
                    uint32_t kk2 = 0;
                    for (; kk2 + 4 <= nfull; kk2 += 4) {
                        unit(kk2);
                        unit(kk2 + 1);
                        unit(kk2 + 2);
                        unit(kk2 + 3);
                    }
                    for (; kk2 < nfull; kk2++) unit(kk2);
                    if (lane < (nun & 31u)) unit(nfull);
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        uint32_t done;
                        asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(done) : "r"(mcnt) : "memory");
                        if (done == 3) {
                            sts32(mcnt, 0);
                            __threadfence_block();
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            if (has_next) stage_sm(b + kGroupsWS);
                        }
                    }
                } else {
                    const uint2 *__restrict__ psm2 = reinterpret_cast<const uint2 *>(ts.packed_sign_mantissa);
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
                    if (!vec_out)
                        for (uint32_t e = ra + lane; e < rb; e += 32)
                            out[e] = compose_r(ld8(wreg + (e - F)), __ldg(ts.packed_sign_mantissa + e));
                    if (t == 0 && has_next) stage_sm(b + kGroupsWS);
                    __syncwarp();
                }
            }
#ifdef WS_MRG_REGS
            asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(WS_BASE_REGS));
#endif
        }
        // both roles walked the same tiles of this segment
        q += (seg_end > seg_begin + g) ? (seg_end - seg_begin - g + kGroupsWS - 1) / kGroupsWS : 0u;
        seg_begin = seg_end;
    }
#undef K_ROW
#undef K_TOP
#undef K_ENT
#undef K_S24
}

}  // namespace

bool ws_enabled() {
    static const bool on = [] { const char *v = std::getenv("DF11_WS"); return v && v[0] == '1'; }();
    return on;
}

// BF16, T = 256, n = 8, byte tables only (the caller checks)
cudaError_t launch_ws(const Batch &bt, cudaStream_t stream, uint64_t *launches) {
    if (bt.total_tiles == 0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemWS);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    ws_kernel<<<bt.grid, kCtaWS, kSmemWS, stream>>>(bt);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace df11
