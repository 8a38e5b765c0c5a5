// decode_fast.cu — persistent sm_100a DF11 decode kernel (format T = 256, n = 8; narrow or wide LUTs).
//
// Same result as Algorithm 1 — every thread decodes the codewords that start in its
// 8-byte chunk, a block-level exclusive scan turns per-thread counts into output positions
// (P:148-150), phase 2 re-decodes into an SRAM buffer and the block writes BF16 with coalesced stores
// — re-designed for B200:
//
//  * Persistent CTAs, one per SM, 4 groups of 256 threads; group g of CTA c walks the format blocks
//    ("tiles") of a contiguous range.  Each group owns a 16 KB exponent buffer and uses its own
//    named barrier, so groups drift apart and hide each other's memory latency.
//  * Derived decode tables are built in SMEM once per (CTA, tensor) from the format's hierarchical
//    LUTs: for every R-bit prefix (R = 9),
//      T1 = {count of complete codes, their start mask, bits consumed}      (phase 1: counting)
//      T2 = {up to 3 decoded exponents, their count, bits consumed}         (phase 2: decoding)
//    Both are replicated 32x with lane-private banks (word = prefix*32 + lane): every LDS is
//    conflict-free.  Codes longer than R bits (≈0.1 % on LLM-like weights) take the paper's LUT walk
//    over the format tables (global, L1-resident) at a warp-uniform check every 4 steps.
//  * The thread's 8-byte chunk + 4 spill bytes live in 3 registers (big-endian); the 32-bit decode
//    window is a funnel shift — EncodedExponent is read from HBM exactly once (the paper re-reads it
//    from SRAM in phase 2).
//  * The next tile's chunk, gap and BlockOutputPos are prefetched into registers while the current
//    tile decodes; the sign/mantissa bytes of the tile are prefetched with 128-bit loads before
//    phase 1 and consumed by the merge.
//  * Merge: 16 elements per thread per step: LDS.128 exponents + LDG.128 sign/mantissa -> 8 words of
//    BF16 via byte permutes -> two 128-bit stores.  Head/tail groups shared with the neighbouring
//    tiles are written element-wise (disjoint ownership, no races).
#include "decode_common.cuh"

namespace df11 {
namespace {

constexpr int kT = 256;                    // format threads per block == group size
constexpr int kN = 8;                      // bytes per thread
constexpr int kGroups = 4;
constexpr int kCta = kT * kGroups;         // 1024 threads
constexpr int kR = 9;                      // root bits of the derived tables
constexpr int kTabWords = (1 << kR) * 32;  // 32 lane replicas
constexpr int kExpBuf = 8 * kN * kT + 64;  // worst case 1-bit codes + head offset + spill
constexpr size_t kSmemBytes = 2 * (size_t)kTabWords * 4 + (size_t)kGroups * kExpBuf + kGroups * 8 * 4;

struct Smem {
    uint32_t t1[kTabWords];
    uint32_t t2[kTabWords];
    uint8_t expbuf[kGroups][kExpBuf];
    uint32_t wsum[kGroups][8];
};
static_assert(sizeof(Smem) == kSmemBytes, "smem layout");

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Paper's hierarchical LUT walk over the format tables in global memory; returns the
// exponent and its code length.  Bounded: <= 4 levels, child < k, zero length -> 32.
__device__ __forceinline__ uint32_t lut_walk(uint32_t w, const df11_device_tensor &ts, uint32_t &len) {
    const uint8_t *__restrict__ luts = ts.luts;
    const uint32_t eb = ts.lut_entry_bytes, thr = eb == 1 ? 240u : 256u;
    uint32_t table = 0, e = 0;
#pragma unroll 1
    for (int i = 0; i < 4; i++) {
        uint32_t off = table * 256u + ((w >> (24 - 8 * i)) & 0xFFu);
        e = eb == 1 ? (uint32_t)__ldg(luts + off) : ((uint32_t)__ldg(luts + 2 * off) | ((uint32_t)__ldg(luts + 2 * off + 1) << 8));
        if (e < thr) break;
        table = eb == 1 ? 256u - e : e - 256u;
        if (table >= ts.k || i == 3) { e = 0; break; }
    }
    e &= 0xFFu;
    len = __ldg(ts.code_lengths + e);
    if (len == 0) len = 32;
    return e;
}

__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kT) : "memory");
}

// 32-bit MSB-first window at bit `off` (0 <= off < 64) of the 96-bit chunk (w0:w1:w2).
__device__ __forceinline__ uint32_t window(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t off) {
    const bool lo = off < 32;
    const uint32_t hi_w = lo ? w0 : w1, lo_w = lo ? w1 : w2;
    return __funnelshift_l(lo_w, hi_w, off);
}

// Two packed BF16 from x = (E1<<24 | S1<<16 | E0<<8 | S0): (sign<<15) | (E<<7) | mantissa per half.
__device__ __forceinline__ uint32_t compose2(uint32_t x) {
    return (x & 0x007F007Fu) | ((x >> 1) & 0x7F807F80u) | ((x << 8) & 0x80008000u);
}

struct TileIn {              // per-thread registers describing one tile
    uint32_t w0, w1, w2;     // chunk bytes (big-endian words)
    uint32_t gap;
    uint32_t lo, hi;         // clipped BlockOutputPos[b], BlockOutputPos[b+1]
};

__device__ __forceinline__ void load_tile(const df11_device_tensor &ts, uint32_t b, uint32_t t, TileIn &ti) {
    const uint8_t *enc = ts.encoded_exponent + (size_t)b * (kT * kN) + (size_t)t * kN;
    const uint2 v = __ldg(reinterpret_cast<const uint2 *>(enc));
    const uint32_t spill = __ldg(reinterpret_cast<const uint32_t *>(enc + 8));
    ti.w0 = v.x;                              // byte-swapped at use (keeps the loads in flight)
    ti.w1 = v.y;
    ti.w2 = spill;
    const uint64_t bit = 5ull * ((uint64_t)b * kT + t);
    const uint32_t hb = __ldg(ts.gaps + (bit >> 3)), lb = __ldg(ts.gaps + (bit >> 3) + 1);
    ti.gap = ((hb << 8) | lb) >> (11 - (uint32_t)(bit & 7));   // masked at use
    ti.lo = __ldg(ts.block_output_pos + b);
    ti.hi = __ldg(ts.block_output_pos + b + 1);
}

__global__ void __launch_bounds__(kCta, 1) fast_kernel(const __grid_constant__ Batch bt) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const uint32_t tid = threadIdx.x;
    const int g = (int)(tid / kT);
    const uint32_t t = tid % kT;
    const uint32_t lane = tid & 31, wig = t >> 5;
    const uint32_t FULL = 0xFFFFFFFFu;

    const uint32_t total = bt.total_tiles;
    const uint32_t c_begin = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t c_end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    if (c_begin >= c_end) return;

    int ti_idx = tensor_of_tile(bt, c_begin);
    for (uint32_t seg_begin = c_begin; seg_begin < c_end; ti_idx++) {
        const df11_device_tensor &ts = bt.t[ti_idx];
        const uint32_t seg_end = min(c_end, bt.tile_start[ti_idx + 1]);
        const uint32_t base_tile = bt.tile_start[ti_idx];
        if (seg_end <= seg_begin) continue;

        // ---- derived tables for this tensor (CTA-wide)
        __syncthreads();
        for (uint32_t idx = tid; idx < (1u << kR); idx += kCta) {
            const uint32_t W = idx << (32 - kR);
            uint32_t s = 0, cnt = 0, mask = 0, cons = 0, syms = 0, c2 = 0, cons2 = 0;
            while (s < (uint32_t)kR) {
                uint32_t len;
                const uint32_t sym = lut_walk(W << s, ts, len);
                if (len > (uint32_t)kR - s) break;
                mask |= 1u << s;
                cnt++;
                s += len;
                cons = s;
                if (c2 < 3) { syms |= sym << (8 * c2); c2++; cons2 = s; }
            }
            const uint32_t e1 = cnt ? (cnt | (mask << 8) | (cons << 28)) : 0u;
            const uint32_t e2 = c2 ? (syms | (c2 << 24) | (cons2 << 28)) : 0u;
            uint4 *d1 = reinterpret_cast<uint4 *>(S.t1 + idx * 32);
            uint4 *d2 = reinterpret_cast<uint4 *>(S.t2 + idx * 32);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                d1[q] = make_uint4(e1, e1, e1, e1);
                d2[q] = make_uint4(e2, e2, e2, e2);
            }
        }
        __syncthreads();

        const uint32_t N = (uint32_t)ts.num_elements;
        const bool vec_out = ((reinterpret_cast<uintptr_t>(ts.out) & 15) == 0);
        const uint32_t *t1 = S.t1 + lane;
        const uint32_t *t2 = S.t2 + lane;
        uint8_t *ebuf = S.expbuf[g];

        uint32_t tile = seg_begin + g;
        TileIn cur;
        if (tile < seg_end) load_tile(ts, tile - base_tile, t, cur);
        for (; tile < seg_end; tile += kGroups) {
            const uint32_t b = tile - base_tile;
            // prefetch the next tile of this group
            TileIn nxt;
            const bool has_next = tile + kGroups < seg_end;
            if (has_next) load_tile(ts, b + kGroups, t, nxt);

            const uint32_t w0 = bswap32(cur.w0), w1 = bswap32(cur.w1), w2 = bswap32(cur.w2);
            const uint32_t gap = cur.gap & 31u;
            const uint32_t lo = min(cur.lo, N);
            const uint32_t hi = min(max(min(cur.hi, N), lo), lo + (uint32_t)(8 * kN * kT));
            const uint32_t f = lo & ~15u;                      // 16-element aligned frame origin
            const uint32_t g_first = f >> 4, g_last = (hi + 15) >> 4;

            // sign/mantissa prefetch for this thread's first two merge groups
            uint4 smA = make_uint4(0, 0, 0, 0), smB = make_uint4(0, 0, 0, 0);
            const uint32_t gA = g_first + t, gB = g_first + t + kT;
            if (gA < g_last) smA = __ldg(reinterpret_cast<const uint4 *>(ts.packed_sign_mantissa) + gA);
            if (gB < g_last) smB = __ldg(reinterpret_cast<const uint4 *>(ts.packed_sign_mantissa) + gB);

            // ---- phase 1: count codewords starting in [0, 64) (T1, several codes per lookup)
            uint32_t off = gap, cnt = 0, e1 = 1;
            for (;;) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    if (off < 64) {
                        const uint32_t w = window(w0, w1, w2, off);
                        e1 = t1[(w >> (32 - kR)) << 5];
                        cnt += e1 & 15u;
                        off += e1 >> 28;
                    }
                }
                if (!__any_sync(FULL, off < 64)) break;
                const bool esc = off < 64 && e1 == 0;
                if (__any_sync(FULL, esc)) {
                    if (esc) {                                 // code longer than R bits
                        uint32_t len;
                        lut_walk(window(w0, w1, w2, off), ts, len);
                        cnt++;
                        off += len;
                    }
                }
            }
            {   // the last group may hold complete codes that start at or after bit 64: not ours
                const uint32_t last = off - (e1 >> 28);
                const uint32_t keep = __funnelshift_lc(0u, 1u, 64u - min(last, 64u)) - 1u;  // starts s < 64-last
                cnt -= __popc((e1 >> 8) & 0x1FFu & ~keep);
            }

            // ---- block exclusive scan over the 256 counts (warp shuffles + 8 warp totals)
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(FULL, incl, d);
                if (lane >= (uint32_t)d) incl += v;
            }
            if (lane == 31) S.wsum[g][wig] = incl;
            group_bar(g);
            uint32_t wpre = 0;
#pragma unroll
            for (uint32_t q = 0; q < 8; q++) {
                const uint32_t s = S.wsum[g][q];
                wpre += q < wig ? s : 0u;
            }
            uint8_t *wp = ebuf + (lo - f) + wpre + incl - cnt;

            // ---- phase 2: re-decode (T2, up to 3 exponents per lookup) into the SMEM buffer
            off = gap;
            uint32_t j = 0, e2 = 1;
            for (;;) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    if (j < cnt) {
                        const uint32_t w = window(w0, w1, w2, off);
                        e2 = t2[(w >> (32 - kR)) << 5];
                        wp[j] = (uint8_t)e2;
                        if (j + 1 < cnt) wp[j + 1] = (uint8_t)(e2 >> 8);
                        if (j + 2 < cnt) wp[j + 2] = (uint8_t)(e2 >> 16);
                        j += (e2 >> 24) & 3u;
                        off += e2 >> 28;
                    }
                }
                if (!__any_sync(FULL, j < cnt)) break;
                const bool esc = j < cnt && e2 == 0;
                if (__any_sync(FULL, esc)) {
                    if (esc) {
                        uint32_t len;
                        wp[j] = (uint8_t)lut_walk(window(w0, w1, w2, off), ts, len);
                        j++;
                        off += len;
                    }
                }
            }
            group_bar(g);

            // ---- merge: compose BF16 and store, 16 elements per thread per step
            uint16_t *__restrict__ out = ts.out;
            for (uint32_t gi = gA, it = 0; gi < g_last; gi += kT, it++) {
                const uint32_t e0 = gi << 4;
                const uint4 ex = *reinterpret_cast<const uint4 *>(ebuf + (e0 - f));
                uint4 sm;
                if (it == 0) sm = smA;
                else if (it == 1) sm = smB;
                else sm = __ldg(reinterpret_cast<const uint4 *>(ts.packed_sign_mantissa) + gi);
                if (vec_out && e0 >= lo && e0 + 16 <= hi) {
                    uint4 o0, o1;
                    o0.x = compose2(__byte_perm(sm.x, ex.x, 0x5140));
                    o0.y = compose2(__byte_perm(sm.x, ex.x, 0x7362));
                    o0.z = compose2(__byte_perm(sm.y, ex.y, 0x5140));
                    o0.w = compose2(__byte_perm(sm.y, ex.y, 0x7362));
                    o1.x = compose2(__byte_perm(sm.z, ex.z, 0x5140));
                    o1.y = compose2(__byte_perm(sm.z, ex.z, 0x7362));
                    o1.z = compose2(__byte_perm(sm.w, ex.w, 0x5140));
                    o1.w = compose2(__byte_perm(sm.w, ex.w, 0x7362));
                    uint4 *dst = reinterpret_cast<uint4 *>(out + e0);
                    dst[0] = o0;
                    dst[1] = o1;
                } else {
                    const uint32_t exw[4] = {ex.x, ex.y, ex.z, ex.w};
                    const uint32_t smw[4] = {sm.x, sm.y, sm.z, sm.w};
#pragma unroll
                    for (uint32_t q = 0; q < 16; q++) {
                        const uint32_t e = e0 + q;
                        if (e >= lo && e < hi)
                            out[e] = compose((exw[q >> 2] >> (8 * (q & 3))) & 0xFFu, (smw[q >> 2] >> (8 * (q & 3))) & 0xFFu);
                    }
                }
            }
            if (has_next) cur = nxt;
        }
        seg_begin = seg_end;
    }
}

int g_attr_set[64];

}  // namespace

bool fast_supports(const df11_device_tensor &t) {
    return t.T == (uint32_t)kT && t.n == (uint32_t)kN &&
           (reinterpret_cast<uintptr_t>(t.encoded_exponent) & 7) == 0 &&
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
