// encode_gpu.cu — device half of the GPU encoder.
//
// Produces the DF11 arrays of DESIGN.md §2 from a tensor already in HBM (BF16, or FP16 / FP8 words:
// NEXT-4, R25), byte-identical to the host encoder (encode.cpp) for the same codebook:
//   EncodedExponent   canonical Huffman codes of the exponents, MSB-first, tightly packed
//   PackedSignMantissa sign<<7 | mantissa, one byte per element; FP16: the low residual bytes
//                     as a byte plane + the 3 high bits (sign, m9, m8) as a bit plane; FP8: the R-bit
//                     residuals sign << M | mantissa, MSB-first (R25)
//   Gaps              per format thread: bit offset of the first code starting in its n-byte chunk,
//                     0 if none (R13), packed 5 bits MSB-first (R12)
//   BlockOutputPos    per block: number of codes starting before the block's first bit
//
// Kernels (all HBM-bound; per element: 2 B read + 1 B PSM + ~0.33 B stream written):
//   hist_kernel   exponent histogram; per-warp shared-memory counters, 16-B vector loads.
//   pack_kernel   one CTA per 4096-element segment (256 threads x 16 elements).  The bit offset of a
//                 segment is the sum of the code lengths before it: a single-pass decoupled look-back
//                 scan over per-segment totals (segments are taken in order from an atomic ticket, so
//                 every predecessor is resident or finished -> no deadlock).  Inside the CTA a warp-
//                 shuffle scan gives each thread its local first bit; each thread packs its codes
//                 through a 64-bit accumulator into a shared-memory copy of the segment's bits (local
//                 bit 0; only words shared with a neighbour thread use a shared-memory atomic OR) while
//                 the look-back runs; the CTA then writes the segment with one funnel shift by the
//                 global offset, coalesced, and atomic OR only on its first and last global words.
//                 Because every code is <= 32 <= 8n bits, consecutive code starts lie in
//                 the same or the next chunk, so the first start of chunk c / block b is detected from
//                 the previous start alone (one compare per element, no division in the loop).
//   gaps_kernel   packs 8 gap values into 5 bytes (40 bits, MSB-first).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <type_traits>

#include "df11.h"
#include "df11_internal.h"

namespace df11 {
namespace {

constexpr int kHistThreads = 512;
constexpr int kPackThreads = 256;
constexpr int kPerThread = 16;
constexpr int kSeg = kPackThreads * kPerThread;   // 4096 elements per segment
static_assert(kSeg == DF11_ENCODE_SEGMENT, "workspace sizing in encode.cpp");

constexpr unsigned long long kFlagAgg = 1ull << 62;   // look-back word: status in bits 62..63
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// value formats (df11.h DF11_VF_*): exponent field at bits [M, M + E) of a word
template <uint32_t kVF>
struct VFT {
    static constexpr uint32_t M = kVF == DF11_VF_BF16 ? 7 : kVF == DF11_VF_FP16 ? 10 : kVF == DF11_VF_FP8_E4M3 ? 3 : 2;
    static constexpr uint32_t E = kVF == DF11_VF_BF16 ? 8 : kVF == DF11_VF_FP8_E4M3 ? 4 : 5;
    static constexpr uint32_t R = 1 + M;
    static constexpr uint32_t WB = (kVF == DF11_VF_BF16 || kVF == DF11_VF_FP16) ? 2 : 1;   // word bytes
    using W = typename std::conditional<WB == 2, uint16_t, uint8_t>::type;
    __device__ static uint32_t exp_of(uint32_t x) { return (x >> M) & ((1u << E) - 1u); }
    __device__ static uint32_t res_of(uint32_t x) { return ((x >> (E + M)) << M) | (x & ((1u << M) - 1u)); }
};

template <uint32_t kVF>
__global__ void __launch_bounds__(kHistThreads) hist_kernel(const typename VFT<kVF>::W *__restrict__ w, uint64_t n,
                                                            unsigned long long *__restrict__ hist) {
    using F = VFT<kVF>;
    constexpr uint32_t kPerVec = 16 / F::WB;                 // words per 16-byte load
    constexpr int kWarps = kHistThreads / 32;
    __shared__ uint32_t h[kWarps][256];
    for (int i = threadIdx.x; i < kWarps * 256; i += kHistThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t *mine = h[threadIdx.x >> 5];
    const uint64_t gt = (uint64_t)blockIdx.x * kHistThreads + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * kHistThreads;
    // elements before the first 16-byte boundary (w is aligned to its word size)
    const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(w) & 15u) / F::WB);
    const uint64_t head = mis ? (n < kPerVec - mis ? n : kPerVec - mis) : 0;
    if (gt < head) atomicAdd(&mine[F::exp_of(w[gt])], 1u);
    const uint4 *v = reinterpret_cast<const uint4 *>(w + head);
    const uint64_t nv = (n - head) / kPerVec;
    for (uint64_t q = gt; q < nv; q += stride) {
        uint4 x;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(v + q));
        const uint32_t ws[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
#pragma unroll
            for (uint32_t k = 0; k < 4 / F::WB; k++) atomicAdd(&mine[F::exp_of(ws[j] >> (8 * F::WB * k))], 1u);
        }
    }
    const uint64_t tail = head + nv * kPerVec;
    for (uint64_t i = tail + gt; i < n; i += stride) atomicAdd(&mine[F::exp_of(w[i])], 1u);
    __syncthreads();
    for (int s = threadIdx.x; s < 256; s += kHistThreads) {
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < kWarps; k++) c += h[k][s];
        if (c) atomicAdd(&hist[s], (unsigned long long)c);
    }
}

struct PackParams {
    const void *w;
    uint64_t n;                       // elements
    uint32_t *stream;                 // EncodedExponent as 32-bit words (zeroed)
    uint64_t stream_words;            // clip bound
    uint8_t *psm;
    uint8_t *gapv;                    // one byte per format thread (zeroed)
    uint32_t *bop;                    // B+1 entries (pre-filled with N)
    unsigned long long *flags;        // look-back words, one per segment (zeroed)
    uint32_t *ticket;                 // zeroed
    uint64_t chunk_bits, block_bits;  // 8n, 8nT
    uint64_t chunks;                  // B*T
    uint32_t B;
    uint32_t aligned;                 // w and psm 16-byte aligned
    uint32_t vf;
    uint32_t codes[256];
    uint8_t lens[256];
};

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <uint32_t kVF>
__global__ void __launch_bounds__(kPackThreads) pack_kernel(const __grid_constant__ PackParams p) {
    using F = VFT<kVF>;
    using W = typename F::W;
    const W *__restrict__ wp = static_cast<const W *>(p.w);
    __shared__ uint32_t s_code[256];
    __shared__ uint32_t s_len[256];
    __shared__ uint32_t s_warp[kPackThreads / 32];
    __shared__ uint32_t s_seg;
    __shared__ uint32_t s_geo[4];            // c0, r0, b0-low, rb0: the segment start in chunk/block units
    __shared__ unsigned long long s_prefix;
    __shared__ __align__(16) uint32_t s_words[kSeg + 4];   // the segment's codes at local bit 0
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int i = t; i < (kSeg + 4) / 4; i += kPackThreads) reinterpret_cast<uint4 *>(s_words)[i] = make_uint4(0, 0, 0, 0);
    s_code[t] = p.codes[t];
    s_len[t] = p.lens[t];
    if (t == 0) s_seg = atomicAdd(p.ticket, 1u);
    __syncthreads();
    const uint64_t seg = s_seg;
    const uint64_t base = seg * kSeg + (uint64_t)t * kPerThread;
    const int cnt = base >= p.n ? 0 : (p.n - base >= kPerThread ? kPerThread : (int)(p.n - base));

    constexpr uint32_t kPer32 = 4 / F::WB;                    // words per register
    uint32_t x[kPerThread / kPer32];
    if (cnt == kPerThread && p.aligned) {
#pragma unroll
        for (int q = 0; q < (int)(kPerThread * F::WB / 16); q++) {
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x[4 * q]), "=r"(x[4 * q + 1]), "=r"(x[4 * q + 2]), "=r"(x[4 * q + 3])
                         : "l"(wp + base + (16 / F::WB) * q));
        }
    } else {
#pragma unroll
        for (int j = 0; j < kPerThread / (int)kPer32; j++) {
            uint32_t v = 0;
#pragma unroll
            for (uint32_t k = 0; k < kPer32; k++)
                v |= (j * kPer32 + k < (uint32_t)cnt ? (uint32_t)wp[base + j * kPer32 + k] : 0u) << (8 * F::WB * k);
            x[j] = v;
        }
    }
#define ELEM(j) ((x[(j) / kPer32] >> (8 * F::WB * ((j) % kPer32))) & (F::WB == 2 ? 0xFFFFu : 0xFFu))
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < kPerThread; j++) bits += j < cnt ? s_len[F::exp_of(ELEM(j))] : 0u;

    // CTA exclusive scan of per-thread bit counts
    uint32_t incl = bits;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kPackThreads / 32; k++) {
        const uint32_t v = s_warp[k];
        wpre += k < warp ? v : 0u;
        total += v;
    }
    const uint32_t excl = wpre + incl - bits;

    // warp 0: publish the segment total and resolve its global bit offset (decoupled look-back);
    // the other warps pack meanwhile
    if (warp == 0) {
        unsigned long long acc = 0;
        if (seg == 0) {
            if (lane == 0) st_relaxed(&p.flags[0], kFlagIncl | total);
        } else {
            if (lane == 0) st_relaxed(&p.flags[seg], kFlagAgg | total);
            int64_t look = (int64_t)seg - 1;
            while (true) {
                const int64_t idx = look - lane;
                const unsigned long long f = idx >= 0 ? ld_relaxed(&p.flags[idx]) : kFlagIncl;
                const uint32_t st = (uint32_t)(f >> 62);
                if (__any_sync(0xFFFFFFFFu, st == 0)) continue;   // a predecessor has not published yet
                const uint32_t incl_mask = __ballot_sync(0xFFFFFFFFu, st == 2);
                const int first = incl_mask ? __ffs(incl_mask) - 1 : 32;
                unsigned long long v = lane <= first ? (f & kValMask) : 0ull;
#pragma unroll
                for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
                acc += v;
                if (incl_mask) break;
                look -= 32;
            }
            if (lane == 0) st_relaxed(&p.flags[seg], kFlagIncl | (acc + total));
        }
        if (lane == 0) {
            s_prefix = acc;
            const uint64_t c0 = acc / p.chunk_bits, b0 = acc / p.block_bits;
            s_geo[0] = (uint32_t)c0;                              // < 2^32: bits < 2^37, 8n >= 32
            s_geo[1] = (uint32_t)(acc - c0 * p.chunk_bits);
            s_geo[2] = (uint32_t)b0;
            s_geo[3] = (uint32_t)(acc - b0 * p.block_bits);
        }
    }

    // pack this thread's codes into s_words at local bit `excl`; only words shared with a
    // neighbouring thread need the shared-memory atomic OR
    {
        const uint32_t off = excl & 31u;
        uint32_t widx = excl >> 5;
        unsigned long long acc = 0;
        uint32_t nb = off;
        bool shared = off != 0;
#pragma unroll
        for (int j = 0; j < kPerThread; j++) {
            if (j >= cnt) break;
            const uint32_t e = F::exp_of(ELEM(j));
            const uint32_t l = s_len[e];
            acc = (acc << l) | s_code[e];
            nb += l;
            if (nb >= 32) {
                nb -= 32;
                const uint32_t word = (uint32_t)(acc >> nb);
                if (shared) atomicOr(&s_words[widx], word);
                else s_words[widx] = word;
                shared = false;
                widx++;
                acc &= (1ull << nb) - 1ull;
            }
        }
        if (nb > 0 && bits) atomicOr(&s_words[widx], (uint32_t)(acc << (32 - nb)));
    }
    __syncthreads();

    // write the segment's words at global bit S0: funnel shift by S0 & 31; the first and last global
    // words are shared with the neighbouring segments (atomic OR into the zeroed stream)
    const uint64_t S0 = s_prefix;
    if (total) {
        const uint32_t o0 = (uint32_t)(S0 & 31u);
        const uint64_t W0 = S0 >> 5, W1 = (S0 + total - 1) >> 5;
        const uint32_t nw = (uint32_t)(W1 - W0 + 1);
        const bool head_shared = o0 != 0, tail_shared = ((S0 + total) & 31u) != 0;
        for (uint32_t j = t; j < nw; j += kPackThreads) {
            const uint32_t cur = s_words[j];
            const uint32_t prv = j ? s_words[j - 1] : 0u;
            const uint32_t word = o0 ? (prv << (32 - o0)) | (cur >> o0) : cur;
            const uint64_t g = W0 + j;
            if (g >= p.stream_words) continue;
            const uint32_t be = __byte_perm(word, 0, 0x0123);   // MSB-first bytes in memory
            if ((j == 0 && head_shared) || (j == nw - 1 && tail_shared)) {
                if (be) atomicOr(&p.stream[g], be);
            } else {
                p.stream[g] = be;
            }
        }
    }
    if (cnt == 0) return;

    // PackedSignMantissa: sign << 7 | mantissa (BF16); FP16: byte plane + 3-bit plane; FP8: 16 R-bit
    // residuals = 2R bytes at byte R * base / 8, MSB-first (base is a multiple of 16: every thread's
    // range is whole bytes)
    if constexpr (kVF == DF11_VF_BF16) {
        if (cnt == kPerThread && p.aligned) {
            uint32_t o[kPerThread / 4];
#pragma unroll
            for (int q = 0; q < kPerThread / 4; q++) {
                const uint32_t a = x[2 * q], b = x[2 * q + 1];
                // bytes: e0 = a lo, e1 = a hi, e2 = b lo, e3 = b hi; psm = (w >> 8 & 0x80) | (w & 0x7F)
                const uint32_t sgn = __byte_perm(a, b, 0x7531) & 0x80808080u;   // high bytes -> sign bits
                const uint32_t man = __byte_perm(a, b, 0x6420) & 0x7F7F7F7Fu;   // low bytes -> mantissa
                o[q] = sgn | man;
            }
#pragma unroll
            for (int q = 0; q < kPerThread / 16; q++)
                *reinterpret_cast<uint4 *>(p.psm + base + 16 * q) = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < kPerThread; j++)
                if (j < cnt) p.psm[base + j] = (uint8_t)(((ELEM(j) >> 8) & 0x80u) | (ELEM(j) & 0x7Fu));
        }
    } else if constexpr (kVF == DF11_VF_FP16) {
        // byte plane: the low 8 residual bits at byte i; then the 3-bit plane (sign, m9, m8) at
        // roundup(N, 16) + 3 i / 8 bits, MSB-first (R25): 16 elements = 6 whole bytes at 3 base / 8
#pragma unroll
        for (int j = 0; j < kPerThread; j++)
            if (j < cnt) p.psm[base + j] = (uint8_t)F::res_of(ELEM(j));
        uint8_t *dst = p.psm + ((p.n + 15) & ~15ull) + base / 8 * 3;
        unsigned long long acc = 0;
#pragma unroll
        for (int j = 0; j < kPerThread; j++) acc = (acc << 3) | (j < cnt ? (F::res_of(ELEM(j)) >> 8) : 0u);
        const uint32_t nbytes = (cnt * 3 + 7) / 8;
#pragma unroll
        for (uint32_t k = 0; k < 6; k++)
            if (k < nbytes) dst[k] = (uint8_t)(acc >> (40 - 8 * k));
    } else {
        uint8_t *dst = p.psm + base / 8 * F::R;
        unsigned long long acc = 0;
        uint32_t nb = 0, k = 0;
#pragma unroll
        for (int j = 0; j < kPerThread; j++) {
            acc = (acc << F::R) | (j < cnt ? F::res_of(ELEM(j)) : 0u);
            nb += F::R;
            while (nb >= 8) {
                nb -= 8;
                if (k < (uint32_t)((cnt * F::R + 7) / 8)) dst[k] = (uint8_t)(acc >> nb);
                k++;
            }
        }
    }

    // Gaps and BlockOutputPos: position of this thread's first code relative to its chunk / block,
    // all in 32-bit arithmetic from the segment's start (excl < 2^17, 8nT <= 2^18)
    const uint32_t CB = (uint32_t)p.chunk_bits, BB = (uint32_t)p.block_bits;
    const uint32_t lc = s_geo[1] + excl, lb = s_geo[3] + excl;
    uint64_t chunk = (uint64_t)s_geo[0] + lc / CB;
    uint64_t blk = (uint64_t)s_geo[2] + lb / BB;
    uint32_t rc = lc % CB, rb = lb % BB;
    const uint32_t lprev = base > 0 ? s_len[F::exp_of(wp[base - 1])] : 0u;
    if (base == 0 || rc < lprev) {       // the previous code started in an earlier chunk
        if (chunk < p.chunks) p.gapv[chunk] = (uint8_t)rc;
    }
    if (base == 0 || rb < lprev) {
        if (blk < p.B) p.bop[blk] = (uint32_t)base;
    }
#pragma unroll
    for (int j = 0; j < kPerThread - 1; j++) {
        if (j + 1 >= cnt) break;
        const uint32_t l = s_len[F::exp_of(ELEM(j))];
        rc += l;
        rb += l;
        if (rc >= CB) {                  // codes are <= 32 <= 8n bits: at most one boundary per code
            rc -= CB;
            chunk++;
            if (chunk < p.chunks) p.gapv[chunk] = (uint8_t)rc;
        }
        if (rb >= BB) {
            rb -= BB;
            blk++;
            if (blk < p.B) p.bop[blk] = (uint32_t)(base + j + 1);
        }
    }
#undef ELEM
}

// Small host->device copies as kernel parameters (always asynchronous, unlike a pageable memcpy).
constexpr int kBlobBytes = 4000;
struct Blob {
    uint8_t *dst;
    uint32_t bytes;
    uint8_t data[kBlobBytes];
};
__global__ void blob_kernel(const __grid_constant__ Blob b) {
    for (uint32_t i = threadIdx.x; i < b.bytes; i += blockDim.x) b.dst[i] = b.data[i];
}

__global__ void fill_u32_kernel(uint32_t *p, uint64_t count, uint32_t v) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// 8 gap values -> 5 bytes, field g at stream bits [5g, 5g+5) (R12)
__global__ void gaps_kernel(const uint8_t *__restrict__ gapv, uint64_t count, uint8_t *__restrict__ out) {
    const uint64_t groups = (count + 7) / 8;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < groups;
         q += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t v = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t g = q * 8 + j;
            v = (v << 5) | (g < count ? (uint64_t)(gapv[g] & 31u) : 0ull);
        }
#pragma unroll
        for (int j = 0; j < 5; j++) out[q * 5 + j] = (uint8_t)(v >> (32 - 8 * j));
    }
}

int num_sms() {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) return 148;
    return v;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace
}  // namespace df11

namespace df11 {
namespace {
template <uint32_t kVF>
cudaError_t launch_hist(const void *d, uint64_t n, uint64_t *hist, cudaStream_t stream) {
    using F = VFT<kVF>;
    const uint64_t vec = n / (16 / F::WB);
    uint64_t want = (vec + kHistThreads - 1) / kHistThreads;
    const uint64_t cap = (uint64_t)num_sms() * 4;
    const unsigned grid = (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
    hist_kernel<kVF><<<grid, kHistThreads, 0, stream>>>(static_cast<const typename F::W *>(d), n,
                                                        reinterpret_cast<unsigned long long *>(hist));
    return cudaGetLastError();
}
uint32_t word_bytes(uint32_t vf) { return vf == DF11_VF_BF16 || vf == DF11_VF_FP16 ? 2u : 1u; }
uint32_t residual_bits(uint32_t vf) {
    return vf == DF11_VF_FP16 ? 11u : vf == DF11_VF_FP8_E4M3 ? 4u : vf == DF11_VF_FP8_E5M2 ? 3u : 8u;
}
}  // namespace
}  // namespace df11

extern "C" df11_status df11_histogram_device(const void *d_values, uint64_t n, uint32_t value_format, uint64_t *d_hist,
                                             void *stream) {
    using namespace df11;
    if (!d_hist || (n && !d_values)) return df11_fail(DF11_E_INVALID_ARGUMENT, "NULL argument");
    if (value_format > DF11_VF_FP8_E5M2) return df11_fail(DF11_E_INVALID_ARGUMENT, "bad value_format");
    if (reinterpret_cast<uintptr_t>(d_values) & (word_bytes(value_format) - 1))
        return df11_fail(DF11_E_INVALID_ARGUMENT, "d_values not aligned to the word size");
    if (n == 0) return DF11_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    switch (value_format) {
        case DF11_VF_FP16: e = launch_hist<DF11_VF_FP16>(d_values, n, d_hist, s); break;
        case DF11_VF_FP8_E4M3: e = launch_hist<DF11_VF_FP8_E4M3>(d_values, n, d_hist, s); break;
        case DF11_VF_FP8_E5M2: e = launch_hist<DF11_VF_FP8_E5M2>(d_values, n, d_hist, s); break;
        default: e = launch_hist<DF11_VF_BF16>(d_values, n, d_hist, s); break;
    }
    if (e != cudaSuccess) return df11_cuda_fail((int)e, "histogram launch");
    df11_count_launches(1);
    return DF11_OK;
}

extern "C" df11_status df11_encode_device(const void *d_values, const df11_encode_plan *plan,
                                          const df11_device_buffers *dst, void *workspace, uint64_t workspace_bytes,
                                          void *stream_) {
    using namespace df11;
    if (!plan || !dst) return df11_fail(DF11_E_INVALID_ARGUMENT, "NULL plan or dst");
    const uint64_t N = plan->num_elements;
    const uint64_t chunks = (uint64_t)plan->B * plan->T;
    if (!dst->encoded_exponent || !dst->packed_sign_mantissa || !dst->gaps || !dst->luts || !dst->code_lengths ||
        !dst->block_output_pos || (N && !d_values) || !workspace)
        return df11_fail(DF11_E_INVALID_ARGUMENT, "NULL buffer");
    if (workspace_bytes < plan->workspace_bytes) return df11_fail(DF11_E_INVALID_ARGUMENT, "workspace too small");
    if (!aligned16(dst->encoded_exponent) || !aligned16(dst->packed_sign_mantissa) || !aligned16(dst->gaps) ||
        !aligned16(dst->block_output_pos) || !aligned16(workspace))
        return df11_fail(DF11_E_INVALID_ARGUMENT, "device buffers must be 16-byte aligned");
    if (plan->value_format > DF11_VF_FP8_E5M2) return df11_fail(DF11_E_INVALID_ARGUMENT, "bad value_format");
    const uint32_t vf = plan->value_format;
    if (reinterpret_cast<uintptr_t>(d_values) & (word_bytes(vf) - 1))
        return df11_fail(DF11_E_INVALID_ARGUMENT, "d_values not aligned to the word size");
    if (plan->n < 4 || plan->n > 32 || plan->T < 32 || plan->T > 1024 || plan->max_code_len > 32)
        return df11_fail(DF11_E_INVALID_ARGUMENT, "plan geometry out of range");
    cudaStream_t st = (cudaStream_t)stream_;
    uint64_t launches = 0;
    cudaError_t e;
#define DF11_TRY(call, what)                                                     \
    do {                                                                         \
        e = (call);                                                              \
        if (e != cudaSuccess) return df11_cuda_fail((int)e, what);               \
    } while (0)
    // workspace: gap values | look-back words | ticket
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    const uint64_t gapv_bytes = (chunks + 15) / 16 * 16;
    const uint64_t segments = (N + kSeg - 1) / kSeg;
    uint8_t *gapv = ws;
    unsigned long long *flags = reinterpret_cast<unsigned long long *>(ws + gapv_bytes);
    uint32_t *ticket = reinterpret_cast<uint32_t *>(ws + gapv_bytes + 8 * ((segments + 1) / 2 * 2));
    DF11_TRY(cudaMemsetAsync(ws, 0, plan->workspace_bytes, st), "workspace memset");
    DF11_TRY(cudaMemsetAsync(dst->encoded_exponent, 0, plan->encoded_exponent_bytes, st), "stream memset");
    DF11_TRY(cudaMemsetAsync(dst->gaps, 0, plan->gaps_bytes, st), "gaps memset");
    {   // residual bytes past the last element's (its partial byte is written whole by the pack kernel);
        // FP16's two planes (R25) leave gaps between them: zero the whole array
        const uint64_t used = vf == DF11_VF_FP16 ? 0 : N * residual_bits(vf) / 8;
        DF11_TRY(cudaMemsetAsync(dst->packed_sign_mantissa + used, 0, plan->packed_sign_mantissa_bytes - used, st),
                 "psm memset");
    }
    {   // CodeLengths + LUTs through kernel parameters (no host synchronisation)
        Blob b;
        b.dst = dst->code_lengths;
        b.bytes = 256;
        std::memcpy(b.data, plan->code_lengths, 256);
        blob_kernel<<<1, 256, 0, st>>>(b);
        DF11_TRY(cudaGetLastError(), "blob launch");
        launches++;
        for (uint64_t o = 0; o < plan->luts_bytes; o += kBlobBytes) {
            const uint64_t m = plan->luts_bytes - o < (uint64_t)kBlobBytes ? plan->luts_bytes - o : kBlobBytes;
            b.dst = dst->luts + o;
            b.bytes = (uint32_t)m;
            std::memcpy(b.data, plan->luts + o, m);
            blob_kernel<<<1, 256, 0, st>>>(b);
            DF11_TRY(cudaGetLastError(), "blob launch");
            launches++;
        }
    }
    const int sms = num_sms();
    {
        const uint64_t cnt = (uint64_t)plan->B + 1;
        unsigned g = (unsigned)((cnt + 255) / 256);
        if (g > (unsigned)sms * 4) g = sms * 4;
        fill_u32_kernel<<<g, 256, 0, st>>>(dst->block_output_pos, cnt, (uint32_t)N);
        DF11_TRY(cudaGetLastError(), "fill launch");
        launches++;
    }
    if (N) {
        PackParams p;
        std::memset(&p, 0, sizeof(p));
        p.w = d_values;
        p.vf = vf;
        p.n = N;
        p.stream = reinterpret_cast<uint32_t *>(dst->encoded_exponent);
        p.stream_words = plan->encoded_exponent_bytes / 4;
        p.psm = dst->packed_sign_mantissa;
        p.gapv = gapv;
        p.bop = dst->block_output_pos;
        p.flags = flags;
        p.ticket = ticket;
        p.chunk_bits = 8ull * plan->n;
        p.block_bits = 8ull * plan->n * plan->T;
        p.chunks = chunks;
        p.B = plan->B;
        p.aligned = aligned16(d_values) ? 1u : 0u;
        std::memcpy(p.codes, plan->codes, sizeof(p.codes));
        std::memcpy(p.lens, plan->code_lengths, 256);
        if (segments > 0x7FFFFFFFull) return df11_fail(DF11_E_TOO_LARGE, "too many segments");
        switch (vf) {
            case DF11_VF_FP16: pack_kernel<DF11_VF_FP16><<<(unsigned)segments, kPackThreads, 0, st>>>(p); break;
            case DF11_VF_FP8_E4M3: pack_kernel<DF11_VF_FP8_E4M3><<<(unsigned)segments, kPackThreads, 0, st>>>(p); break;
            case DF11_VF_FP8_E5M2: pack_kernel<DF11_VF_FP8_E5M2><<<(unsigned)segments, kPackThreads, 0, st>>>(p); break;
            default: pack_kernel<DF11_VF_BF16><<<(unsigned)segments, kPackThreads, 0, st>>>(p); break;
        }
        DF11_TRY(cudaGetLastError(), "pack launch");
        launches++;
        const uint64_t groups = (chunks + 7) / 8;
        unsigned g = (unsigned)((groups + 255) / 256);
        if (g > (unsigned)sms * 8) g = sms * 8;
        if (g == 0) g = 1;
        gaps_kernel<<<g, 256, 0, st>>>(gapv, chunks, dst->gaps);
        DF11_TRY(cudaGetLastError(), "gaps launch");
        launches++;
    }
#undef DF11_TRY
    df11_count_launches(launches);
    return DF11_OK;
}
