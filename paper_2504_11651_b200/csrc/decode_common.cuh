// decode_common.cuh — device-side batch descriptor and small helpers shared by the decode kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "df11.h"

namespace df11 {

// One launch decodes up to DF11_MAX_BATCH tensors ("decompress all DFloat11 weight matrices
// within a transformer block as a single batch").  Passed by value as a __grid_constant__ kernel
// parameter: no workspace, no H2D copy, graph-capturable.
constexpr int kMaxEntries = 2 * DF11_MAX_BATCH;   // a tensor may be split into several tile ranges
constexpr int kMaxCta = 256;                      // persistent grid bound for per-CTA tile ranges

struct Batch {
    df11_device_tensor t[kMaxEntries];
    uint32_t tile_start[kMaxEntries + 1];      // exclusive prefix of the entries' tile counts
    uint32_t tile_off[kMaxEntries];            // first format block of entry i within its tensor
    uint32_t count;
    uint32_t total_tiles;
    uint32_t grid;                             // CTAs the launcher will use (fast kernel)
    uint32_t cta_ranges;                       // 1: CTA c walks tiles [cta_start[c], cta_start[c+1])
    uint32_t cta_start[kMaxCta + 1];
    // powers of two used as IMAD multipliers (field extraction on the FMA pipe); read from the
    // constant bank so the compiler cannot strength-reduce them into ALU shifts (set by the launcher)
    uint32_t kpow[12];
};

// Tensor owning global tile `g` (binary search over tile_start).
__device__ __forceinline__ int tensor_of_tile(const Batch &bt, uint32_t g) {
    int lo = 0, hi = (int)bt.count - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (bt.tile_start[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Alg. 1 compose: (Sign << 8) | (Exponent << 7) | Mantissa with Sign = Byte & 0x80.
__device__ __forceinline__ uint16_t compose(uint32_t exponent, uint32_t psm) {
    return (uint16_t)(((psm & 0x80u) << 8) | (exponent << 7) | (psm & 0x7Fu));
}

// 5-bit gap field g, MSB-first at bits [5g, 5g+5) (R12).
__device__ __forceinline__ uint32_t load_gap(const uint8_t *__restrict__ gaps, uint64_t g) {
    uint64_t bit = 5ull * g;
    uint32_t hi = __ldg(gaps + (bit >> 3));
    uint32_t lo = __ldg(gaps + (bit >> 3) + 1);
    uint32_t two = (hi << 8) | lo;
    return (two >> (11 - (uint32_t)(bit & 7))) & 31u;
}

}  // namespace df11
