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

// b of the format's LUTs (0 = 8, the paper's byte tables).
__host__ __device__ __forceinline__ uint32_t lut_bits_of(const df11_device_tensor &t) {
#ifdef DF11_LB8_ONLY
    return 8u;                                   // A/B knob (register-pressure experiment)
#else
    return t.lut_bits ? t.lut_bits : 8u;
#endif
}

// Value formats (df11.h DF11_VF_*, R25): M mantissa bits, E exponent bits, residual R = 1 + M bits in
// PackedSignMantissa (load_residual), words of 2 (BF16/FP16) or 1 (FP8) bytes.
struct VF {
    uint32_t M, E, R, emask, word_bytes;
};
__host__ __device__ constexpr VF vf_of(uint32_t value_format) {
    switch (value_format) {
        case DF11_VF_FP16: return {10, 5, 11, 31, 2};
        case DF11_VF_FP8_E4M3: return {3, 4, 4, 15, 1};
        case DF11_VF_FP8_E5M2: return {2, 5, 3, 31, 1};
        default: return {7, 8, 8, 255, 2};
    }
}
// sign << (E + M) | exponent << M | mantissa from the residual r = sign << M | mantissa
__device__ __forceinline__ uint32_t compose_vf(const VF &f, uint32_t e, uint32_t r) {
    return ((r >> f.M) << (f.E + f.M)) | ((e & f.emask) << f.M) | (r & ((1u << f.M) - 1u));
}
// Residual of element i of a tensor of n elements (R25): R = 8 (BF16) byte i; R = 11 (FP16) byte i of the
// byte plane (low 8 bits) + the 3 high bits at bit 3i of the plane after roundup(n, 16) bytes; R < 8
// (FP8) R bits MSB-first at bit R*i.
__device__ __forceinline__ uint32_t load_residual(const VF &f, const uint8_t *__restrict__ psm, uint64_t i,
                                                  uint64_t n) {
    if (f.R == 8) return __ldg(psm + i);
    if (f.R == 11) {
        const uint64_t bit = 3ull * i;
        const uint8_t *p = psm + ((n + 15) & ~15ull) + (bit >> 3);
        const uint32_t v = ((uint32_t)__ldg(p) << 8) | __ldg(p + 1);   // 3 bits inside 2 bytes
        return (((v >> (13u - (uint32_t)(bit & 7))) & 7u) << 8) | __ldg(psm + i);
    }
    const uint64_t bit = (uint64_t)f.R * i;
    const uint8_t *p = psm + (bit >> 3);
    const uint32_t v = ((uint32_t)__ldg(p) << 16) | ((uint32_t)__ldg(p + 1) << 8) | __ldg(p + 2);
    return (v >> (24u - (uint32_t)(bit & 7) - f.R)) & ((1u << f.R) - 1u);
}
__device__ __forceinline__ void store_word(const VF &f, void *out, uint64_t i, uint32_t v) {
    if (f.word_bytes == 2) static_cast<uint16_t *>(out)[i] = (uint16_t)v;
    else static_cast<uint8_t *>(out)[i] = (uint8_t)v;
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
