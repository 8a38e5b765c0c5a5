// decode_alg1.cu — the paper's two-phase kernel, Algorithm 1 "DF11ToBF16", written
// literally for sm_100a.  It is the baseline the product kernel (decode_sp12.cu) is measured against,
// and the fallback for format parameters that kernel does not specialise (any T multiple of 32, any n
// in [4, 32], narrow or wide LUTs of any size and any b, every value format).
//
//   one CTA per format block b, blockDim = T
//   SRAM: EncodedExponent_b (+4 spill bytes), LUT_1..LUT_k, CodeLengths
//   phase 1: per-thread LUT walk + count, BitOffset from Gaps[bT+t]
//   Blelloch work-efficient exclusive scan of the counts
//   phase 2: re-decode, compose with PackedSignMantissa[pos] into a WriteBuffer
//            (value formats other than BF16: the residual is the R-bit field at bit R*pos, R25)
//   one batch of coalesced writes of WriteBuffer to Outputs[BOP[b]..BOP[b+1])
//
// Robustness (df11.h): positions are clipped to [BOP[b], BOP[b+1]) ∩ [0, N) and to the buffer size;
// LUT walks stop after ceil(32/b) levels or on a child index >= k; a zero code length advances 32 bits.
#include "decode_common.cuh"

namespace df11 {

template <bool kLutInSmem, bool kUseWriteBuffer>
__global__ void __launch_bounds__(1024) alg1_kernel(const __grid_constant__ Batch bt) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t g_tile = blockIdx.x;
    const int ti = tensor_of_tile(bt, g_tile);
    const df11_device_tensor &ts = bt.t[ti];
    const uint32_t b = g_tile - bt.tile_start[ti];
    const uint32_t T = ts.T, n = ts.n, k = ts.k, eb = ts.lut_entry_bytes;
    const uint32_t lb = lut_bits_of(ts), tsize = 1u << lb;       // b-bit tables (App. I.2)
    const VF vf = vf_of(ts.value_format);
    const uint32_t t = threadIdx.x;
    const uint64_t N = ts.num_elements;

    // ---- SRAM carve-up
    const uint32_t lut_bytes = kLutInSmem ? k * tsize * eb : 0u;
    uint8_t *s_lut = smem;                                         // k*2^b*eb
    uint8_t *s_len = smem + ((lut_bytes + 15u) & ~15u);            // 256
    uint8_t *s_chunk = s_len + 256;                                // T*n + 4 (rounded to 16)
    uint32_t *s_count = (uint32_t *)(s_chunk + ((T * n + 4u + 15u) & ~15u));  // pow2 >= T
    uint32_t p2 = 1;
    while (p2 < T) p2 <<= 1;
    uint16_t *s_wbuf = (uint16_t *)(s_count + p2);                 // 8nT (worst case: 1-bit codes)

    // Load EncodedExponent_b into SRAM: T*n bytes plus the 4 spill bytes the last thread's
    // window may read (the array is zero-padded by 16 bytes, R16).
    const uint8_t *enc = ts.encoded_exponent + (uint64_t)b * T * n;
    for (uint32_t i = t; i < T * n + 4u; i += T) s_chunk[i] = __ldg(enc + i);
    // Load LUT_1..LUT_k and CodeLengths.
    if (kLutInSmem)
        for (uint32_t i = t; i < lut_bytes; i += T) s_lut[i] = __ldg(ts.luts + i);
    for (uint32_t i = t; i < 256u; i += T) s_len[i] = __ldg(ts.code_lengths + i);
    __syncthreads();

    const uint8_t *lut = kLutInSmem ? s_lut : ts.luts;
    auto lut_at = [&](uint32_t table, uint32_t idx) -> uint32_t {
        uint32_t off = (table << lb) + idx;
        if (eb == 1) return kLutInSmem ? lut[off] : __ldg(lut + off);
        uint32_t lo = kLutInSmem ? lut[2 * off] : __ldg(lut + 2 * off);
        uint32_t hi = kLutInSmem ? lut[2 * off + 1] : __ldg(lut + 2 * off + 1);
        return lo | (hi << 8);
    };
    const uint32_t ptr_threshold = eb == 1 ? 240u : 256u;

    // "Read the next 4 bytes ... starting from the BitOffset-th bit" (R2): big-endian window.
    auto window = [&](uint32_t bit_offset) -> uint32_t {
        const uint8_t *p = s_chunk + t * n + (bit_offset >> 3);
        uint64_t v = ((uint64_t)p[0] << 32) | ((uint64_t)p[1] << 24) | ((uint64_t)p[2] << 16) |
                     ((uint64_t)p[3] << 8) | (uint64_t)p[4];
        return (uint32_t)(v >> (8u - (bit_offset & 7u)));
    };
    // LUT walk: Exponent >= 240 is a pointer to LUT_{257-Exponent} (narrow), >= 256 (wide).
    // Level i reads window bits [b(i-1), bi) (b = 8: Byte_i), zero-extended past bit 32 (R28).
    const uint32_t levels = (32u + lb - 1u) / lb;
    auto level_idx = [&](uint32_t w, uint32_t i) -> uint32_t {    // i: 1-based level
        const uint64_t w64 = (uint64_t)w << 32;
        return (uint32_t)(w64 >> (64u - lb * i)) & (tsize - 1u);
    };
    auto decode_one = [&](uint32_t w, uint32_t &len) -> uint32_t {
        uint32_t e = lut_at(0, level_idx(w, 1));
        uint32_t i = 1;
        while (e >= ptr_threshold) {
            i++;
            uint32_t table = eb == 1 ? 256u - e : e - 256u;
            if (i > levels || table >= k) { e = 0; break; }        // malformed: bounded
            e = lut_at(table, level_idx(w, i));
        }
        e &= vf.emask;                                             // a symbol is an exponent field
        len = s_len[e];
        if (len == 0) len = 32;                                    // malformed: still advances
        return e;
    };

    const uint32_t chunk_bits = 8u * n;
    const uint32_t gap = load_gap(ts.gaps, (uint64_t)b * T + t);

    // ---- Phase 1
    uint32_t count = 0;
    for (uint32_t bit_offset = gap; bit_offset < chunk_bits;) {
        uint32_t len;
        decode_one(window(bit_offset), len);
        bit_offset += len;
        count++;
    }
    // ---- Blelloch scan: exclusive prefix of NumElements over the block
    s_count[t] = count;
    for (uint32_t i = T + t; i < p2; i += T) s_count[i] = 0;
    __syncthreads();
    for (uint32_t d = 1; d < p2; d <<= 1) {                        // up-sweep
        for (uint32_t j = t; j < p2 / (2 * d); j += T) {
            uint32_t ai = (2 * j + 1) * d - 1, bi = (2 * j + 2) * d - 1;
            s_count[bi] += s_count[ai];
        }
        __syncthreads();
    }
    if (t == 0) s_count[p2 - 1] = 0;
    __syncthreads();
    for (uint32_t d = p2 >> 1; d >= 1; d >>= 1) {                  // down-sweep
        for (uint32_t j = t; j < p2 / (2 * d); j += T) {
            uint32_t ai = (2 * j + 1) * d - 1, bi = (2 * j + 2) * d - 1;
            uint32_t tmp = s_count[ai];
            s_count[ai] = s_count[bi];
            s_count[bi] += tmp;
        }
        __syncthreads();
    }
    const uint64_t bop_lo = min((uint64_t)ts.block_output_pos[b], N);
    uint64_t bop_hi = min((uint64_t)ts.block_output_pos[b + 1], N);
    if (bop_hi < bop_lo) bop_hi = bop_lo;
    if (bop_hi - bop_lo > (uint64_t)chunk_bits * T) bop_hi = bop_lo + (uint64_t)chunk_bits * T;
    uint64_t pos = bop_lo + s_count[t];                           // ThreadOutputPos[t]

    // ---- Phase 2
    for (uint32_t bit_offset = gap; bit_offset < chunk_bits;) {
        uint32_t len;
        uint32_t e = decode_one(window(bit_offset), len);
        if (pos < bop_hi) {
            const uint16_t v = (uint16_t)compose_vf(vf, e, load_residual(vf, ts.packed_sign_mantissa, pos, ts.num_elements));
            if (kUseWriteBuffer) s_wbuf[pos - bop_lo] = v;
            else store_word(vf, ts.out, pos, v);
        }
        bit_offset += len;
        pos++;
    }
    // ---- coalesced write-back
    if (kUseWriteBuffer) {
        __syncthreads();
        const uint32_t cnt = (uint32_t)(bop_hi - bop_lo);
        for (uint32_t i = t; i < cnt; i += T) store_word(vf, ts.out, bop_lo + i, s_wbuf[i]);
    }
}

// Host side: one launch per distinct T in the batch (blockDim must equal T).
size_t alg1_smem_bytes(uint32_t T, uint32_t n, size_t lut_bytes, bool lut_in_smem, bool wbuf) {
    uint32_t p2 = 1;
    while (p2 < T) p2 <<= 1;
    size_t lut = lut_in_smem ? ((lut_bytes + 15) & ~(size_t)15) : 0;
    size_t s = lut + 256 + (((size_t)T * n + 4 + 15) & ~(size_t)15) + (size_t)p2 * 4;
    if (wbuf) s += (size_t)8 * n * T * 2;
    return s;
}

cudaError_t launch_alg1(const Batch &bt, uint32_t T, size_t max_smem, cudaStream_t stream, uint64_t *launches) {
    if (bt.total_tiles == 0) return cudaSuccess;
    uint32_t n_max = 0;
    size_t lut_max = 0;
    for (uint32_t i = 0; i < bt.count; i++) {
        if (bt.t[i].B == 0) continue;
        n_max = max(n_max, bt.t[i].n);
        lut_max = max(lut_max, (size_t)bt.t[i].k * ((size_t)1 << lut_bits_of(bt.t[i])) * bt.t[i].lut_entry_bytes);
    }
    bool lut_smem = true, wbuf = true;
    size_t need = alg1_smem_bytes(T, n_max, lut_max, true, true);
    if (need > max_smem) { wbuf = false; need = alg1_smem_bytes(T, n_max, lut_max, true, false); }
    if (need > max_smem) { lut_smem = false; wbuf = true; need = alg1_smem_bytes(T, n_max, 0, false, true); }
    if (need > max_smem) { wbuf = false; need = alg1_smem_bytes(T, n_max, 0, false, false); }
    if (need > max_smem) return cudaErrorInvalidConfiguration;
    void (*kern)(const Batch) = nullptr;
    if (lut_smem && wbuf) kern = alg1_kernel<true, true>;
    else if (lut_smem) kern = alg1_kernel<true, false>;
    else if (wbuf) kern = alg1_kernel<false, true>;
    else kern = alg1_kernel<false, false>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    if (err != cudaSuccess) return err;
    kern<<<bt.total_tiles, T, need, stream>>>(bt);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace df11
