// api.cu — the C ABI (include/df11.h): validation, kernel selection, launches, diagnostics.
//
// df11_decompress_block: all tensors of a transformer block are described in ONE
// __grid_constant__ Batch and decoded by ONE launch of the product kernel (decode_sp12.cu).  Tensors it
// does not specialise (format parameters other than T = 256, n = 8, or buffers not 16-byte aligned) go
// through the literal Algorithm 1 kernel (decode_alg1.cu), one launch per distinct T; the eligible rest
// of the batch still takes the product kernel (df11_last_kernel_mask reports which kernels ran).
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>

#include "decode_common.cuh"
#include "df11_internal.h"

namespace df11 {
cudaError_t launch_alg1(const Batch &bt, uint32_t T, size_t max_smem, cudaStream_t stream, uint64_t *launches);
cudaError_t launch_sp12(const Batch &bt, int device, cudaStream_t stream, uint64_t *launches);
bool fast_supports(const df11_device_tensor &t);
uint32_t fast_grid(uint32_t total_tiles, int num_sms);
}  // namespace df11

namespace {
thread_local char g_msg[512] = "";
thread_local int g_cuda_err = 0;
thread_local uint64_t g_launches = 0;
thread_local uint32_t g_kernel_mask = 0;   // bit 0: Algorithm 1 kernel ran, bit 1: product kernel ran

int g_max_smem[64];
int g_num_sms[64];
std::once_flag g_attr_once[64];

void device_attrs(int dev, int &max_smem, int &num_sms) {
    if (dev < 0 || dev >= 64) { max_smem = 48 * 1024; num_sms = 1; return; }
    std::call_once(g_attr_once[dev], [dev] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        g_max_smem[dev] = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms[dev] = v;
    });
    max_smem = g_max_smem[dev];
    num_sms = g_num_sms[dev];
}

df11_status cuda_fail(cudaError_t e, const char *what) {
    g_cuda_err = (int)e;
    std::snprintf(g_msg, sizeof(g_msg), "%s: %s", what, cudaGetErrorString(e));
    return DF11_E_CUDA;
}

df11_status validate(const df11_device_tensor &t, uint32_t idx) {
    char buf[160];
    auto bad = [&](const char *why) {
        std::snprintf(buf, sizeof(buf), "descriptor %u: %s", idx, why);
        return df11_fail(DF11_E_INVALID_ARGUMENT, buf);
    };
    if (t.reserved != 0) return bad("reserved field must be 0");
    if (t.value_format > DF11_VF_FP8_E5M2) return bad("bad value_format");
    if (t.lut_bits > 16) return bad("lut_bits must be in [1, 16] (0 = 8)");
    if (t.num_elements >= (1ull << 32)) return df11_fail(DF11_E_TOO_LARGE, "N >= 2^32");
    if (t.num_elements == 0) return DF11_OK;                     // empty tensor: no-op (R11)
    if (t.B == 0) return bad("B == 0 with N > 0");
    if (t.T < 32 || t.T > 1024 || t.T % 32) return bad("T must be a multiple of 32 in [32, 1024]");
    if (t.n < 4 || t.n > 32) return bad("n must be in [4, 32]");
    if (t.lut_entry_bytes != 1 && t.lut_entry_bytes != 2) return bad("lut_entry_bytes must be 1 or 2");
    if (t.k == 0) return bad("k == 0 with N > 0");
    if (t.lut_entry_bytes == 1 && t.k > 17) return bad("narrow LUTs allow at most 17 tables");
    // a codebook of <= 256 symbols has <= 255 internal nodes, so <= 256 tables; the bound also keeps
    // every LUT byte offset k * 2^b * entry_bytes (<= 32 MB) inside 32-bit arithmetic in the kernels
    if (t.k > 256) return bad("at most 256 LUTs");
    if ((uint64_t)t.B * t.T * t.n * 8 > (uint64_t)t.num_elements * 32 + (uint64_t)t.T * t.n * 8)
        return bad("B too large for N (codes are at most 32 bits)");
    if (!t.encoded_exponent || !t.packed_sign_mantissa || !t.gaps || !t.luts || !t.code_lengths ||
        !t.block_output_pos || !t.out)
        return bad("NULL device pointer");
    return DF11_OK;
}
}  // namespace

extern "C" df11_status df11_fail(df11_status st, const char *msg) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", msg ? msg : "");
    return st;
}

extern "C" void df11_plan_cta_ranges(const uint32_t *entry_start, uint32_t count, uint32_t grid,
                                     uint32_t switch_tiles, uint32_t *cta_start) {
    // W(x) = x + switch_tiles * #{entry starts e, 0 < e <= x}; boundary c is the first x with
    // W(x) >= c * W(total) / grid, so a boundary snaps to an entry start when its target falls inside
    // that start's jump, and a CTA whose range holds an entry start gets switch_tiles fewer tiles.
    if (!grid) return;
    const uint32_t total = count ? entry_start[count] : 0;
    const uint64_t P = switch_tiles;
    const uint64_t wtot = (uint64_t)total + P * (count ? count - 1 : 0);
    uint32_t ei = 1;                                // next entry start not yet counted
    for (uint32_t c = 0; c <= grid; c++) {
        const uint64_t target = wtot * c / grid;
        while (ei < count && (uint64_t)entry_start[ei] + P * ei <= target) ei++;
        uint64_t x = target - P * (ei - 1);         // entries 1..ei-1 counted
        if (ei < count) x = std::min<uint64_t>(x, entry_start[ei]);
        cta_start[c] = (uint32_t)std::min<uint64_t>(x, total);
    }
    cta_start[0] = 0;
    cta_start[grid] = total;
}

namespace {
// Product-kernel launch for tensors ts[idx[0..n)] (all fast_supports, non-empty).
df11_status launch_fast_batch(const df11_device_tensor *ts, const uint32_t *idx, uint32_t n, int num_sms,
                              int dev, cudaStream_t stream, uint32_t max_ctas) {
    static thread_local df11::Batch bt;   // ~12 KB: keep it off the stack
    // Tile schedule (the block-batched launcher).  CTA c of the persistent kernel walks a
    // contiguous global tile range and rebuilds its SMEM decode tables at every tensor boundary inside
    // it.  Small tensors (biases, norm scales) would pile up in a few CTAs and turn them into
    // stragglers, so each small tensor is placed exactly at a CTA range boundary (big tensors are split
    // there), spreading them over distinct CTAs.
    std::memset(&bt, 0, sizeof(bt));
    constexpr uint32_t kSmall = 16;                     // tiles
    uint32_t big[DF11_MAX_BATCH], small[DF11_MAX_BATCH], nbig = 0, nsmall = 0, total = 0;
    for (uint32_t k = 0; k < n; k++) {
        const uint32_t i = idx[k];
        (ts[i].B < kSmall ? small[nsmall++] : big[nbig++]) = i;
        total += ts[i].B;
    }
    uint32_t G = df11::fast_grid(total, num_sms);
    // DF11_MAX_GRID (debug knob, read once): cap the persistent grid, e.g. so that a small input walks
    // many tiles per group under compute-sanitizer
    static const int max_grid = [] { const char *v = std::getenv("DF11_MAX_GRID"); return v ? std::atoi(v) : 0; }();
    if (max_grid > 0) G = std::min<uint32_t>(G, (uint32_t)max_grid);
    if (max_ctas > 0) G = std::min<uint32_t>(G, max_ctas);          // SM budget (overlap with compute)
    auto boundary = [&](uint32_t c) { return (uint32_t)(((uint64_t)total * c) / G); };
    uint32_t pos = 0, bi = 0, boff = 0;
    auto push = [&](uint32_t ti, uint32_t off, uint32_t cnt) {
        bt.t[bt.count] = ts[ti];
        bt.tile_start[bt.count] = pos;
        bt.tile_off[bt.count] = off;
        bt.count++;
        pos += cnt;
    };
    auto fill_big_until = [&](uint32_t target) {
        while (pos < target && bi < nbig) {
            const uint32_t left = ts[big[bi]].B - boff, take = std::min(left, target - pos);
            push(big[bi], boff, take);
            boff += take;
            if (boff == ts[big[bi]].B) { bi++; boff = 0; }
        }
    };
    for (uint32_t k = 0; k < nsmall; k++) {
        const uint32_t c = (uint32_t)(((uint64_t)(2 * k + 1) * G) / (2 * nsmall));
        fill_big_until(boundary(c));
        push(small[k], 0, ts[small[k]].B);
    }
    fill_big_until(total);
    bt.tile_start[bt.count] = pos;
    bt.total_tiles = pos;
    bt.grid = G;
    // Per-CTA tile ranges of equal work (df11_plan_cta_ranges): CTAs that switch tensors get fewer
    // tiles.  A switch costs 9 tiles (with the original table build 12 measured best: 3: +1.3 %, 8:
    // +2.9 %, 12: +3.1 % on the Llama-8B block vs uniform ranges; after the faster build, 9).
    if (G <= (uint32_t)df11::kMaxCta) {
#ifndef DF11_SWITCH_TILES
#define DF11_SWITCH_TILES 9
#endif
        // DF11_SWITCH_TILES_ENV (A/B knob, read once) overrides the compiled switch cost
        static const uint32_t sw = [] {
            const char *v = std::getenv("DF11_SWITCH_TILES_ENV");
            return v ? (uint32_t)std::atoi(v) : (uint32_t)DF11_SWITCH_TILES;
        }();
        df11_plan_cta_ranges(bt.tile_start, bt.count, G, sw, bt.cta_start);
        bt.cta_ranges = 1;
    }
    const uint32_t kpow[12] = {1u << 12, 1u << 4, 1u << 8, 8u, 0, 0, 0, 0, 0, 0, 0, 0};
    std::memcpy(bt.kpow, kpow, sizeof(kpow));
    cudaError_t e = df11::launch_sp12(bt, dev, stream, &g_launches);
    if (e != cudaSuccess) return cuda_fail(e, "fast decode launch");
    g_kernel_mask |= 2u;
    return DF11_OK;
}

// Algorithm 1 launches (one per distinct T) for tensors ts[idx[0..n)].
df11_status launch_alg1_batch(const df11_device_tensor *ts, const uint32_t *idx, uint32_t n, size_t max_smem,
                              cudaStream_t stream) {
    static thread_local df11::Batch bt;
    bool done[DF11_MAX_BATCH] = {};
    for (uint32_t a = 0; a < n; a++) {
        if (done[a]) continue;
        const uint32_t T = ts[idx[a]].T;
        std::memset(&bt, 0, sizeof(bt));
        uint32_t acc = 0;
        for (uint32_t b = a; b < n; b++) {
            const uint32_t j = idx[b];
            if (done[b] || ts[j].T != T) continue;
            done[b] = true;
            bt.t[bt.count] = ts[j];
            bt.tile_start[bt.count] = acc;
            acc += ts[j].B;
            bt.count++;
        }
        bt.tile_start[bt.count] = acc;
        bt.total_tiles = acc;
        cudaError_t e = df11::launch_alg1(bt, T, max_smem, stream, &g_launches);
        if (e != cudaSuccess) return cuda_fail(e, "Alg. 1 decode launch");
        g_kernel_mask |= 1u;
    }
    return DF11_OK;
}
}  // namespace

extern "C" df11_status df11_decompress_block_budget(const df11_device_tensor *ts, uint32_t count,
                                                    void *stream_v, int kernel, uint32_t max_ctas) {
    if (count > DF11_MAX_BATCH) return df11_fail(DF11_E_INVALID_ARGUMENT, "count > DF11_MAX_BATCH");
    if (count && !ts) return df11_fail(DF11_E_INVALID_ARGUMENT, "descriptor array is NULL");
    if (kernel < DF11_KERNEL_AUTO || kernel > DF11_KERNEL_FAST) return df11_fail(DF11_E_INVALID_ARGUMENT, "bad kernel");
    g_kernel_mask = 0;
    uint32_t fast_idx[DF11_MAX_BATCH], slow_idx[DF11_MAX_BATCH], nfast = 0, nslow = 0;
    uint64_t total = 0;
    for (uint32_t i = 0; i < count; i++) {
        df11_status st = validate(ts[i], i);
        if (st != DF11_OK) return st;
        if (!ts[i].num_elements) continue;
        total += ts[i].B;
        if (kernel != DF11_KERNEL_ALG1 && df11::fast_supports(ts[i])) fast_idx[nfast++] = i;
        else slow_idx[nslow++] = i;
    }
    if (total == 0) return DF11_OK;
    if (total >= (1ull << 32)) return df11_fail(DF11_E_TOO_LARGE, "batch has >= 2^32 format blocks");
    if (kernel == DF11_KERNEL_FAST && nslow)
        return df11_fail(DF11_E_UNSUPPORTED,
                         "fast kernel: a tensor is outside its parameter range (T=256, n=8 or T=128, n=16; 16-byte "
                         "aligned buffers, output aligned to its word size)");
    cudaStream_t stream = (cudaStream_t)stream_v;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int max_smem = 0, num_sms = 0;
    device_attrs(dev, max_smem, num_sms);
    if (nfast) {
        // one product launch per (chunk size, value format, byte tables or not): each takes its own
        // kernel build
        uint32_t grp[16][DF11_MAX_BATCH], cnt[16] = {};
        for (uint32_t k = 0; k < nfast; k++) {
            const df11_device_tensor &t = ts[fast_idx[k]];
            const uint32_t key = (df11::lut_bits_of(t) == 8 ? 0u : 8u) + (t.n == 16 ? 4u : 0u) + t.value_format;
            grp[key][cnt[key]++] = fast_idx[k];
        }
        for (uint32_t key = 0; key < 16; key++) {
            if (!cnt[key]) continue;
            df11_status st = launch_fast_batch(ts, grp[key], cnt[key], num_sms, dev, stream, max_ctas);
            if (st != DF11_OK) return st;
        }
    }
    if (nslow) return launch_alg1_batch(ts, slow_idx, nslow, (size_t)max_smem, stream);
    return DF11_OK;
}

extern "C" df11_status df11_decompress_block_ex(const df11_device_tensor *ts, uint32_t count, void *stream,
                                                int kernel) {
    return df11_decompress_block_budget(ts, count, stream, kernel, 0);
}

extern "C" df11_status df11_decompress_block(const df11_device_tensor *ts, uint32_t count, void *stream) {
    return df11_decompress_block_ex(ts, count, stream, DF11_KERNEL_AUTO);
}

extern "C" df11_status df11_decompress(const df11_device_tensor *t, void *stream) {
    if (!t) return df11_fail(DF11_E_INVALID_ARGUMENT, "descriptor is NULL");
    return df11_decompress_block_ex(t, 1, stream, DF11_KERNEL_AUTO);
}

extern "C" df11_status df11_decompress_host(const df11_host_tensor *h, const df11_device_tensor *d,
                                            void *host_out, void *stream_v) {
    if (!h || !d) return df11_fail(DF11_E_INVALID_ARGUMENT, "NULL argument");
    if (d->num_elements != h->num_elements || d->B != h->B || d->T != h->T || d->n != h->n || d->k != h->k ||
        d->lut_entry_bytes != h->lut_entry_bytes || d->value_format != h->value_format ||
        df11::lut_bits_of(*d) != (h->lut_bits ? h->lut_bits : 8u))
        return df11_fail(DF11_E_INVALID_ARGUMENT, "device descriptor does not match the host tensor");
    if (h->num_elements == 0) return DF11_OK;
    cudaStream_t s = (cudaStream_t)stream_v;
    struct { void *dst; const void *src; uint64_t n; } cp[] = {
        {(void *)d->encoded_exponent, h->encoded_exponent, h->encoded_exponent_bytes},
        {(void *)d->packed_sign_mantissa, h->packed_sign_mantissa, h->packed_sign_mantissa_bytes},
        {(void *)d->gaps, h->gaps, h->gaps_bytes},
        {(void *)d->luts, h->luts, h->luts_bytes},
        {(void *)d->code_lengths, h->code_lengths, 256},
        {(void *)d->block_output_pos, h->block_output_pos, 4ull * (h->B + 1)},
    };
    for (auto &c : cp) {
        if (!c.dst) return df11_fail(DF11_E_INVALID_ARGUMENT, "NULL device staging pointer");
        cudaError_t e = cudaMemcpyAsync(c.dst, c.src, c.n, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    }
    df11_status st = df11_decompress(d, stream_v);
    if (st != DF11_OK) return st;
    if (!host_out) return DF11_OK;                   // decode only: the result stays in d->out
    const uint64_t out_bytes = (uint64_t)df11::vf_of(h->value_format).word_bytes * h->num_elements;
    cudaError_t e = cudaMemcpyAsync(host_out, d->out, out_bytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
    return DF11_OK;
}

extern "C" df11_status df11_decompress_host_block(const df11_host_tensor *hs, const df11_device_tensor *ds,
                                                  void *const *host_outs, uint32_t count, void *stream_v,
                                                  void *copy_stream_v) {
    if (count && (!hs || !ds || !host_outs)) return df11_fail(DF11_E_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = (cudaStream_t)stream_v, cs = (cudaStream_t)copy_stream_v;
    if (cs == s) {                                   // one stream: no overlap, plain per-tensor calls
        for (uint32_t i = 0; i < count; i++) {
            df11_status st = df11_decompress_host(&hs[i], &ds[i], host_outs[i], stream_v);
            if (st != DF11_OK) return st;
        }
        return DF11_OK;
    }
    // H2D + decode of tensor i+1 on `stream` overlap the D2H of tensor i on `copy_stream` (PCIe is full
    // duplex); `stream` finally waits for the copies, so synchronising `stream` covers everything.
    // (Chunking tensors into block ranges was measured: no gain, the host link saturates at ~70 GB/s
    // of combined H2D + D2H traffic.)
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    df11_status st = DF11_OK;
    for (uint32_t i = 0; i < count && st == DF11_OK; i++) {
        const df11_host_tensor *h = &hs[i];
        const df11_device_tensor *d = &ds[i];
        if (h->num_elements && !host_outs[i]) { st = df11_fail(DF11_E_INVALID_ARGUMENT, "NULL host output"); break; }
        st = df11_decompress_host(h, d, nullptr, stream_v);   // H2D + decode
        if (st != DF11_OK || !h->num_elements) continue;
        if ((e = cudaEventRecord(ev, s)) != cudaSuccess || (e = cudaStreamWaitEvent(cs, ev, 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(host_outs[i], d->out,
                                 (uint64_t)df11::vf_of(h->value_format).word_bytes * h->num_elements,
                                 cudaMemcpyDeviceToHost, cs)) !=
                cudaSuccess)
            st = cuda_fail(e, "D2H copy");
    }
    // join the copy stream back into `stream` on every path (D2H copies already enqueued for earlier
    // tensors must be covered by a synchronisation of `stream` even when a later tensor failed)
    if ((e = cudaEventRecord(ev, cs)) != cudaSuccess || (e = cudaStreamWaitEvent(s, ev, 0)) != cudaSuccess) {
        if (st == DF11_OK) st = cuda_fail(e, "stream join");
    }
    cudaEventDestroy(ev);                            // released once the pending work completes
    return st;
}

extern "C" const char *df11_status_string(df11_status s) {
    switch (s) {
        case DF11_OK: return "DF11_OK";
        case DF11_E_INVALID_ARGUMENT: return "DF11_E_INVALID_ARGUMENT";
        case DF11_E_RESERVED_EXPONENT: return "DF11_E_RESERVED_EXPONENT";
        case DF11_E_LUT_OVERFLOW: return "DF11_E_LUT_OVERFLOW";
        case DF11_E_TOO_LARGE: return "DF11_E_TOO_LARGE";
        case DF11_E_CORRUPT: return "DF11_E_CORRUPT";
        case DF11_E_CUDA: return "DF11_E_CUDA";
        case DF11_E_ALLOC: return "DF11_E_ALLOC";
        case DF11_E_UNSUPPORTED: return "DF11_E_UNSUPPORTED";
    }
    return "DF11_E_UNKNOWN";
}

extern "C" df11_status df11_cuda_fail(int e, const char *what) { return cuda_fail((cudaError_t)e, what); }
extern "C" void df11_count_launches(uint64_t k) { g_launches += k; }
extern "C" int df11_last_cuda_error(void) { return g_cuda_err; }
extern "C" const char *df11_last_error_message(void) { return g_msg; }
extern "C" const char *df11_version(void) { return "df11-b200 0.2 (sm_100a; BF16 / FP16 / FP8 E4M3 / FP8 E5M2, b-bit LUTs)"; }
extern "C" uint32_t df11_last_kernel_mask(void) { return g_kernel_mask; }
extern "C" uint64_t df11_launch_count(int reset) {
    uint64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}
