/*
 * df11.h — C ABI of the B200-native DFloat11 library (arXiv 2504.11651).
 *
 * Citations: "P:n" = PAPER.md line n.  The bit-exact format is DESIGN.md §2; the readings where the
 * paper is silent are DESIGN.md §3 (R1..R24).
 *
 * Conventions
 *  - Every call returns df11_status; no C++ exception crosses the ABI.
 *  - Host encode calls allocate their outputs; free them with df11_host_tensor_free().
 *  - Device calls take device pointers OWNED BY THE CALLER (e.g. torch tensors) and a cudaStream_t
 *    (passed as void*; NULL = the legacy default stream).  They only enqueue work: device faults
 *    surface at the caller's next synchronisation (CUDA semantics).  They never allocate, never copy
 *    host<->device and are CUDA-graph capturable.
 *  - Robustness: malformed device metadata may produce wrong output but never an out-of-bounds
 *    access: every write is clipped to [BlockOutputPos[b], BlockOutputPos[b+1]) ∩ [0, N), LUT walks
 *    are bounded to ceil(32/b) levels and k tables, and every code step advances at least one bit.
 *  - Thread safety: no mutable global state except cached device attributes and the last CUDA error.
 */
#ifndef DF11_H
#define DF11_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DF11_OK = 0,
    DF11_E_INVALID_ARGUMENT = 1,   /* null pointer, bad T/n/mode, inconsistent descriptor */
    DF11_E_RESERVED_EXPONENT = 2,  /* exponent >= 240 present with lut_mode NARROW (R8) */
    DF11_E_LUT_OVERFLOW = 3,       /* > 16 child LUTs with lut_mode NARROW (R9) */
    DF11_E_TOO_LARGE = 4,          /* N >= 2^32 per tensor: BlockOutputPos is uint32 */
    DF11_E_CORRUPT = 5,            /* host-side metadata check failed */
    DF11_E_CUDA = 6,               /* launch/config error; see df11_last_cuda_error() */
    DF11_E_ALLOC = 7,              /* host allocation failed */
    DF11_E_UNSUPPORTED = 8         /* a forced kernel variant cannot handle these parameters */
} df11_status;

enum { DF11_LUT_AUTO = 0, DF11_LUT_NARROW = 1, DF11_LUT_WIDE = 2 };

/* Value formats (NEXT-4; DESIGN.md §2 and R25-R27).  The paper codes BF16; P:609 names
 * FP16 and FP8 as its limitation.  Every format is split the same way: the exponent field is the
 * Huffman symbol, and the residual r = sign << M | mantissa (R = 1 + M bits) is stored raw in
 * PackedSignMantissa: BF16 (R = 8) one byte per element, sign in bit 7, mantissa in bits 6..0 (the
 * paper's layout); FP16 (R = 11) the low 8 bits of r as a byte plane of roundup(N, 16) bytes,
 * then the 3 high bits (sign, m9, m8) MSB-first at bits [3i, 3i + 3) of a plane after it; FP8 (R = 4 / 3)
 * r MSB-first at bits [R*i, R*i + R).
 *   BF16      16-bit words, exponent bits 14..7  (8), R = 8
 *   FP16      16-bit words, exponent bits 14..10 (5), R = 11
 *   FP8_E4M3  8-bit words,  exponent bits 6..3   (4), R = 4
 *   FP8_E5M2  8-bit words,  exponent bits 6..2   (5), R = 3 */
enum { DF11_VF_BF16 = 0, DF11_VF_FP16 = 1, DF11_VF_FP8_E4M3 = 2, DF11_VF_FP8_E5M2 = 3 };

/* lut_bits (encoder option): b of the b-bit hierarchical LUTs (App. I.2; 0 or 8 = the paper's 256-entry
 * tables), or DF11_LUT_BITS_MONOLITHIC: one table of 2^L entries (App. I.1),
 * legal when the longest code L <= 16 (R28). */
#define DF11_LUT_BITS_MONOLITHIC 255u

/* Kernel selection for df11_decompress_block_ex (AUTO = fast kernel when eligible). */
enum { DF11_KERNEL_AUTO = 0, DF11_KERNEL_ALG1 = 1, DF11_KERNEL_FAST = 2 };

#define DF11_MAX_BATCH 64          /* tensors per df11_decompress_block call */

typedef struct {
    uint32_t threads_per_block;    /* T: multiple of 32 in [32, 1024]; default 256 (R17) */
    uint32_t bytes_per_thread;     /* n: [4, 32]; default 8 */
    uint32_t lut_mode;             /* DF11_LUT_AUTO | NARROW (paper format) | WIDE */
    uint32_t num_threads;          /* host encoder threads; 0 = all hardware threads */
    uint32_t value_format;         /* DF11_VF_*; 0 = BF16 (the paper) */
    uint32_t lut_bits;             /* b in [1, 16], 0 = 8 (the paper), or DF11_LUT_BITS_MONOLITHIC */
} df11_encode_opts;

/* Host-side DF11 tensor.  All arrays are library-owned, zero-padded as stated. */
typedef struct {
    uint64_t num_elements;                 /* N */
    uint64_t encoded_bits;                 /* sum of code lengths */
    uint32_t T, n, B, k;                   /* threads/block, bytes/thread, #blocks, #LUTs */
    uint32_t lut_entry_bytes;              /* 1 = narrow (paper), 2 = wide (R8) */
    uint32_t max_code_len;                 /* L <= 32 */
    uint32_t value_format;                 /* DF11_VF_* */
    uint32_t lut_bits;                     /* b: every LUT has 2^b entries (8 = the paper) */
    uint8_t  code_lengths[256];            /* CodeLengths */
    uint8_t  *luts;              uint64_t luts_bytes;                  /* k*2^b*lut_entry_bytes; table 0 = root */
    uint8_t  *encoded_exponent;  uint64_t encoded_exponent_bytes;      /* B*T*n + 16 */
    uint8_t  *packed_sign_mantissa; uint64_t packed_sign_mantissa_bytes; /* FP8: roundup(R*roundup(N,16)/8,16) + 16;
                                                                            BF16: roundup(N,16) + 16; FP16:
                                                                            roundup(N,16) + roundup(3*roundup(N,16)/8,16) + 16 */
    uint8_t  *gaps;              uint64_t gaps_bytes;                  /* roundup(ceil(5BT/8),16) + 16 */
    uint32_t *block_output_pos;                                        /* B+1 entries, [B] = N */
} df11_host_tensor;

/* Device view of one DF11 tensor.  Every pointer is a device pointer owned by the caller; arrays
 * must have the sizes of df11_host_tensor (including the zero padding).  `code_lengths` points at
 * 256 device bytes.  `out` receives N words of the value format (16-bit BF16/FP16, 8-bit FP8; 16-byte
 * alignment recommended: the fast kernel then writes 128-bit stores). */
typedef struct {
    const uint8_t  *encoded_exponent;
    const uint8_t  *packed_sign_mantissa;
    const uint8_t  *gaps;
    const uint8_t  *luts;
    const uint8_t  *code_lengths;
    const uint32_t *block_output_pos;
    void           *out;
    uint64_t        num_elements;
    uint32_t        T, n, B, k, lut_entry_bytes;
    uint32_t        value_format;          /* DF11_VF_* (0 = BF16) */
    uint32_t        lut_bits;              /* b in [1, 16]; 0 = 8 (the paper) */
    uint32_t        reserved;              /* must be 0 */
} df11_device_tensor;

/* ---- host encoder --------------------------------------
 * df11_encode: one tensor of N words of opts->value_format (BF16 by default: uint16 bit patterns;
 * FP16 uint16; FP8 uint8; row-major) -> DF11 with a per-tensor codebook.  opts may be NULL
 * (defaults).  N = 0 is legal (B = 0).  Errors: DF11_E_INVALID_ARGUMENT (bad options, or a monolithic
 * table with L > 16), DF11_E_RESERVED_EXPONENT / DF11_E_LUT_OVERFLOW (NARROW only), DF11_E_TOO_LARGE,
 * DF11_E_ALLOC.  On error *out is left zeroed. */
df11_status df11_encode(const void *values, uint64_t n_elems, const df11_encode_opts *opts,
                        df11_host_tensor *out);

/* df11_encode_group: `count` tensors; shared_codebook != 0 builds one codebook from the summed
 * histogram of the group (R5: "a Huffman tree based on the distribution of exponents in model
 * weights") and stores a copy of it in every output; otherwise one codebook per tensor. */
df11_status df11_encode_group(const void *const *tensors, const uint64_t *n_elems, uint32_t count,
                              const df11_encode_opts *opts, int shared_codebook, df11_host_tensor *outs);

void df11_host_tensor_free(df11_host_tensor *t);

/* ---- device decoder (rows a1-a9; Alg. 1; block batching P:153-157) --------------------
 * df11_decompress: one tensor, one launch.  df11_decompress_block: every tensor of a transformer
 * block in ONE launch (count <= DF11_MAX_BATCH; empty tensors allowed).  On a validation error the
 * message names the offending descriptor index (df11_last_error_message()).  `stream` is a
 * cudaStream_t.  Stream semantics: the product kernel is launched as a programmatic dependent launch,
 * so when it directly follows another product-kernel decode on the same stream it may start reading
 * its OWN inputs (LUTs, CodeLengths, BlockOutputPos, the first stream chunks) while that decode is
 * still running; it writes its outputs only after that decode has completed (griddepcontrol.wait).
 * Every other predecessor (copies, events, other kernels) is waited for in full, as usual.  A decode
 * must therefore not take as input a buffer that the immediately preceding decode on its stream
 * writes (no DF11 input is ever a decode output). */
df11_status df11_decompress(const df11_device_tensor *t, void *stream);
df11_status df11_decompress_block(const df11_device_tensor *ts, uint32_t count, void *stream);
/* Same with an explicit kernel: DF11_KERNEL_ALG1 (literal Alg. 1, any valid T/n) or DF11_KERNEL_FAST
 * (persistent sm_100a kernel, every value format and LUT width; DF11_E_UNSUPPORTED if a tensor is
 * outside its parameter range: T = 256, n = 8 or T = 128, n = 16, encoded_exponent / gaps /
 * packed_sign_mantissa 16-byte aligned, out aligned to its word size, residual stream < 4 GiB, i.e.
 * FP16 tensors below ~3.1 G elements).  With
 * DF11_KERNEL_AUTO the batch is split: tensors in that range take ONE product-kernel launch, the rest
 * the Alg. 1 kernel (one launch per distinct T); df11_last_kernel_mask() says which ran. */
df11_status df11_decompress_block_ex(const df11_device_tensor *ts, uint32_t count, void *stream,
                                     int kernel);
/* Same with an SM budget (NEXT-1, decode/compute overlap): the product kernel runs at
 * most `max_ctas` persistent CTAs (one per SM; 0 = one per SM of the device), so that a decode
 * prefetched on a side stream leaves the other SMs to the GEMMs of the current block.  Results are
 * identical for every budget.  `max_ctas` does not affect Algorithm 1 launches. */
df11_status df11_decompress_block_budget(const df11_device_tensor *ts, uint32_t count, void *stream,
                                         int kernel, uint32_t max_ctas);

/* ---- launcher planning (host; used by df11_decompress_block, exported for tests) ----------------
 * df11_plan_cta_ranges: tile ranges of the persistent decode grid.  entry_start[0..count] are the
 * exclusive prefix sums of the batch entries' format-block counts (entry_start[count] = total);
 * CTA c walks [cta_start[c], cta_start[c+1]) (cta_start has grid + 1 entries, non-decreasing,
 * cta_start[0] = 0, cta_start[grid] = total).  Ranges have equal work, where an entry start strictly
 * inside a range costs switch_tiles tiles (the CTA rebuilds its decode table there). */
void df11_plan_cta_ranges(const uint32_t *entry_start, uint32_t count, uint32_t grid, uint32_t switch_tiles,
                          uint32_t *cta_start);

/* ---- end-to-end from host memory --------------------------------------------------------------
 * df11_decompress_host: copies the host arrays of `h` into the caller-provided device staging
 * buffers described by `d` (same sizes as h's arrays), decodes into d->out and copies the result
 * into `host_out` (N words of the value format; pinned memory recommended; NULL = leave the result in
 * d->out), all enqueued on `stream`.
 * Returns after enqueueing; synchronise the stream before reading host_out. */
df11_status df11_decompress_host(const df11_host_tensor *h, const df11_device_tensor *d,
                                 void *host_out, void *stream);

/* df11_decompress_host_block: df11_decompress_host for `count` tensors (a transformer block),
 * pipelined over two caller-owned streams: the H2D copies and decode of tensor i+1 run on `stream`
 * while the BF16 result of tensor i is copied back on `copy_stream` (PCIe is full duplex).  On return
 * everything is enqueued and `stream` waits for the last copy, so synchronising `stream` suffices.
 * host_outs[i] may be NULL for an empty tensor; copy_stream == stream degrades to sequential calls.
 * Errors: as df11_decompress_host; DF11_E_CUDA for stream/event failures. */
df11_status df11_decompress_host_block(const df11_host_tensor *hs, const df11_device_tensor *ds,
                                       void *const *host_outs, uint32_t count, void *stream,
                                       void *copy_stream);

/* ---- device encoder (format P:97; Table `time` P:471-486) -------
 * The same bytes as df11_encode, produced on the GPU in three steps so that the caller owns every
 * device allocation:
 *   1. df11_histogram_device   exponent histogram of a device BF16 tensor (one launch; accumulates).
 *   2. df11_encode_plan_create codebook (Huffman, 32-bit cap, canonical codes, LUTs) and buffer sizes,
 *                              on the host, from the histogram(s) copied back by the caller.
 *   3. df11_encode_device      bit packing, PackedSignMantissa, Gaps and BlockOutputPos on the GPU
 *                              (single pass with a decoupled look-back scan of per-segment bit counts).
 * The output is byte-identical to df11_encode with the same options and histogram. */

/* Device buffers written by df11_encode_device; sizes are the plan's *_bytes fields.  All pointers
 * are caller-owned device pointers, 16-byte aligned. */
typedef struct {
    uint8_t  *encoded_exponent;       /* plan.encoded_exponent_bytes */
    uint8_t  *packed_sign_mantissa;   /* plan.packed_sign_mantissa_bytes */
    uint8_t  *gaps;                   /* plan.gaps_bytes */
    uint8_t  *luts;                   /* plan.luts_bytes (>= 1) */
    uint8_t  *code_lengths;           /* 256 */
    uint32_t *block_output_pos;       /* plan.B + 1 entries */
} df11_device_buffers;

/* Codebook + geometry of one tensor, built on the host.  `luts` is library-owned host memory: free
 * the plan with df11_encode_plan_free.  Every value format and lut_bits of df11_encode_opts. */
typedef struct {
    uint64_t num_elements;            /* N = sum of tensor_hist */
    uint64_t encoded_bits;            /* sum over the tensor of code lengths */
    uint32_t T, n, B, k, lut_entry_bytes, max_code_len;
    uint32_t lut_bits;                /* b (the plan's tables have 2^b entries) */
    uint32_t value_format;            /* DF11_VF_* of the words df11_encode_device reads */
    uint8_t  code_lengths[256];
    uint32_t codes[256];              /* canonical codes, right-aligned, MSB-first when emitted */
    uint8_t  *luts;             uint64_t luts_bytes;
    uint64_t encoded_exponent_bytes, packed_sign_mantissa_bytes, gaps_bytes;
    uint64_t workspace_bytes;         /* device scratch df11_encode_device needs */
} df11_encode_plan;

/* Adds the exponent histogram of d_values[0..n) (words of value_format, DF11_VF_*) to d_hist (256
 * uint64 counters in device memory; zero them first).  d_values must be aligned to its word size.
 * Enqueues on `stream`; does not synchronise. */
df11_status df11_histogram_device(const void *d_values, uint64_t n, uint32_t value_format, uint64_t *d_hist,
                                  void *stream);

/* codebook_hist: host histogram the codebook is built from (the tensor's own, or the sum over a
 * group for a shared codebook, R5).  tensor_hist: the tensor's own host histogram (NULL = same as
 * codebook_hist); it fixes N and the encoded size.  Errors: every exponent in tensor_hist must have a
 * code (DF11_E_INVALID_ARGUMENT), RESERVED_EXPONENT / LUT_OVERFLOW with NARROW, TOO_LARGE (N >= 2^32).
 * On error *plan is zeroed. */
df11_status df11_encode_plan_create(const uint64_t *codebook_hist, const uint64_t *tensor_hist,
                                    const df11_encode_opts *opts, df11_encode_plan *plan);
void df11_encode_plan_free(df11_encode_plan *plan);

/* Encodes d_values[0..plan->num_elements) (words of plan->value_format) into `dst` on `stream`
 * (memsets + kernels only; CodeLengths and LUTs travel as kernel parameters, so the call never waits
 * for the stream).  d_values must hold exactly the tensor the plan's tensor_hist was taken from; a
 * mismatch yields a wrong encoding but no out-of-bounds access (the bit packer clips to the planned
 * sizes).  `workspace`: >= plan->workspace_bytes of device memory, 16-byte aligned.
 * Returns after enqueueing. */
df11_status df11_encode_device(const void *d_values, const df11_encode_plan *plan,
                               const df11_device_buffers *dst, void *workspace, uint64_t workspace_bytes,
                               void *stream);

/* ---- diagnostics ------------------------------------------------------------------------------ */
const char *df11_status_string(df11_status s);
int         df11_last_cuda_error(void);            /* cudaError_t of the last failing CUDA call */
const char *df11_last_error_message(void);         /* thread-local, human readable */
const char *df11_version(void);
/* Number of kernel launches enqueued by this thread since the last reset (for bench accounting). */
uint64_t    df11_launch_count(int reset);
/* Kernels the calling thread's last df11_decompress* call launched: bit 0 = Alg. 1 kernel, bit 1 =
 * product kernel (0 = nothing launched, e.g. an empty batch or a validation error). */
uint32_t    df11_last_kernel_mask(void);

#ifdef __cplusplus
}
#endif
#endif /* DF11_H */
