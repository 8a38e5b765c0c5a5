/*
 * df11_oracle.c — plain, slow, obviously-correct CPU oracle for DFloat11 (arXiv 2504.11651).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (paper_2504_11651_b200/) never
 * does, and this file shares no code, header, table or constant generator with it.
 *
 * Citations: "P:n" = PAPER.md line n (section / algorithm in brackets).  Readings where the paper is
 * silent are numbered R1..R28 and listed in DESIGN.md §3 ("Readings").
 *
 * Contents (bulk loops only; the small per-codebook steps E3-E5 are pure Python in huffman.py):
 *   E1 split                 P:50-52 [§2.1, Eq. 1]; inverse of Alg. 1 compose P:429-434
 *   E2 histogram             P:97 [§2.3] "distribution of exponents"
 *   E6 bit packing           P:97 "tightly bit-packed into a byte array, EncodedExponent"; MSB-first (R1)
 *   E7 gaps                  P:146 [§2.3.2] "offset of the first valid Huffman code relative to the
 *                            thread's assigned starting byte ... stored using only 5 bits" (R12, R13)
 *   E8 BlockOutputPos        P:148 [§2.3.2] "output position only for the first element of each
 *                            thread block"; B+1 entries (R14)
 *   D1 sequential decoder    P:108 [§2.3] / P:533-546 [App. I.1]: canonical bit-by-bit decode that uses
 *                            only CodeLengths, the stream and PackedSignMantissa
 *   D2 Alg. 1 emulator       P:376-446 [App. Alg. 1 DF11ToBF16], block by block, thread by thread
 *   format variants (NEXT-4) value formats FP16 / FP8 beside BF16 (P:609 names them as the limitation;
 *                            readings R25-R27) and b-bit LUTs (App. I.2, generic b; b = L is
 *                            the monolithic table of App. I.1; R28)
 *
 * Every function is single-threaded scalar C with no blocking, fusion or reordering beyond the
 * definition it follows.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

/* ---------------------------------------------------------------- E1: split / compose
 * P:50-52 [§2.1]: a BF16 word is 1 sign bit (15), 8 exponent bits (14..7), 7 mantissa bits (6..0).
 * P:430-431 [Alg. 1]: PackedSignMantissa holds the sign in bit 7 (mask 0b10000000) and the mantissa
 * in bits 6..0 (mask 0b01111111). */
void df11o_split(const uint16_t *w, uint64_t n, uint8_t *exponent, uint8_t *packed_sign_mantissa)
{
    for (uint64_t i = 0; i < n; i++) {
        uint16_t word = w[i];
        uint8_t sign = (uint8_t)((word >> 15) & 1u);
        uint8_t expo = (uint8_t)((word >> 7) & 0xFFu);
        uint8_t mant = (uint8_t)(word & 0x7Fu);
        exponent[i] = expo;
        packed_sign_mantissa[i] = (uint8_t)((sign << 7) | mant);
    }
}

/* P:429-434 [Alg. 1]: (Sign << 8) | (Exponent << 7) | Mantissa, with Sign = Byte & 0x80 and
 * Mantissa = Byte & 0x7F.  (Sign is already the masked high bit, so Sign << 8 == 0x8000.) */
uint16_t df11o_compose(uint8_t exponent, uint8_t packed_sign_mantissa)
{
    uint16_t sign = (uint16_t)(packed_sign_mantissa & 0x80u);
    uint16_t mant = (uint16_t)(packed_sign_mantissa & 0x7Fu);
    return (uint16_t)((sign << 8) | ((uint16_t)exponent << 7) | mant);
}

/* ---------------------------------------------------------------- value formats (NEXT-4, R25-R27)
 * A value of format vf is split exactly like BF16: its exponent field becomes the Huffman symbol and
 * the remaining bits (sign, then mantissa) are kept raw.
 *   vf 0 BF16        16 bits: sign 15, exponent 14..7  (8 bits), mantissa 6..0 (7 bits)
 *   vf 1 FP16 (IEEE binary16)  16 bits: sign 15, exponent 14..10 (5 bits), mantissa 9..0 (10 bits)
 *   vf 2 FP8 E4M3              8 bits:  sign 7,  exponent 6..3   (4 bits), mantissa 2..0 (3 bits)
 *   vf 3 FP8 E5M2              8 bits:  sign 7,  exponent 6..2   (5 bits), mantissa 1..0 (2 bits)
 * Residual of element i: r = sign << M | mantissa (R = 1 + M bits) in PackedSignMantissa (R25):
 *   R >= 8 (BF16, FP16): the low 8 bits of r are byte i of a byte plane of roundup(n, 16) bytes; the
 *            R - 8 high bits follow in a bit plane, MSB-first at bits [(R-8) i, (R-8) i + R - 8).
 *            For BF16 (R = 8) the bit plane is empty and byte i is sign << 7 | mantissa: the paper's
 *            layout.
 *   R < 8  (FP8): r MSB-first at bits [R i, R i + R). */
static const int VF_WORD_BITS[4] = {16, 16, 8, 8};
static const int VF_EXP_BITS[4] = {8, 5, 4, 5};
static const int VF_MAN_BITS[4] = {7, 10, 3, 2};

int df11o_vf_residual_bits(int vf) { return 1 + VF_MAN_BITS[vf]; }

static uint32_t word_at(const void *w, int vf, uint64_t i)
{
    if (VF_WORD_BITS[vf] == 16) return ((const uint16_t *)w)[i];
    return ((const uint8_t *)w)[i];
}

/* residual stream (MSB-first, R1 order) */
static void put_bits(uint8_t *buf, uint64_t bit, uint32_t v, int nbits);
static uint32_t get_bits(const uint8_t *buf, uint64_t nbytes, uint64_t bit, int nbits);

/* bytes of the byte plane of n residuals (R >= 8), 0 otherwise */
static uint64_t byte_plane_bytes(int R, uint64_t n) { return R >= 8 ? (n + 15) / 16 * 16 : 0; }

static void put_residual(uint8_t *buf, int R, uint64_t n, uint64_t i, uint32_t r)
{
    if (R >= 8) {
        buf[i] = (uint8_t)(r & 0xFFu);
        if (R > 8) put_bits(buf + byte_plane_bytes(R, n), (uint64_t)(R - 8) * i, r >> 8, R - 8);
    } else {
        put_bits(buf, (uint64_t)R * i, r, R);
    }
}

static uint32_t get_residual(const uint8_t *buf, uint64_t nbytes, int R, uint64_t n, uint64_t i)
{
    if (R >= 8) {
        uint32_t lo = i < nbytes ? buf[i] : 0u;
        if (R == 8) return lo;
        uint64_t hb = byte_plane_bytes(R, n);
        uint32_t hi = hb < nbytes ? get_bits(buf + hb, nbytes - hb, (uint64_t)(R - 8) * i, R - 8) : 0u;
        return (hi << 8) | lo;
    }
    return get_bits(buf, nbytes, (uint64_t)R * i, R);
}

/* `residual` must be zeroed and hold the array described above. */
void df11o_split_v(const void *w, uint64_t n, int vf, uint8_t *exponent, uint8_t *residual)
{
    int M = VF_MAN_BITS[vf], E = VF_EXP_BITS[vf], R = 1 + M;
    for (uint64_t i = 0; i < n; i++) {
        uint32_t word = word_at(w, vf, i);
        uint32_t sign = (word >> (E + M)) & 1u;
        uint32_t expo = (word >> M) & ((1u << E) - 1u);
        uint32_t mant = word & ((1u << M) - 1u);
        exponent[i] = (uint8_t)expo;
        put_residual(residual, R, n, i, (sign << M) | mant);
    }
}

/* Inverse: sign << (E + M) | exponent << M | mantissa (for BF16 this is Alg. 1's compose). */
uint32_t df11o_compose_v(int vf, uint32_t exponent, uint32_t residual)
{
    int M = VF_MAN_BITS[vf], E = VF_EXP_BITS[vf];
    uint32_t sign = (residual >> M) & 1u;
    uint32_t mant = residual & ((1u << M) - 1u);
    return (sign << (E + M)) | (exponent << M) | mant;
}

static void store_word(void *out, int vf, uint64_t i, uint32_t v)
{
    if (VF_WORD_BITS[vf] == 16) ((uint16_t *)out)[i] = (uint16_t)v;
    else ((uint8_t *)out)[i] = (uint8_t)v;
}

/* ---------------------------------------------------------------- E2: histogram */
void df11o_histogram(const uint8_t *exponent, uint64_t n, uint64_t *hist /*256*/)
{
    for (int s = 0; s < 256; s++) hist[s] = 0;
    for (uint64_t i = 0; i < n; i++) hist[exponent[i]]++;
}

/* ---------------------------------------------------------------- bit helpers (MSB-first, R1)
 * Stream bit i is bit 7-(i mod 8) of byte floor(i/8). */
static int get_bit(const uint8_t *buf, uint64_t nbytes, uint64_t bit)
{
    uint64_t byte = bit >> 3;
    if (byte >= nbytes) return 0;                 /* zero-extended past the end (R16) */
    return (buf[byte] >> (7 - (bit & 7))) & 1;
}

static void set_bit(uint8_t *buf, uint64_t bit)
{
    buf[bit >> 3] |= (uint8_t)(1u << (7 - (bit & 7)));
}

/* nbits of v, most significant first, at stream bits [bit, bit + nbits) (buffer zeroed) */
static void put_bits(uint8_t *buf, uint64_t bit, uint32_t v, int nbits)
{
    for (int j = nbits - 1; j >= 0; j--) {
        if ((v >> j) & 1u) set_bit(buf, bit);
        bit++;
    }
}

static uint32_t get_bits(const uint8_t *buf, uint64_t nbytes, uint64_t bit, int nbits)
{
    uint32_t v = 0;
    for (int j = 0; j < nbits; j++) v = (v << 1) | (uint32_t)get_bit(buf, nbytes, bit + (uint64_t)j);
    return v;
}

/* ---------------------------------------------------------------- E6: bit packing
 * Concatenate the codeword of every element, MSB of each codeword first (R1).  `out` must be zeroed
 * by the caller and hold at least ceil(sum(len)/8) bytes.  Returns the number of bits written. */
uint64_t df11o_pack_bits(const uint8_t *exponent, uint64_t n, const uint8_t *code_len /*256*/,
                         const uint32_t *code /*256*/, uint8_t *out)
{
    uint64_t bit = 0;
    for (uint64_t i = 0; i < n; i++) {
        uint8_t e = exponent[i];
        int len = code_len[e];
        uint32_t c = code[e];
        for (int j = len - 1; j >= 0; j--) {      /* most significant code bit first */
            if ((c >> j) & 1u) set_bit(out, bit);
            bit++;
        }
    }
    return bit;
}

/* ---------------------------------------------------------------- E7 + E8: gaps and BlockOutputPos
 * Thread g (global index bT+t, R23) owns stream bits [8n*g, 8n*(g+1)).
 *   gap[g] = (first codeword start >= 8n*g) - 8n*g   if that start is < 8n*(g+1), else 0  (R13)
 *   bop[b] = number of codewords that start before bit 8nT*b  (b < B);  bop[B] = N      (R14)
 * Computed directly from the definition by walking the codeword start positions once. */
int df11o_gaps_bop(const uint8_t *exponent, uint64_t n, const uint8_t *code_len /*256*/,
                   uint32_t T, uint32_t n_bytes, uint32_t B,
                   uint8_t *gap_values /*B*T*/, uint32_t *bop /*B+1*/)
{
    uint64_t chunk_bits = 8ull * n_bytes;
    uint64_t block_bits = chunk_bits * T;
    uint64_t threads = (uint64_t)B * T;
    for (uint64_t g = 0; g < threads; g++) gap_values[g] = 0;
    for (uint32_t b = 0; b <= B; b++) bop[b] = 0;

    /* starts[i] = sum of code lengths of elements before i */
    uint64_t start = 0;
    uint64_t next_chunk = 0;    /* smallest chunk index whose gap is not yet assigned */
    uint64_t next_block = 0;    /* smallest block index whose bop is not yet assigned */
    for (uint64_t i = 0; i < n; i++) {
        /* every chunk g with 8n*g <= start and not yet assigned: this is its first start >= 8n*g */
        while (next_chunk < threads && next_chunk * chunk_bits <= start) {
            uint64_t c0 = next_chunk * chunk_bits;
            uint64_t gap = start - c0;
            gap_values[next_chunk] = (gap < chunk_bits) ? (uint8_t)gap : 0;
            if (gap < chunk_bits && gap > 31) return -1;    /* cannot be stored in 5 bits */
            next_chunk++;
        }
        while (next_block < B && next_block * block_bits <= start) {
            bop[next_block] = (uint32_t)i;               /* codes starting before 8nT*b: elements 0..i-1 */
            next_block++;
        }
        start += code_len[exponent[i]];
    }
    /* remaining chunks have no codeword start at or after their beginning: gap 0 (R13) */
    while (next_block < B) { bop[next_block] = (uint32_t)n; next_block++; }
    bop[B] = (uint32_t)n;
    return 0;
}

/* Pack 5-bit gap values MSB-first: field g occupies stream bits [5g, 5g+5) (R12).
 * `out` must be zeroed and hold ceil(5*count/8) bytes. */
void df11o_pack_gaps(const uint8_t *gap_values, uint64_t count, uint8_t *out)
{
    for (uint64_t g = 0; g < count; g++) {
        uint8_t v = gap_values[g];
        for (int j = 4; j >= 0; j--)
            if ((v >> j) & 1u) set_bit(out, 5 * g + (uint64_t)(4 - j));
    }
}

/* Read back one 5-bit field (used by D2). */
static uint32_t read_gap(const uint8_t *gaps, uint64_t gaps_bytes, uint64_t g)
{
    uint32_t v = 0;
    for (int j = 0; j < 5; j++) v = (v << 1) | (uint32_t)get_bit(gaps, gaps_bytes, 5 * g + (uint64_t)j);
    return v;
}

/* ---------------------------------------------------------------- D1: sequential canonical decoder
 * Uses only CodeLengths (canonical reconstruction, R3/E4), the stream, PackedSignMantissa and N;
 * value format vf (R25): element i = compose_v(symbol, residual bits [R*i, R*i + R)), written as a
 * 16-bit (BF16, FP16) or 8-bit (FP8) word.
 * Canonical codes: symbols sorted by (length, symbol); code_0 = 0, code_i = (code_{i-1}+1) << (l_i - l_{i-1}).
 * Bit by bit: append the next stream bit to `code`; after l bits, if code - first_code[l] < count[l]
 * the codeword is complete and names symbol sorted[offset[l] + code - first_code[l]].
 * Returns 0 on success, -1 if the stream runs out (corrupt), -2 on a malformed codebook. */
int df11o_decode_sequential_range(const uint8_t *stream, uint64_t stream_bytes, const uint8_t *code_len /*256*/,
                                  const uint8_t *packed_sign_mantissa, uint64_t psm_bytes, uint64_t total,
                                  uint64_t start_bit, uint64_t first, uint64_t n, int vf, void *out);

int df11o_decode_sequential(const uint8_t *stream, uint64_t stream_bytes, const uint8_t *code_len /*256*/,
                            const uint8_t *packed_sign_mantissa, uint64_t psm_bytes, uint64_t n, int vf,
                            void *out)
{
    return df11o_decode_sequential_range(stream, stream_bytes, code_len, packed_sign_mantissa, psm_bytes, n, 0, 0, n,
                                         vf, out);
}

/* D1 from the middle of the stream: the same decode started at stream bit `start_bit` with output index
 * `first`, for n elements.  A format block b's first code starts at bit 8nT*b + Gaps[bT] and is element
 * BlockOutputPos[b], so the blocks of a tensor can be decoded independently. */
int df11o_decode_sequential_range(const uint8_t *stream, uint64_t stream_bytes, const uint8_t *code_len /*256*/,
                                  const uint8_t *packed_sign_mantissa, uint64_t psm_bytes, uint64_t total,
                                  uint64_t start_bit, uint64_t first, uint64_t n, int vf, void *out)
{
    const int R = 1 + VF_MAN_BITS[vf];
    uint32_t count[33] = {0};
    uint32_t first_code[33] = {0};
    uint32_t offset[33] = {0};
    uint8_t sorted[256];
    int nsym = 0;
    for (int l = 1; l <= 32; l++) {
        offset[l] = (uint32_t)nsym;
        for (int s = 0; s < 256; s++)
            if (code_len[s] == l) { sorted[nsym++] = (uint8_t)s; count[l]++; }
    }
    for (int s = 0; s < 256; s++) if (code_len[s] > 32) return -2;
    for (int s = 1 << VF_EXP_BITS[vf]; s < 256; s++) if (code_len[s]) return -2;   /* not an exponent */
    if (n > 0 && nsym == 0) return -2;
    /* first canonical code of each length */
    uint64_t code = 0;
    int prev_len = 0;
    int have_prev = 0;
    for (int l = 1; l <= 32; l++) {
        if (count[l] == 0) continue;
        if (have_prev) code = (code + 1) << (l - prev_len);
        else code = 0;
        /* code is now the first code of length l; the last one is code + count - 1 */
        first_code[l] = (uint32_t)code;
        code = code + count[l] - 1;
        prev_len = l;
        have_prev = 1;
    }

    uint64_t total_bits = stream_bytes * 8;
    uint64_t bit = start_bit;
    for (uint64_t i = first; i < first + n; i++) {
        uint64_t c = 0;
        int l = 0;
        int found = -1;
        while (found < 0) {
            if (bit >= total_bits) return -1;
            c = (c << 1) | (uint64_t)get_bit(stream, stream_bytes, bit);
            bit++;
            l++;
            if (l > 32) return -1;
            if (count[l] && c >= first_code[l] && c - first_code[l] < count[l])
                found = sorted[offset[l] + (uint32_t)(c - first_code[l])];
        }
        store_word(out, vf, i, df11o_compose_v(vf, (uint32_t)found,
                                               get_residual(packed_sign_mantissa, psm_bytes, R, total, i)));
    }
    return 0;
}

/* ---------------------------------------------------------------- D2: Alg. 1 emulator
 * P:382-443.  "Read the next 4 bytes ... starting from the BitOffset-th bit, into Byte_{1..4}":
 * a big-endian 32-bit window at the absolute stream bit chunk_start + BitOffset (R2), zero-extended
 * past the buffer end (R16).  Exponent >= 240 is a pointer to LUT_{257-Exponent} (1-based), i.e. the
 * 0-based table 256-Exponent (narrow, entry_bytes = 1); wide tables (entry_bytes = 2, R8) use
 * entries >= 256 as pointers to table (entry-256).  Tables have 2^b entries (App. I.2, generic b; the
 * paper's b = 8 reads Byte_1..Byte_4): level i (1-based) is indexed by window bits [b(i-1), bi),
 * zero-extended past bit 32 (R28).  Outputs are clipped to [BOP[b], BOP[b+1]) (R15).
 * check_counts = 1 additionally asserts that every non-final block decodes exactly
 * BOP[b+1]-BOP[b] elements (returns -3 if not).  Returns 0 on success, -4 on a malformed LUT walk. */
static uint32_t window32(const uint8_t *stream, uint64_t stream_bytes, uint64_t bit)
{
    uint32_t w = 0;
    for (int j = 0; j < 32; j++) w = (w << 1) | (uint32_t)get_bit(stream, stream_bytes, bit + (uint64_t)j);
    return w;
}

static int lut_entry(const uint8_t *luts, uint32_t entry_bytes, uint32_t b, uint32_t table, uint32_t idx)
{
    uint64_t off = ((uint64_t)table << b) + idx;
    if (entry_bytes == 1) return luts[off];
    const uint8_t *p = luts + off * 2;
    return (int)p[0] | ((int)p[1] << 8);           /* little-endian uint16 entries */
}

static int is_pointer(int e, uint32_t entry_bytes) { return entry_bytes == 1 ? e >= 240 : e >= 256; }
static uint32_t pointer_target(int e, uint32_t entry_bytes)
{
    return entry_bytes == 1 ? (uint32_t)(256 - e) : (uint32_t)(e - 256);
}

/* Window bits [b(i-1), bi) as an index (bits past 32 read as zero). */
static uint32_t level_index(uint32_t window, uint32_t b, int i)
{
    uint32_t idx = 0;
    for (uint32_t j = 0; j < b; j++) {
        uint32_t bit = b * (uint32_t)(i - 1) + j;
        idx = (idx << 1) | (bit < 32 ? (window >> (31 - bit)) & 1u : 0u);
    }
    return idx;
}

/* One LUT walk: returns the decoded exponent or -1 on a malformed walk. */
static int alg1_decode_one(uint32_t window, const uint8_t *luts, uint32_t entry_bytes, uint32_t k, uint32_t b)
{
    int i = 1;
    const int levels = (int)((32 + b - 1) / b);              /* a code of <= 32 bits */
    int e = lut_entry(luts, entry_bytes, b, 0, level_index(window, b, 1));   /* LUT_1 = root */
    while (is_pointer(e, entry_bytes)) {
        i = i + 1;
        if (i > levels) return -1;
        uint32_t table = pointer_target(e, entry_bytes);
        if (table >= k) return -1;
        e = lut_entry(luts, entry_bytes, b, table, level_index(window, b, i));
    }
    return e;
}

int df11o_decode_alg1(const uint8_t *luts, uint32_t entry_bytes, uint32_t k, uint32_t lut_bits,
                      const uint8_t *code_len, const uint8_t *stream, uint64_t stream_bytes,
                      const uint8_t *gaps, uint64_t gaps_bytes, const uint32_t *bop,
                      const uint8_t *packed_sign_mantissa, uint64_t psm_bytes, uint32_t B, uint32_t T,
                      uint32_t n_bytes, uint64_t N, int vf, int check_counts, void *out)
{
    const int R = 1 + VF_MAN_BITS[vf];
    if (lut_bits < 1 || lut_bits > 16) return -4;
    uint64_t chunk_bits = 8ull * n_bytes;
    uint32_t *num_elements = (uint32_t *)calloc(T ? T : 1, sizeof(uint32_t));
    uint64_t *thread_output_pos = (uint64_t *)calloc(T ? T : 1, sizeof(uint64_t));
    if (!num_elements || !thread_output_pos) { free(num_elements); free(thread_output_pos); return -5; }
    int rc = 0;
    for (uint32_t b = 0; b < B && rc == 0; b++) {
        /* Phase 1: each thread counts the codewords that start in its chunk. */
        for (uint32_t t = 0; t < T; t++) {
            uint64_t g = (uint64_t)b * T + t;
            uint64_t chunk_start = g * chunk_bits;
            uint64_t bit_offset = read_gap(gaps, gaps_bytes, g);
            num_elements[t] = 0;
            while (bit_offset < chunk_bits) {
                uint32_t w = window32(stream, stream_bytes, chunk_start + bit_offset);
                int e = alg1_decode_one(w, luts, entry_bytes, k, lut_bits);
                if (e < 0 || code_len[e] == 0) { rc = -4; break; }
                bit_offset += code_len[e];
                num_elements[t]++;
            }
            if (rc) break;
        }
        if (rc) break;
        /* Prefix sum: ThreadOutputPos[t] = BlockOutputPos[b] + sum_{i<t} NumElements[i]. */
        uint64_t running = 0;
        for (uint32_t t = 0; t < T; t++) { thread_output_pos[t] = bop[b] + running; running += num_elements[t]; }
        if (check_counts && b + 1 < B && running != (uint64_t)bop[b + 1] - bop[b]) { rc = -3; break; }
        /* Phase 2: re-decode and write, clipped to [BOP[b], BOP[b+1]) and N (R15). */
        for (uint32_t t = 0; t < T; t++) {
            uint64_t g = (uint64_t)b * T + t;
            uint64_t chunk_start = g * chunk_bits;
            uint64_t bit_offset = read_gap(gaps, gaps_bytes, g);
            uint64_t pos = thread_output_pos[t];
            while (bit_offset < chunk_bits) {
                uint32_t w = window32(stream, stream_bytes, chunk_start + bit_offset);
                int e = alg1_decode_one(w, luts, entry_bytes, k, lut_bits);
                if (e < 0 || code_len[e] == 0 || e >= (1 << VF_EXP_BITS[vf])) { rc = -4; break; }
                if (pos < bop[b + 1] && pos < N)
                    store_word(out, vf, pos, df11o_compose_v(vf, (uint32_t)e,
                                                             get_residual(packed_sign_mantissa, psm_bytes, R, N,
                                                                          pos)));
                bit_offset += code_len[e];
                pos++;
            }
            if (rc) break;
        }
    }
    free(num_elements);
    free(thread_output_pos);
    return rc;
}
