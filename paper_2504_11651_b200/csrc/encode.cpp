// encode.cpp — host DF11 encoder: df11_encode / df11_encode_group.
//
// Produces the bit-exact format of DESIGN.md §2 from the paper's description:
//   split -> exponent histogram -> Huffman code lengths with the 32-bit
//   cap (R3 tie rule, R4 package-merge) -> canonical codes -> hierarchical 2^b-entry LUTs
//   (App. I.2; b = 8 by default, b = L for the monolithic table of App. I.1; R6
//   breadth-first children, R8 wide fallback, R28) -> MSB-first bit packing of EncodedExponent (P:97,
//   R1) -> Gaps (R12/R13) and BlockOutputPos (R14).  Value formats FP16 / FP8 (NEXT-4,
//   R25-R27) split the same way: exponent field -> symbol, sign + mantissa -> residual planes.
//
// Built for speed, not for reading against the paper (that is oracle/'s job): every O(N) pass is
// split over host threads; the bit packer gives every thread a bit range computed by a prefix sum of
// per-segment code-length totals and ORs the two bytes it shares with its neighbours atomically.
// This file shares no code with oracle/; byte-for-byte agreement is checked by tests/test_encoder_parity.py.
#include "df11.h"
#include "df11_internal.h"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <thread>
#include <vector>

namespace {

constexpr int kMaxCodeLen = 32;

// ------------------------------------------------------------------------------------ threading
struct Pool {
    unsigned nthreads;
    explicit Pool(unsigned requested, uint64_t work) {
        unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        nthreads = requested ? requested : hw;
        // below ~256K elements per thread the spawn cost dominates
        uint64_t cap = std::max<uint64_t>(1, work / (1u << 18));
        if (nthreads > cap) nthreads = (unsigned)cap;
        if (nthreads < 1) nthreads = 1;
    }
    // run f(tid, begin, end) over [0, n) split into nthreads contiguous ranges
    void run(uint64_t n, const std::function<void(unsigned, uint64_t, uint64_t)> &f) const {
        if (nthreads == 1) { f(0, 0, n); return; }
        std::vector<std::thread> ts;
        ts.reserve(nthreads);
        for (unsigned t = 0; t < nthreads; t++) {
            uint64_t b = n * t / nthreads, e = n * (t + 1) / nthreads;
            ts.emplace_back([&f, t, b, e] { f(t, b, e); });
        }
        for (auto &th : ts) th.join();
    }
};

inline uint64_t roundup(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

// ------------------------------------------------------------------------------------ value formats
// Word of `word_bytes` bytes: sign | exponent (exp_bits) | mantissa (man_bits); residual R = 1 + M.
struct VFmt {
    uint32_t word_bytes, exp_bits, man_bits;
    uint32_t R() const { return 1 + man_bits; }
    uint32_t emask() const { return (1u << exp_bits) - 1u; }
};
constexpr VFmt kVF[4] = {{2, 8, 7}, {2, 5, 10}, {1, 4, 3}, {1, 5, 2}};   // BF16, FP16, FP8 E4M3, E5M2

inline uint32_t word_at(const void *w, const VFmt &f, uint64_t i) {
    return f.word_bytes == 2 ? (uint32_t)static_cast<const uint16_t *>(w)[i] : (uint32_t)static_cast<const uint8_t *>(w)[i];
}
inline uint32_t symbol_of(uint32_t word, const VFmt &f) { return (word >> f.man_bits) & f.emask(); }
inline uint32_t residual_of(uint32_t word, const VFmt &f) {
    return ((word >> (f.exp_bits + f.man_bits)) << f.man_bits) | (word & ((1u << f.man_bits) - 1u));
}
// PackedSignMantissa (R25): R >= 8 -> a byte plane of the low 8 bits (roundup(n, 16) bytes) followed by
// the (R - 8)-bit plane of the high bits (FP16: sign, m9, m8), MSB-first; R < 8 -> one R-bit plane.
inline uint64_t residual_bytes(uint64_t n, const VFmt &f) {
    const uint64_t L = roundup(n, 16), R = f.R();
    return R >= 8 ? L + roundup((R - 8) * L / 8, 16) + 16 : roundup(R * L / 8, 16) + 16;
}

// ------------------------------------------------------------------------------------ histogram
template <typename W>
void histogram_t(const W *w, uint64_t n, const VFmt &f, const Pool &pool, uint64_t hist[256]) {
    std::vector<uint64_t> part((size_t)pool.nthreads * 256, 0);
    const uint32_t sh = f.man_bits, m = f.emask();
    pool.run(n, [&](unsigned t, uint64_t b, uint64_t e) {
        uint64_t local[4][256] = {};
        uint64_t i = b;
        for (; i + 4 <= e; i += 4) {                      // 4 sub-histograms hide store-to-load stalls
            local[0][(w[i] >> sh) & m]++;
            local[1][(w[i + 1] >> sh) & m]++;
            local[2][(w[i + 2] >> sh) & m]++;
            local[3][(w[i + 3] >> sh) & m]++;
        }
        for (; i < e; i++) local[0][(w[i] >> sh) & m]++;
        for (int s = 0; s < 256; s++) part[(size_t)t * 256 + s] = local[0][s] + local[1][s] + local[2][s] + local[3][s];
    });
    for (int s = 0; s < 256; s++) {
        uint64_t acc = 0;
        for (unsigned t = 0; t < pool.nthreads; t++) acc += part[(size_t)t * 256 + s];
        hist[s] = acc;
    }
}
void histogram(const void *w, uint64_t n, const VFmt &f, const Pool &pool, uint64_t hist[256]) {
    if (f.word_bytes == 2) histogram_t(static_cast<const uint16_t *>(w), n, f, pool, hist);
    else histogram_t(static_cast<const uint8_t *>(w), n, f, pool, hist);
}

// ------------------------------------------------------------------------------------ code lengths
// Leaves in (count asc, symbol asc) order.
std::vector<int> ranked_symbols(const uint64_t hist[256]) {
    std::vector<int> syms;
    for (int s = 0; s < 256; s++) if (hist[s]) syms.push_back(s);
    std::stable_sort(syms.begin(), syms.end(), [&](int a, int b) { return hist[a] < hist[b]; });
    return syms;   // stable sort over ascending symbols => ties broken by symbol
}

// Two-queue Huffman (R3).  With leaves sorted by (count, symbol) the queue of internal nodes is sorted
// by creation, so comparing the two queue fronts on (weight, key) reproduces a min-heap keyed by
// (weight, key) where leaves have keys 0..|S|-1 and internal nodes |S|+creation index: on equal
// weight the leaf wins.
void huffman_lengths(const uint64_t hist[256], const std::vector<int> &ranked, uint8_t len[256]) {
    const int m = (int)ranked.size();
    std::memset(len, 0, 256);
    if (m == 0) return;
    if (m == 1) { len[ranked[0]] = 1; return; }
    // nodes 0..m-1 = leaves (rank order), m.. = internal nodes in creation order
    std::vector<uint64_t> weight(2 * m - 1);
    std::vector<int> parent(2 * m - 1, -1);
    for (int i = 0; i < m; i++) weight[i] = hist[ranked[i]];
    int leaf = 0, inner = m, next = m;
    auto pop = [&]() {
        bool take_leaf = leaf < m && (inner >= next || weight[leaf] <= weight[inner]);
        return take_leaf ? leaf++ : inner++;
    };
    while (next < 2 * m - 1) {
        int a = pop();
        int b = pop();
        weight[next] = weight[a] + weight[b];
        parent[a] = parent[b] = next;
        next++;
    }
    std::vector<uint8_t> depth(2 * m - 1, 0);
    for (int v = 2 * m - 3; v >= 0; v--) depth[v] = (uint8_t)std::min(255, depth[parent[v]] + 1);
    for (int i = 0; i < m; i++) len[ranked[i]] = depth[i];
}

// Package-merge with cap L (R4): level lists built bottom-up; an item is a leaf (rank r) or a package
// of two consecutive items of the list below.  Selection of the first 2(|S|-1) items of the top list
// is pushed down level by level.
void package_merge_lengths(const uint64_t hist[256], const std::vector<int> &ranked, int cap, uint8_t len[256]) {
    const int m = (int)ranked.size();
    std::memset(len, 0, 256);
    if (m == 0) return;
    if (m == 1) { len[ranked[0]] = 1; return; }
    struct Item { uint64_t w; int leaf; int child; };   // leaf >= 0: leaf rank; else package of list[child], list[child+1]
    std::vector<std::vector<Item>> lists(cap);
    lists[0].reserve(m);
    for (int r = 0; r < m; r++) lists[0].push_back({hist[ranked[r]], r, -1});
    for (int lvl = 1; lvl < cap; lvl++) {
        const std::vector<Item> &below = lists[lvl - 1];
        std::vector<Item> &cur = lists[lvl];
        cur.reserve(m + below.size() / 2);
        size_t npk = below.size() / 2;
        size_t li = 0, pi = 0;
        while (li < (size_t)m || pi < npk) {
            uint64_t pw = pi < npk ? below[2 * pi].w + below[2 * pi + 1].w : 0;
            if (pi >= npk || (li < (size_t)m && hist[ranked[li]] <= pw)) {
                cur.push_back({hist[ranked[li]], (int)li, -1});
                li++;
            } else {
                cur.push_back({pw, -1, (int)(2 * pi)});
                pi++;
            }
        }
    }
    // selection mask, top level first
    std::vector<char> sel(lists[cap - 1].size(), 0);
    size_t take = std::min<size_t>(2 * (size_t)(m - 1), sel.size());
    std::fill(sel.begin(), sel.begin() + take, 1);
    std::vector<int> count(m, 0);
    for (int lvl = cap - 1; lvl >= 0; lvl--) {
        const std::vector<Item> &cur = lists[lvl];
        std::vector<char> below_sel(lvl > 0 ? lists[lvl - 1].size() : 0, 0);
        for (size_t i = 0; i < cur.size(); i++) {
            if (!sel[i]) continue;
            if (cur[i].leaf >= 0) count[cur[i].leaf]++;
            else { below_sel[cur[i].child] = 1; below_sel[cur[i].child + 1] = 1; }
        }
        sel.swap(below_sel);
    }
    for (int r = 0; r < m; r++) len[ranked[r]] = (uint8_t)count[r];
}

// ------------------------------------------------------------------------------------ canonical codes
void canonical_codes(const uint8_t len[256], uint32_t code[256]) {
    std::memset(code, 0, 256 * sizeof(uint32_t));
    uint32_t bl_count[kMaxCodeLen + 1] = {};
    for (int s = 0; s < 256; s++) if (len[s]) bl_count[len[s]]++;
    // first code of each length (DEFLATE-style recurrence; equals the (length, symbol) sort rule)
    uint32_t next_code[kMaxCodeLen + 2] = {};
    uint64_t c = 0;
    for (int l = 1; l <= kMaxCodeLen; l++) {
        c = (c + bl_count[l - 1]) << 1;
        next_code[l] = (uint32_t)c;
    }
    for (int s = 0; s < 256; s++) if (len[s]) code[s] = next_code[len[s]]++;
}

// ------------------------------------------------------------------------------------ LUTs
// Explicit code tree, then every table enumerates the 2^b b-bit paths from its subtree root.
struct Tree {
    std::vector<int> child0, child1, symbol;   // symbol >= 0 at leaves
    int add() { child0.push_back(-1); child1.push_back(-1); symbol.push_back(-1); return (int)symbol.size() - 1; }
};

df11_status build_luts(const uint8_t len[256], const uint32_t code[256], int lut_mode, uint32_t b,
                       std::vector<uint8_t> &out, uint32_t &k, uint32_t &entry_bytes) {
    const uint32_t size = 1u << b;
    out.clear();
    k = 0;
    entry_bytes = 1;
    int nsym = 0, only = -1;
    bool reserved = false;
    for (int s = 0; s < 256; s++) if (len[s]) { nsym++; only = s; if (s >= 240) reserved = true; }
    if (nsym == 0) return DF11_OK;
    Tree tree;
    int root = tree.add();
    for (int s = 0; s < 256; s++) {
        if (!len[s]) continue;
        int v = root;
        for (int i = len[s] - 1; i >= 0; i--) {
            int bit = (code[s] >> i) & 1;
            int nxt = bit ? tree.child1[v] : tree.child0[v];
            if (nxt < 0) {
                nxt = tree.add();                                  // may reallocate: index afresh
                (bit ? tree.child1 : tree.child0)[v] = nxt;
            }
            v = nxt;
        }
        tree.symbol[v] = s;
    }
    // tables: BFS queue of subtree roots; entry value: >= 0 symbol, < 0 => -(child table index)
    std::vector<int> table_root{root};
    std::vector<int> entries;
    for (size_t t = 0; t < table_root.size(); t++) {
        for (uint32_t idx = 0; idx < size; idx++) {
            int v = table_root[t];
            int val = INT32_MIN;
            for (int bit = (int)b - 1; bit >= 0 && val == INT32_MIN; bit--) {
                int bb = (idx >> bit) & 1;
                int nv = bb ? tree.child1[v] : tree.child0[v];
                if (nv < 0) { val = only; break; }           // unreachable: only when |S| = 1 (R7)
                v = nv;
                if (tree.symbol[v] >= 0) val = tree.symbol[v];
            }
            if (val == INT32_MIN) {                          // still inside the tree after b bits
                int j = -1;
                for (size_t q = t + 1; q < table_root.size(); q++) if (table_root[q] == v) { j = (int)q; break; }
                if (j < 0) { table_root.push_back(v); j = (int)table_root.size() - 1; }
                val = -j;
            }
            entries.push_back(val);
        }
    }
    k = (uint32_t)table_root.size();
    bool narrow_ok = !reserved && k - 1 <= 16;
    bool wide;
    if (lut_mode == DF11_LUT_NARROW) {
        if (reserved) return DF11_E_RESERVED_EXPONENT;
        if (k - 1 > 16) return DF11_E_LUT_OVERFLOW;
        wide = false;
    } else if (lut_mode == DF11_LUT_WIDE) {
        wide = true;
    } else {
        wide = !narrow_ok;
    }
    entry_bytes = wide ? 2 : 1;
    out.resize((size_t)k * size * entry_bytes);
    for (size_t i = 0; i < entries.size(); i++) {
        int e = entries[i];
        uint32_t v = e >= 0 ? (uint32_t)e : (wide ? 256u + (uint32_t)(-e) : 256u - (uint32_t)(-e));
        if (wide) { out[2 * i] = (uint8_t)(v & 0xFF); out[2 * i + 1] = (uint8_t)(v >> 8); }
        else out[i] = (uint8_t)v;
    }
    return DF11_OK;
}

// ------------------------------------------------------------------------------------ codebook
struct Codebook {
    uint8_t len[256];
    uint32_t code[256];
    uint32_t max_len;
    std::vector<uint8_t> luts;
    uint32_t k, entry_bytes, lut_bits;
};

// lut_bits: 1..16, or DF11_LUT_BITS_MONOLITHIC (b = L, one table; L <= 16)
df11_status make_codebook(const uint64_t hist[256], int lut_mode, uint32_t lut_bits, Codebook &cb) {
    std::vector<int> ranked = ranked_symbols(hist);
    huffman_lengths(hist, ranked, cb.len);
    cb.max_len = 0;
    for (int s = 0; s < 256; s++) cb.max_len = std::max<uint32_t>(cb.max_len, cb.len[s]);
    if (cb.max_len > kMaxCodeLen) {
        package_merge_lengths(hist, ranked, kMaxCodeLen, cb.len);
        cb.max_len = 0;
        for (int s = 0; s < 256; s++) cb.max_len = std::max<uint32_t>(cb.max_len, cb.len[s]);
    }
    canonical_codes(cb.len, cb.code);
    if (lut_bits == DF11_LUT_BITS_MONOLITHIC) {
        if (cb.max_len > 16) return df11_fail(DF11_E_INVALID_ARGUMENT, "monolithic LUT needs max code length <= 16");
        lut_bits = std::max<uint32_t>(cb.max_len, 1);
    }
    cb.lut_bits = lut_bits;
    df11_status st = build_luts(cb.len, cb.code, lut_mode, lut_bits, cb.luts, cb.k, cb.entry_bytes);
    if (st == DF11_E_RESERVED_EXPONENT) return df11_fail(st, "exponent >= 240 with NARROW LUTs");
    if (st == DF11_E_LUT_OVERFLOW) return df11_fail(st, "more than 16 child LUTs with NARROW LUTs");
    return st;
}

// ------------------------------------------------------------------------------------ packing
inline void or_byte(uint8_t *p, uint8_t v) { __atomic_fetch_or(p, v, __ATOMIC_RELAXED); }

template <typename W>
df11_status encode_with_codebook(const W *w, uint64_t n, const VFmt &f, uint32_t vf, uint32_t T, uint32_t nb,
                                 const Codebook &cb, const Pool &pool, df11_host_tensor *out) {
    const uint32_t sh = f.man_bits, em = f.emask();
    df11_host_tensor r;
    std::memset(&r, 0, sizeof(r));
    r.num_elements = n;
    r.T = T;
    r.n = nb;
    std::memcpy(r.code_lengths, cb.len, 256);
    r.k = cb.k;
    r.lut_entry_bytes = cb.entry_bytes;
    r.max_code_len = cb.max_len;
    r.value_format = vf;
    r.lut_bits = cb.lut_bits;

    // per-thread bit totals -> exclusive prefix (bit offset of each segment)
    const unsigned P = pool.nthreads;
    std::vector<uint64_t> seg_bits(P + 1, 0);
    pool.run(n, [&](unsigned t, uint64_t b, uint64_t e) {
        uint64_t acc = 0;
        for (uint64_t i = b; i < e; i++) acc += cb.len[(w[i] >> sh) & em];
        seg_bits[t + 1] = acc;
    });
    for (unsigned t = 0; t < P; t++) seg_bits[t + 1] += seg_bits[t];
    const uint64_t total_bits = seg_bits[P];
    const uint64_t chunk_bits = 8ull * nb, block_bits = chunk_bits * T;
    const uint64_t B64 = (total_bits + block_bits - 1) / block_bits;
    if (B64 > 0xFFFFFFFFull) return DF11_E_TOO_LARGE;
    const uint32_t B = (uint32_t)B64;
    r.B = B;
    r.encoded_bits = total_bits;

    r.luts_bytes = cb.luts.size();
    r.encoded_exponent_bytes = (uint64_t)B * T * nb + 16;
    r.packed_sign_mantissa_bytes = residual_bytes(n, f);
    r.gaps_bytes = roundup((5ull * B * T + 7) / 8, 16) + 16;
    r.luts = (uint8_t *)std::calloc(std::max<uint64_t>(r.luts_bytes, 1), 1);
    r.encoded_exponent = (uint8_t *)std::calloc(r.encoded_exponent_bytes, 1);
    r.packed_sign_mantissa = (uint8_t *)std::calloc(r.packed_sign_mantissa_bytes, 1);
    r.gaps = (uint8_t *)std::calloc(r.gaps_bytes, 1);
    r.block_output_pos = (uint32_t *)std::calloc((size_t)B + 1, sizeof(uint32_t));
    std::vector<uint8_t> gap_vals((size_t)B * T, 0);
    if (!r.luts || !r.encoded_exponent || !r.packed_sign_mantissa || !r.gaps || !r.block_output_pos) {
        df11_host_tensor_free(&r);
        return DF11_E_ALLOC;
    }
    if (r.luts_bytes) std::memcpy(r.luts, cb.luts.data(), r.luts_bytes);

    uint8_t *stream = r.encoded_exponent;
    uint8_t *psm = r.packed_sign_mantissa;
    uint32_t *bop = r.block_output_pos;
    const uint64_t nthreads_fmt = (uint64_t)B * T;
    pool.run(n, [&](unsigned t, uint64_t b, uint64_t e) {
        if (b >= e) return;
        uint64_t bit = seg_bits[t];
        // bit packer: acc holds `nacc` pending bits left-aligned in the low 64; emit whole bytes
        uint64_t byte_pos = bit >> 3;
        uint64_t acc = 0;
        int nacc = (int)(bit & 7);             // leading bits belong to the previous segment (zeros here)
        bool first_byte = true;
        // gaps/BOP: chunks whose first codeword start lies in this segment
        uint64_t prev_start = (b == 0) ? 0 : bit - cb.len[(w[b - 1] >> sh) & em];
        uint64_t next_chunk = (b == 0) ? 0 : prev_start / chunk_bits + 1;
        uint64_t next_block = (b == 0) ? 0 : prev_start / block_bits + 1;
        for (uint64_t i = b; i < e; i++) {
            const uint32_t word = w[i];
            const uint32_t ex = (word >> sh) & em;
            if (f.R() >= 8) psm[i] = (uint8_t)residual_of(word, f);   // byte plane; BF16: P:430-431
            // first codeword start at or after chunk / block boundaries
            while (next_chunk < nthreads_fmt && next_chunk * chunk_bits <= bit) {
                uint64_t gap = bit - next_chunk * chunk_bits;
                gap_vals[next_chunk] = gap < chunk_bits ? (uint8_t)gap : 0;
                next_chunk++;
            }
            while (next_block < B && next_block * block_bits <= bit) bop[next_block++] = (uint32_t)i;
            const int l = cb.len[ex];
            acc = (acc << l) | cb.code[ex];
            nacc += l;
            bit += l;
            while (nacc >= 8) {
                uint8_t v = (uint8_t)(acc >> (nacc - 8));
                if (first_byte) { or_byte(stream + byte_pos, v); first_byte = false; }
                else stream[byte_pos] = v;
                byte_pos++;
                nacc -= 8;
            }
            acc &= (nacc ? ((1ull << nacc) - 1) : 0);
        }
        if (nacc > 0) or_byte(stream + byte_pos, (uint8_t)(acc << (8 - nacc)));
    });
    // chunks / blocks past the last codeword start
    {
        // last start = total_bits - len(last)
        uint64_t last_start = n ? total_bits - cb.len[(w[n - 1] >> sh) & em] : 0;
        (void)last_start;
        for (uint32_t b = 0; b < B; b++) if (b > 0 && bop[b] == 0 && (uint64_t)b * block_bits > last_start) bop[b] = (uint32_t)n;
        bop[B] = (uint32_t)n;
    }
    // residual bit plane of the other value formats (R25): 8 elements = P bytes, MSB-first; P = R - 8 high
    // bits after the byte plane (FP16), P = R bits (FP8)
    if (f.R() != 8) {
        const uint32_t R = f.R(), P = R > 8 ? R - 8 : R, shift = R > 8 ? 8 : 0;
        uint8_t *plane = psm + (R > 8 ? roundup(n, 16) : 0);
        pool.run((n + 7) / 8, [&](unsigned, uint64_t qb, uint64_t qe) {
            for (uint64_t q = qb; q < qe; q++) {
                uint64_t acc = 0;                          // 8 * P <= 32 bits
                for (uint64_t j = 0; j < 8; j++) {
                    const uint64_t i = q * 8 + j;
                    acc = (acc << P) | (i < n ? residual_of(w[i], f) >> shift : 0u);
                }
                for (uint32_t j = 0; j < P; j++) plane[q * P + j] = (uint8_t)(acc >> (8 * (P - 1 - j)));
            }
        });
    }
    // pack gaps: 8 fields = 40 bits = 5 bytes, MSB-first
    Pool gpool(pool.nthreads, nthreads_fmt);
    uint64_t groups = (nthreads_fmt + 7) / 8;
    gpool.run(groups, [&](unsigned, uint64_t gb, uint64_t ge) {
        for (uint64_t q = gb; q < ge; q++) {
            uint64_t v = 0;
            for (int j = 0; j < 8; j++) {
                uint64_t g = q * 8 + j;
                v = (v << 5) | (g < nthreads_fmt ? (gap_vals[g] & 31u) : 0u);
            }
            for (int j = 0; j < 5; j++) {
                uint64_t at = q * 5 + j;
                if (at < r.gaps_bytes) r.gaps[at] = (uint8_t)(v >> (32 - 8 * j));
            }
        }
    });
    *out = r;
    return DF11_OK;
}

df11_status check_opts(const df11_encode_opts *opts, df11_encode_opts &o) {
    o.threads_per_block = 256;
    o.bytes_per_thread = 8;
    o.lut_mode = DF11_LUT_AUTO;
    o.num_threads = 0;
    o.value_format = DF11_VF_BF16;
    o.lut_bits = 8;
    if (opts) o = *opts;
    if (o.lut_bits == 0) o.lut_bits = 8;
    if (o.value_format > DF11_VF_FP8_E5M2) return df11_fail(DF11_E_INVALID_ARGUMENT, "bad value_format");
    if (o.lut_bits > 16 && o.lut_bits != DF11_LUT_BITS_MONOLITHIC)
        return df11_fail(DF11_E_INVALID_ARGUMENT, "lut_bits must be in [1, 16] or DF11_LUT_BITS_MONOLITHIC");
    if (o.threads_per_block < 32 || o.threads_per_block > 1024 || o.threads_per_block % 32)
        return df11_fail(DF11_E_INVALID_ARGUMENT, "threads_per_block must be a multiple of 32 in [32, 1024]");
    if (o.bytes_per_thread < 4 || o.bytes_per_thread > 32)
        return df11_fail(DF11_E_INVALID_ARGUMENT, "bytes_per_thread must be in [4, 32]");
    if (o.lut_mode > DF11_LUT_WIDE) return df11_fail(DF11_E_INVALID_ARGUMENT, "bad lut_mode");
    return DF11_OK;
}

}  // namespace

namespace {
df11_status encode_values(const void *w, uint64_t n, const df11_encode_opts &o, const Codebook &cb, const Pool &pool,
                          df11_host_tensor *out) {
    const VFmt &f = kVF[o.value_format];
    if (f.word_bytes == 2)
        return encode_with_codebook(static_cast<const uint16_t *>(w), n, f, o.value_format, o.threads_per_block,
                                    o.bytes_per_thread, cb, pool, out);
    return encode_with_codebook(static_cast<const uint8_t *>(w), n, f, o.value_format, o.threads_per_block,
                                o.bytes_per_thread, cb, pool, out);
}
}  // namespace

extern "C" df11_status df11_encode(const void *values, uint64_t n_elems, const df11_encode_opts *opts,
                                   df11_host_tensor *out) {
    if (!out) return df11_fail(DF11_E_INVALID_ARGUMENT, "out is NULL");
    std::memset(out, 0, sizeof(*out));
    if (!values && n_elems) return df11_fail(DF11_E_INVALID_ARGUMENT, "values is NULL");
    df11_encode_opts o;
    df11_status st = check_opts(opts, o);
    if (st != DF11_OK) return st;
    if (n_elems >= (1ull << 32)) return df11_fail(DF11_E_TOO_LARGE, "N >= 2^32 (BlockOutputPos is uint32)");
    try {
        Pool pool(o.num_threads, n_elems);
        uint64_t hist[256];
        histogram(values, n_elems, kVF[o.value_format], pool, hist);
        Codebook cb;
        st = make_codebook(hist, (int)o.lut_mode, o.lut_bits, cb);
        if (st != DF11_OK) return st;
        return encode_values(values, n_elems, o, cb, pool, out);
    } catch (const std::bad_alloc &) {
        return df11_fail(DF11_E_ALLOC, "host allocation failed");
    }
}

extern "C" df11_status df11_encode_group(const void *const *tensors, const uint64_t *n_elems, uint32_t count,
                                         const df11_encode_opts *opts, int shared_codebook, df11_host_tensor *outs) {
    if (!outs || (count && (!tensors || !n_elems))) return df11_fail(DF11_E_INVALID_ARGUMENT, "NULL argument");
    for (uint32_t i = 0; i < count; i++) std::memset(&outs[i], 0, sizeof(outs[i]));
    if (!shared_codebook) {
        for (uint32_t i = 0; i < count; i++) {
            df11_status st = df11_encode(tensors[i], n_elems[i], opts, &outs[i]);
            if (st != DF11_OK) {
                for (uint32_t j = 0; j < i; j++) df11_host_tensor_free(&outs[j]);
                return st;
            }
        }
        return DF11_OK;
    }
    df11_encode_opts o;
    df11_status st = check_opts(opts, o);
    if (st != DF11_OK) return st;
    try {
        uint64_t hist[256] = {};
        uint64_t total = 0;
        for (uint32_t i = 0; i < count; i++) {
            if (!tensors[i] && n_elems[i]) return df11_fail(DF11_E_INVALID_ARGUMENT, "tensor pointer is NULL");
            if (n_elems[i] >= (1ull << 32)) return df11_fail(DF11_E_TOO_LARGE, "N >= 2^32");
            Pool pool(o.num_threads, n_elems[i]);
            uint64_t h[256];
            histogram(tensors[i], n_elems[i], kVF[o.value_format], pool, h);
            for (int s = 0; s < 256; s++) hist[s] += h[s];
            total += n_elems[i];
        }
        Codebook cb;
        st = make_codebook(hist, (int)o.lut_mode, o.lut_bits, cb);
        if (st != DF11_OK) return st;
        for (uint32_t i = 0; i < count; i++) {
            Pool pool(o.num_threads, n_elems[i]);
            st = encode_values(tensors[i], n_elems[i], o, cb, pool, &outs[i]);
            if (st != DF11_OK) {
                for (uint32_t j = 0; j < i; j++) df11_host_tensor_free(&outs[j]);
                return df11_fail(st, "group encode failed");
            }
        }
        (void)total;
        return DF11_OK;
    } catch (const std::bad_alloc &) {
        return df11_fail(DF11_E_ALLOC, "host allocation failed");
    }
}

extern "C" void df11_host_tensor_free(df11_host_tensor *t) {
    if (!t) return;
    std::free(t->luts);
    std::free(t->encoded_exponent);
    std::free(t->packed_sign_mantissa);
    std::free(t->gaps);
    std::free(t->block_output_pos);
    std::memset(t, 0, sizeof(*t));
}

// ------------------------------------------------------------------------------------ device-encoder plan
// Host half of the GPU encoder (NEXT-3): the codebook is tiny (256 symbols), so it is built here with
// the same code as df11_encode; df11_encode_device (encode_gpu.cu) does the per-element work.
extern "C" df11_status df11_encode_plan_create(const uint64_t *codebook_hist, const uint64_t *tensor_hist,
                                               const df11_encode_opts *opts, df11_encode_plan *plan) {
    if (!plan) return df11_fail(DF11_E_INVALID_ARGUMENT, "plan is NULL");
    std::memset(plan, 0, sizeof(*plan));
    if (!codebook_hist) return df11_fail(DF11_E_INVALID_ARGUMENT, "codebook_hist is NULL");
    if (!tensor_hist) tensor_hist = codebook_hist;
    df11_encode_opts o;
    df11_status st = check_opts(opts, o);
    if (st != DF11_OK) return st;
    try {
        Codebook cb;
        st = make_codebook(codebook_hist, (int)o.lut_mode, o.lut_bits, cb);
        if (st != DF11_OK) return st;
        uint64_t n = 0, bits = 0;
        for (int s = 0; s < 256; s++) {
            if (tensor_hist[s] && !cb.len[s])
                return df11_fail(DF11_E_INVALID_ARGUMENT, "tensor_hist has an exponent the codebook does not code");
            n += tensor_hist[s];
            bits += tensor_hist[s] * cb.len[s];
        }
        if (n >= (1ull << 32)) return df11_fail(DF11_E_TOO_LARGE, "N >= 2^32 (BlockOutputPos is uint32)");
        const uint64_t block_bits = 8ull * o.bytes_per_thread * o.threads_per_block;
        const uint64_t B = (bits + block_bits - 1) / block_bits;
        plan->luts = (uint8_t *)std::calloc(std::max<size_t>(cb.luts.size(), 1), 1);
        if (!plan->luts) return df11_fail(DF11_E_ALLOC, "host allocation failed");
        if (!cb.luts.empty()) std::memcpy(plan->luts, cb.luts.data(), cb.luts.size());
        plan->luts_bytes = cb.luts.size();
        plan->num_elements = n;
        plan->encoded_bits = bits;
        plan->T = o.threads_per_block;
        plan->n = o.bytes_per_thread;
        plan->B = (uint32_t)B;
        plan->k = cb.k;
        plan->lut_entry_bytes = cb.entry_bytes;
        plan->max_code_len = cb.max_len;
        plan->lut_bits = cb.lut_bits;
        plan->value_format = o.value_format;
        std::memcpy(plan->code_lengths, cb.len, 256);
        std::memcpy(plan->codes, cb.code, sizeof(plan->codes));
        plan->encoded_exponent_bytes = B * o.threads_per_block * o.bytes_per_thread + 16;
        plan->packed_sign_mantissa_bytes = residual_bytes(n, kVF[o.value_format]);
        plan->gaps_bytes = roundup((5ull * B * o.threads_per_block + 7) / 8, 16) + 16;
        // workspace: one gap byte per format thread | one look-back word per pack segment | ticket
        const uint64_t segments = (n + DF11_ENCODE_SEGMENT - 1) / DF11_ENCODE_SEGMENT;
        plan->workspace_bytes = roundup(B * o.threads_per_block, 16) + 8 * roundup(segments, 2) + 16;
        return DF11_OK;
    } catch (const std::bad_alloc &) {
        return df11_fail(DF11_E_ALLOC, "host allocation failed");
    }
}

extern "C" void df11_encode_plan_free(df11_encode_plan *plan) {
    if (!plan) return;
    std::free(plan->luts);
    std::memset(plan, 0, sizeof(*plan));
}
