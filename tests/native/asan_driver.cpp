// ASan / UBSan driver: the host encoder (paper_2504_11651_b200/csrc/encode.cpp) and
// the CPU oracle (oracle/df11_oracle.c) compiled with -fsanitize=address,undefined, run over edge-case
// and random inputs of every value format and LUT width; every library encoding is decoded by the
// oracle's D1 and D2 and must give the input back.  Test infrastructure (tests/test_native_sanitizers.py
// builds and runs it); exit code 0 = no sanitizer report and every round trip exact.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "df11.h"

extern "C" {
// the library's error recorder lives in api.cu (CUDA); the encoder only needs this much of it
df11_status df11_fail(df11_status st, const char *) { return st; }
int df11o_decode_sequential(const uint8_t *, uint64_t, const uint8_t *, const uint8_t *, uint64_t, uint64_t, int,
                            void *);
int df11o_decode_alg1(const uint8_t *, uint32_t, uint32_t, uint32_t, const uint8_t *, const uint8_t *, uint64_t,
                      const uint8_t *, uint64_t, const uint32_t *, const uint8_t *, uint64_t, uint32_t, uint32_t,
                      uint32_t, uint64_t, int, int, void *);
}

static int failures = 0;

static void check(const std::vector<uint8_t> &words, uint64_t n, uint32_t vf, uint32_t T, uint32_t nb,
                  uint32_t lut_bits, uint32_t lut_mode, const char *what) {
    df11_encode_opts o{T, nb, lut_mode, 0, vf, lut_bits};
    df11_host_tensor h;
    df11_status st = df11_encode(words.data(), n, &o, &h);
    if (st != DF11_OK) {
        if (!(lut_bits == DF11_LUT_BITS_MONOLITHIC && st == DF11_E_INVALID_ARGUMENT) &&
            !(lut_mode == DF11_LUT_NARROW && (st == DF11_E_RESERVED_EXPONENT || st == DF11_E_LUT_OVERFLOW))) {
            std::printf("FAIL encode %s vf=%u b=%u: status %d\n", what, vf, lut_bits, (int)st);
            failures++;
        }
        return;
    }
    const uint32_t wb = vf < 2 ? 2 : 1;
    std::vector<uint8_t> d1(n * wb + 1), d2(n * wb + 1);
    if (n) {
        int r1 = df11o_decode_sequential(h.encoded_exponent, h.encoded_exponent_bytes, h.code_lengths,
                                         h.packed_sign_mantissa, h.packed_sign_mantissa_bytes, n, (int)vf, d1.data());
        int r2 = df11o_decode_alg1(h.luts, h.lut_entry_bytes, h.k, h.lut_bits, h.code_lengths, h.encoded_exponent,
                                   h.encoded_exponent_bytes, h.gaps, h.gaps_bytes, h.block_output_pos,
                                   h.packed_sign_mantissa, h.packed_sign_mantissa_bytes, h.B, h.T, h.n, n, (int)vf, 1,
                                   d2.data());
        if (r1 || r2 || std::memcmp(d1.data(), words.data(), n * wb) || std::memcmp(d2.data(), words.data(), n * wb)) {
            std::printf("FAIL round trip %s vf=%u b=%u T=%u n=%u: %d %d\n", what, vf, lut_bits, T, nb, r1, r2);
            failures++;
        }
    }
    df11_host_tensor_free(&h);
}

int main() {
    std::mt19937_64 rng(12345);
    const uint32_t geoms[][2] = {{256, 8}, {128, 16}, {32, 4}, {64, 32}};
    const uint32_t bits[] = {8, 1, 5, 12, 16, DF11_LUT_BITS_MONOLITHIC};
    const uint64_t sizes[] = {0, 1, 7, 16, 17, 4097, 70001};
    int cases = 0;
    for (uint32_t vf = 0; vf < 4; vf++) {
        const uint32_t wb = vf < 2 ? 2 : 1;
        for (uint64_t n : sizes) {
            for (int kind = 0; kind < 3; kind++) {
                std::vector<uint8_t> w(n * wb + 1);
                std::normal_distribution<float> nd(0.f, 1.f);
                for (uint64_t i = 0; i < n; i++) {
                    uint32_t v;
                    if (kind == 0) v = (uint32_t)rng();                                   // every pattern
                    else if (kind == 1) v = vf < 2 ? 0x3C00u : 0x38u;                     // one symbol
                    else {                                                                  // skewed exponents
                        const uint32_t e = (uint32_t)std::min(30.0f, std::fabs(nd(rng)) * 4.0f);
                        v = (uint32_t)rng() & (vf == 0 ? 0x807Fu : vf == 1 ? 0x83FFu : vf == 2 ? 0x87u : 0x83u);
                        v |= (vf == 0 ? (120u - e) << 7 : vf == 1 ? (15u - std::min(e, 14u)) << 10
                                                        : vf == 2 ? (7u - std::min(e, 6u)) << 3 : (15u - std::min(e, 14u)) << 2);
                    }
                    if (wb == 2) { w[2 * i] = (uint8_t)v; w[2 * i + 1] = (uint8_t)(v >> 8); }
                    else w[i] = (uint8_t)v;
                }
                for (auto &g : geoms)
                    for (uint32_t b : bits) {
                        check(w, n, vf, g[0], g[1], b, DF11_LUT_AUTO, "case");
                        cases++;
                    }
                check(w, n, vf, 256, 8, 8, DF11_LUT_NARROW, "narrow");
                check(w, n, vf, 256, 8, 8, DF11_LUT_WIDE, "wide");
                cases += 2;
            }
        }
    }
    std::printf("%d cases, %d failures\n", cases, failures);
    return failures ? 1 : 0;
}
