#!/usr/bin/env python
"""Write a clock64 phase-instrumented copy of decode_sp12.cu (profiling tooling, never the product build):

    python scripts/apply_prof_instrumentation.py OUT.cu

Then build a variant from it with -DSP12_PROF (see scripts/phase_profile.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "paper_2504_11651_b200", "csrc", "decode_sp12.cu")).read()


def ins(marker, code, after=False):
    global s
    assert s.count(marker) == 1, marker
    s = s.replace(marker, marker + code if after else code + marker)


ins("// kVF: value format (DF11_VF_*, NEXT-4).  Decode, scan and compaction", """__device__ unsigned long long g_sp12_prof[148 * 32][8];   // per warp: cycles per phase
#define PROF_MARK(i) do { const long long _n = clock64(); if (lane == 0) prof[i] += _n - prof_t; prof_t = _n; } while (0)
""")
ins("    const uint32_t FULL = 0xFFFFFFFFu;\n", """    unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long prof_t = clock64();
""", after=True)
ins("            mbar_wait(mbar, q & 1u);\n", "            PROF_MARK(0);\n")
ins("            mbar_wait(mbar, q & 1u);\n", "            PROF_MARK(1);\n", after=True)
ins("            const uint32_t cnt = cntA + cntB;\n", "            PROF_MARK(2);\n")
ins("            group_bar(g);                          // also: every thread has read this tile's stage\n", "            PROF_MARK(3);\n")
ins("            group_bar(g);                          // also: every thread has read this tile's stage\n", "            PROF_MARK(4);\n", after=True)
ins("                const uint32_t dA = wreg + (wbeg - F) + lpos, dB = dA + cntA;\n", "                PROF_MARK(5);\n")
ins("            // ---- per-warp merge of [ra, rb): compose BF16 and store (P:439-441)\n", "            PROF_MARK(6);\n")
ins("                mbar_wait(smbar, qs & 1u);                                     // PackedSignMantissa staged\n", "                PROF_MARK(7);\n", after=True)
ins("#undef K_ROW\n#undef K_TOP", """    if (lane == 0)
        for (int i = 0; i < 8; i++) g_sp12_prof[blockIdx.x * 32 + (tid >> 5)][i] = prof[i];
""")
ins("cudaError_t launch_sp12(", """extern "C" int df11_debug_sp12_prof(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, g_sp12_prof, sizeof(g_sp12_prof));
}

""")
open(sys.argv[1], "w").write(s)
