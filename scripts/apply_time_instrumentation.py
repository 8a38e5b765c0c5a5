#!/usr/bin/env python
"""Write a copy of decode_sp12.cu that records %globaltimer per CTA (kernel entry, end of the first
table build, exit) and per group (last tile done) — profiling tooling, never the product build:

    python scripts/apply_time_instrumentation.py OUT.cu
    DF11_SRC_OVERRIDE=decode_sp12.cu=OUT.cu python scripts/build_variant.py times -DSP12_TIMES
    DF11_LIB=paper_2504_11651_b200/lib/variants/times.so python scripts/cta_times.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "paper_2504_11651_b200", "csrc", "decode_sp12.cu")).read()


def ins(marker, code, after=False):
    global s
    assert s.count(marker) == 1, marker
    s = s.replace(marker, marker + code if after else code + marker)


ins("// kVF: value format (DF11_VF_*, NEXT-4).  Decode, scan and compaction", """__device__ unsigned long long g_sp12_times[256][12];   // per CTA: entry, table built, exit, 8 groups' ends
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
""")
ins("    if (c_begin >= c_end) return;\n", """    if (tid == 0) { g_sp12_times[blockIdx.x][0] = gtimer(); uint32_t sm; asm("mov.u32 %0, %%smid;" : "=r"(sm)); g_sp12_times[blockIdx.x][11] = sm; }
    bool first_build = true;
""", after=True)
ins("        const uint32_t eb_bytes = ts.lut_entry_bytes, kk = ts.k;\n", """        if (tid == 0 && first_build) g_sp12_times[blockIdx.x][1] = gtimer();
        first_build = false;
""", after=True)
ins("#undef K_ROW\n", """    if (t == 0) g_sp12_times[blockIdx.x][3 + g] = gtimer();
    __syncthreads();
    if (tid == 0) g_sp12_times[blockIdx.x][2] = gtimer();
""")
ins("cudaError_t launch_sp12(", """extern "C" int df11_debug_sp12_times(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, g_sp12_times, sizeof(g_sp12_times));
}

""")
open(sys.argv[1], "w").write(s)
