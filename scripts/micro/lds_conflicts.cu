// Microbenchmark (profiling tooling, not product): shared-memory wavefronts of table lookups under
// the access patterns of the decode kernel.  Run under ncu and read l1tex__data_pipe_lsu_wavefronts_mem_shared
// per kernel.  pattern: 0 = all lanes random rows, 1 = lanes >= act read one common "null" entry,
// 2 = lanes >= act predicated off, 3 = LDS.32 random, 4 = LDS.32 with 2-replica, 5 = all same address.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

template <int PAT>
__global__ void k(uint32_t *out, int iters, int act) {
    extern __shared__ uint2 tab[];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) tab[i] = make_uint2(i, i * 3);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t s = hash(threadIdx.x + 977 * blockIdx.x), acc = 0;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
    for (int it = 0; it < iters; it++) {
        s = hash(s + acc);
        uint32_t row = s & 4095;
        uint32_t lo, hi;
        if (PAT == 0) {
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(base + row * 8));
        } else if (PAT == 1) {
            if (lane >= (uint32_t)act) row = 4096;
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(base + row * 8));
        } else if (PAT == 2) {
            lo = 0; hi = 0;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %3, %4;\n\t@p ld.shared.v2.u32 {%0,%1}, [%2];\n\t}"
                         : "+r"(lo), "+r"(hi) : "r"(base + row * 8), "r"(lane), "r"((uint32_t)act));
        } else if (PAT == 3) {
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(base + row * 4));
            hi = 0;
        } else if (PAT == 4) {
            // 2 replicas of a 2048-word table in bank halves: lane parity picks the half
            const uint32_t r = s & 2047;
            const uint32_t addr = base + (((r >> 4) << 5) | ((lane & 1) << 4) | (r & 15)) * 4;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(addr));
            hi = 0;
        } else if (PAT == 5) {
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(base + 4096 * 8));
        } else if (PAT == 6) {
            // LDS.128 random rows of 16 bytes over 32 KB
            uint32_t c, d;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(lo), "=r"(hi), "=r"(c), "=r"(d) : "r"(base + (row & 2047) * 16));
            lo ^= c ^ d;
        }
        acc += lo ^ hi;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    uint32_t *out;
    cudaMalloc(&out, 148 * 1024 * 4);
    const int smem = 4097 * 8;
    const int iters = 256;
    k<0><<<148, 1024, smem>>>(out, iters, 32);
    for (int a : {8, 16, 24}) k<1><<<148, 1024, smem>>>(out, iters, a);
    for (int a : {8, 16, 24}) k<2><<<148, 1024, smem>>>(out, iters, a);
    k<3><<<148, 1024, smem>>>(out, iters, 32);
    k<4><<<148, 1024, smem>>>(out, iters, 32);
    k<5><<<148, 1024, smem>>>(out, iters, 32);
    k<6><<<148, 1024, smem>>>(out, iters, 32);
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
