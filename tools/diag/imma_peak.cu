// Throughput probe: legacy warp-level mma.sync m16n8k32 u8 (IMMA.16832) on B200.
// Each warp runs 8 independent accumulator chains; reports dense int8 MAC/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_imma(int iters, int* out) {
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
    int c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    if (s == 0x7fffffff) out[0] = s;
}
int main() {
    int* d; cudaMalloc(&d, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int wpb : {4, 8, 16}) {
        const int blocks = 148 * 4;
        k_imma<<<blocks, 32 * wpb>>>(16, d);
        cudaEventRecord(e0);
        k_imma<<<blocks, 32 * wpb>>>(iters, d);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double macs = (double)blocks * wpb * iters * 8 * 16 * 8 * 32;
        printf("{\"probe\": \"imma_m16n8k32_u8\", \"warps_per_cta\": %d, \"ms\": %.3f, \"tmac_per_s\": %.2f, \"hamming_cmp_per_s_256bit\": %.3e}\n",
               wpb, ms, macs / ms / 1e9, macs / 256.0 / ms * 1e3);
    }
    return 0;
}
