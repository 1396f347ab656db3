// POPC throughput probe for the roofline denominator of the Hamming matcher
// (SURVEY.md §8d asks to confirm 16/clk/SM for cc 10.0 before using it).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o popc_peak popc_peak.cu && ./popc_peak
//
// Each thread runs independent chains of popc(x ^ k) + acc over 32-bit words
// (the matcher's inner op); the SASS holds POPC + IADD3/LOP3 per word. Prints
// POPC per clock per SM at the measured SM clock.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_popc(unsigned* out, int iters, unsigned seed) {
    unsigned x[CH], acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        x[c] = seed * (threadIdx.x + 1) + c * 0x9e3779b9u;
        acc[c] = 0;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            acc[c] += __popc(x[c] ^ (unsigned)i);
            x[c] = x[c] * 1664525u + 1013904223u;  // keep the operand live (IMAD)
        }
    }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 0x12345678u) out[0] = s;
}

template <int CH>
__global__ void k_popc_only(unsigned* out, int iters, unsigned seed) {
    // pure POPC: operands are loop-invariant registers, results summed pairwise
    unsigned x[CH], acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        x[c] = seed * (threadIdx.x + 1) + c * 0x9e3779b9u;
        acc[c] = 0;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] += __popc(x[c] ^ acc[(c + 1) % CH]);
    }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 0x12345678u) out[0] = s;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    unsigned* d;
    cudaMalloc(&d, 4);
    const int iters = 1 << 14, threads = 512, blocks = p.multiProcessorCount * 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        for (int kind = 0; kind < 2; ++kind) {
            cudaEventRecord(a);
            if (kind == 0)
                k_popc<8><<<blocks, threads>>>(d, iters, 7);
            else
                k_popc_only<8><<<blocks, threads>>>(d, iters, 7);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double popc = (double)blocks * threads * iters * 8;
            const double per_s = popc / (ms * 1e-3);
            const double per_clk_sm = per_s / (p.multiProcessorCount * 1965e6);
            if (rep)
                printf("{\"kind\": \"%s\", \"sms\": %d, \"ms\": %.3f, \"popc_per_s\": %.4e, "
                       "\"popc_per_clk_per_sm_at_1965MHz\": %.2f, \"attr_clock_khz\": %d}\n",
                       kind ? "popc_chain" : "popc_xor_imad", p.multiProcessorCount, ms, per_s, per_clk_sm,
                       clk_khz);
        }
    }
    return 0;
}
