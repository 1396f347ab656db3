// Does ptxas contract explicit mul.rn.f32x2 + add.rn.f32x2 into FFMA2?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/diag/f32x2_contract tools/diag/f32x2_contract.cu
// (cuobjdump shows FFMA2 even with --fmad=false). Prints both results for an
// input where the fused and the twice-rounded values differ.
#include <cstdio>
__device__ __forceinline__ float2 fmul2x(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2x(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}
__global__ void k(const float2* a, const float2* b, const float2* c, float2* o, float* s) {
    o[0] = fadd2x(c[0], fmul2x(a[0], b[0]));
    s[0] = __fadd_rn(c[0].x, __fmul_rn(a[0].x, b[0].x));
    s[1] = __fmaf_rn(a[0].x, b[0].x, c[0].x);
}
int main() {
    float2 h[3] = {{1.f + 1.f / 4096, 1.f + 1.f / 4096}, {1.f + 1.f / 4096, 1.f + 1.f / 4096}, {-1.f, -1.f}};
    float2 *d, *o; float* s;
    cudaMalloc(&d, sizeof h); cudaMalloc(&o, 8); cudaMalloc(&s, 8);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    k<<<1, 1>>>(d, d + 1, d + 2, o, s);
    float2 ho; float hs[2];
    cudaMemcpy(&ho, o, 8, cudaMemcpyDeviceToHost); cudaMemcpy(hs, s, 8, cudaMemcpyDeviceToHost);
    printf("f32x2 %.10e  unfused %.10e  fused %.10e\n", ho.x, hs[0], hs[1]);
    return 0;
}
