// Validates the hand-built tcgen05 kind::i8 path (smem descriptors for the
// K-major no-swizzle canonical layout, instruction descriptor, TMEM alloc,
// commit -> mbarrier, 32x32b loads) against a host int GEMM:
// D[128 x 256] = A[128 x 256] . B[256 x 256]^T with +-1 s8 entries.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 256, K = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__global__ void __launch_bounds__(128) k_check(const int8_t* __restrict__ a, const int8_t* __restrict__ b,
                                               int32_t* __restrict__ d) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;              // [K/16][M][16]
    uint8_t* sB = sm + M * K;      // [K/16][N][16]
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    for (int i = tid; i < M * K / 16; i += blockDim.x) {
        const int r = i / (K / 16), c = i % (K / 16);
        *reinterpret_cast<uint4*>(sA + c * (M * 16) + r * 16) = *reinterpret_cast<const uint4*>(a + r * K + c * 16);
    }
    for (int i = tid; i < N * K / 16; i += blockDim.x) {
        const int r = i / (K / 16), c = i % (K / 16);
        *reinterpret_cast<uint4*>(sB + c * (N * 16) + r * 16) = *reinterpret_cast<const uint4*>(b + r * K + c * 16);
    }
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&s_tmem)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;
    if (tid == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int s = 0; s < K / 32; ++s) {
            const uint64_t da = umma_desc(smem_u32(sA + 2 * s * (M * 16)), M * 16, 128);
            const uint64_t db = umma_desc(smem_u32(sB + 2 * s * (N * 16)), N * 16, 128);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                         :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(s));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    }
    // wait for the MMAs
    asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" :: "r"(smem_u32(&bar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w reads TMEM lanes 32w..32w+31 (rows), 32 columns at a time
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        const uint32_t addr = tmem + ((uint32_t)(32 * wid) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 32; ++j) d[(32 * wid + lane) * N + c0 + j] = (int32_t)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(256));
}


// K-major SWIZZLE_128B: [K half][row][128 B], 16-byte chunk c of row r stored at c ^ (r % 8)
__global__ void __launch_bounds__(128) k_check_sw(const int8_t* __restrict__ a, const int8_t* __restrict__ b,
                                                  int32_t* __restrict__ d) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;
    uint8_t* sB = sm + M * K;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    for (int i = tid; i < M * K / 16; i += blockDim.x) {
        const int r = i / (K / 16), c = i % (K / 16), kh = c / 8, cc = c % 8;
        *reinterpret_cast<uint4*>(sA + kh * (M * 128) + r * 128 + ((cc ^ (r & 7)) * 16)) =
            *reinterpret_cast<const uint4*>(a + r * K + c * 16);
    }
    for (int i = tid; i < N * K / 16; i += blockDim.x) {
        const int r = i / (K / 16), c = i % (K / 16), kh = c / 8, cc = c % 8;
        *reinterpret_cast<uint4*>(sB + kh * (N * 128) + r * 128 + ((cc ^ (r & 7)) * 16)) =
            *reinterpret_cast<const uint4*>(b + r * K + c * 16);
    }
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&s_tmem)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;
    if (tid == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int s = 0; s < K / 32; ++s) {
            const uint64_t da = umma_desc(smem_u32(sA + (s / 4) * (M * 128) + (s % 4) * 32), 16, 1024, 2);
            const uint64_t db = umma_desc(smem_u32(sB + (s / 4) * (N * 128) + (s % 4) * 32), 16, 1024, 2);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                         :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(s));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" :: "r"(smem_u32(&bar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        const uint32_t addr = tmem + ((uint32_t)(32 * wid) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 32; ++j) d[(32 * wid + lane) * N + c0 + j] = (int32_t)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(256));
}

int main() {
    std::vector<int8_t> a(M * K), b(N * K);
    srand(7);
    for (auto& x : a) x = (rand() & 1) ? 1 : -1;
    for (auto& x : b) x = (rand() & 1) ? 1 : -1;
    int8_t *da, *db; int32_t* dd;
    cudaMalloc(&da, a.size()); cudaMalloc(&db, b.size()); cudaMalloc(&dd, M * N * 4);
    cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
    cudaMemset(dd, 0x7f, M * N * 4);
    const int smem = (M + N) * K;
    int bad_total = 0;
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(dd, 0x7f, M * N * 4);
        if (variant == 0) {
            cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_check<<<1, 128, smem>>>(da, db, dd);
        } else {
            cudaFuncSetAttribute(k_check_sw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_check_sw<<<1, 128, smem>>>(da, db, dd);
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("{\"umma_i8_check\": \"cuda error %s\"}\n", cudaGetErrorString(e)); return 1; }
        std::vector<int32_t> d(M * N);
        cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0, first = -1;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                int s = 0;
                for (int k = 0; k < K; ++k) s += a[i * K + k] * b[j * K + k];
                if (s != d[i * N + j]) { if (first < 0) first = i * N + j; ++bad; }
            }
        printf("{\"umma_i8_check\": \"%s\", \"layout\": \"%s\", \"mismatches\": %d, \"first\": %d}\n",
               bad ? "FAIL" : "ok", variant ? "K-major SWIZZLE_128B" : "K-major no swizzle", bad, first);
        bad_total += bad;
    }
    int bad = bad_total;
    return bad ? 1 : 0;
}
