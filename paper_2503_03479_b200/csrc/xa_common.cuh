// xa_common.cuh — shared device types and helpers for the sm_100a hot path.
//
// Exactness policy: stages whose outputs the reference pins
// bit-for-bit given identical inputs (pyramid resize, FAST, NMS, Harris,
// centroid, sigma=2 blur, rBRIEF, Hamming) use explicitly rounded float/double
// intrinsics so nvcc cannot contract a*b+c into an FMA or reorder a sum; the
// view resamplers (blur + Lanczos) use fast FMA float math and are checked
// against the reference within tolerance.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace xa {

constexpr int kLevels = 8;           // orb.cpp:12
constexpr double kLevelRatio = 1.2;  // orb.cpp:13
constexpr int kFastThr = 20;         // orb.cpp:14
constexpr int kFastThrRelaxed = 7;   // orb.cpp:15
constexpr int kOrientR = 15;         // orb.cpp:16
constexpr int kDetectBorder = 17;    // orb.cpp:17
constexpr int kDescribeBorder = 20;  // orb.cpp:18
constexpr int kMinSide = 32;         // orb.cpp:19
constexpr int kSortCap = 8192;       // top-N sort buffer (entries)
constexpr int kListCap = 8192;       // top-N boundary-bin list (entries)
constexpr int kPyrRows = 64;         // rows per k_pyramid CTA (x 128 columns)
// k_fast_nms core tile. Width 60 keeps every tile origin at (ox-4) % 4 == 1,
// so 4-position groups of the FAST scan are 16-byte aligned in shared memory.
constexpr int kFastTileW = 60, kFastTileH = 30;

// cp.async (sm_80+ async global->shared copies, no register round trip).
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

// TMA bulk copies (cp.async.bulk, sm_90+): one instruction moves a whole
// 16-byte aligned row global -> shared; completion is counted in bytes on an
// mbarrier (expect_tx by one thread, complete_tx by the copy engine).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 2-D tensor TMA: one box of a tensor map (global memory, 64-byte aligned)
// into shared memory (128-byte aligned), completion on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Exact-rounding helpers: one rounding per op, never fused.
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// map_point (geometry.cpp:80-82): (m0*x + m1*y) + m2, no contraction.
__device__ __forceinline__ void map_pt(const double* m, double x, double y, double& ox,
                                       double& oy) {
    ox = dadd(dadd(dmul(m[0], x), dmul(m[1], y)), m[2]);
    oy = dadd(dadd(dmul(m[3], x), dmul(m[4], y)), m[5]);
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <class T>
__device__ __forceinline__ float ld_px(const T* p, size_t i);
template <>
__device__ __forceinline__ float ld_px<float>(const float* p, size_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ float ld_px<uint8_t>(const uint8_t* p, size_t i) {
    return (float)__ldg(p + i);
}

// ORB per-image descriptor shared by the pyramid / detect / describe kernels.
struct OrbImage {
    int nlev;
    int w[kLevels], h[kLevels];
    int pitch[kLevels];        // level row pitch (floats, multiple of 4 -> 16-byte rows)
    long long poff[kLevels];   // level offsets (floats, multiple of 4) into the pyramid buffer
    const void* src;           // level-0 source (u8 or f32), row-major w[0] x h[0]
    int src_type;              // 0 = u8, 1 = f32
    int max_points;
    long long cand_off;        // candidate buffer offset (records)
    int cand_cap;
    int filter;                // apply the coarse content filter (pipeline.cpp:28-40)
    int src_w, src_h;          // content-filter source dims
    double margin;
    double back[6];            // invert(WarpResult::forward), top two rows
    long long kp_off;          // keypoint/descriptor slot offset (max_points per image)
};

// Candidate record written by the FAST/NMS kernel.
//   x | y << 16, level | flags << 8 (bit0 survivor at thr 20, bit1 at thr 7)
struct Cand {
    uint32_t xy;
    uint32_t lf;
};

// Keypoint, layout-identical to xaffine::Keypoint (features.hpp:11-17).
struct xa_kp {
    float x, y, response, orientation, octave_scale;
};

// Per-candidate measured keypoint plus its 96-bit top-N key.
struct CandKey {
    uint32_t k0, k1, k2, idx;  // k0 = descending-response key, k1 = y bits, k2 = x bits
};

// A keypoint selected for description: level coordinates resolved.
struct DescKp {
    int lx, ly, level;
    float orientation;
    float cs, sn;  // glibc cosf/sinf of the orientation (set with it)
};

// Per-image counters (device).
struct ImgCounters {
    int n_cand;        // candidates appended (either set)
    int n20, n7;       // NMS survivors at the two thresholds
    int n_det;         // detect output count (<= max_points)
    int n_desc;        // described keypoints
    int overflow;      // capacity exceeded
    int pad[2];
};

}  // namespace xa
