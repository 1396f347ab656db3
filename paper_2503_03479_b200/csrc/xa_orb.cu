// xa_orb.cu — ORB extraction on sm_100a, batched over images (target + views).
//
// Reference: proj/src/orb.cpp (detect_oriented_corners :182-210,
// describe_binary :212-248 and their helpers :25-172), proj/src/image.cpp
// (resize_bilinear, gaussian_blur), proj/src/pipeline.cpp:28-40
// (filter_to_content). Given identical level-0 pixels every output here is
// bit-identical to the reference (tests/test_gpu_orb.py):
//   k_pyramid    levels resized from level 0, exact float/double replay
//   k_fast_nms   FAST-9 + score + the 3x3 raster-tie NMS per 60x30 tile: a
//                threshold-20 pass over every image, then the auto-relax
//                pass at threshold 7 (orb.cpp:187-188) whose CTAs run only
//                for images left with < max_points/4 threshold-20 corners -
//                the reference's re-run, decided on the device.
//   k_measures   Harris + intensity-centroid per candidate, reference order
//   k_select     per-image top-N: 32-bit radix select on the response key,
//                then a bitonic sort of the survivors on the exact 96-bit key
//                (response desc, y, x); fused with the content filter and the
//                describe-border drop (order preserving)
//   k_describe   one warp per keypoint: 49x49 window -> sigma=2 separable blur
//                in shared memory -> 256 steered comparisons -> 8 ballots
#include <cuda_fp16.h>
#include <math.h>

#include "xa_common.cuh"
#include "xa_kernels.h"

namespace xa {

#include "trig_fixups.inc"  // XA_TRIG_* macros only
struct TrigFix {
    uint32_t x, c, s;
};
#define XA_TRIG_TABLE_BODY
__constant__ TrigFix c_trig[XA_TRIG_FIXUPS] = {
#include "trig_fixups.inc"
};
#undef XA_TRIG_TABLE_BODY

static const int8_t h_pattern[1024] = {
#include "orb_pattern.inc"
};
__device__ int8_t g_pattern[1024] = {
#include "orb_pattern.inc"
};

__constant__ float c_level_scale[kLevels];  // (float)pow(1.2, L) (orb.cpp:195)
__constant__ int c_umax[kOrientR + 1];      // make_umax() (orb.cpp:25-41)
__constant__ float c_blur2[13];             // gaussian_kernel(2.0) (image.cpp:10-21)
__constant__ double c_log_ratio;            // log(1.2)

// Bresenham ring of radius 3 (orb.cpp:21-22) as compile-time offsets, so the
// 16 ring reads fold into immediate shared-memory offsets.
__host__ __device__ constexpr int ring_dx(int r) {
    return r == 0 ? 0 : r == 1 ? 1 : r == 2 ? 2 : r <= 5 ? 3 : r == 6 ? 2 : r == 7 ? 1 : r == 8 ? 0
         : r == 9 ? -1 : r == 10 ? -2 : r <= 13 ? -3 : r == 14 ? -2 : -1;
}
__host__ __device__ constexpr int ring_dy(int r) { return ring_dx((r + 12) & 15); }
static_assert(ring_dy(0) == -3 && ring_dy(4) == 0 && ring_dy(8) == 3 && ring_dy(12) == 0 &&
                  ring_dy(1) == -3 && ring_dy(5) == 1 && ring_dy(15) == -3,
              "ring offsets");

uint64_t pattern_checksum_host() {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int i = 0; i < 1024; ++i) {
        const int32_t v = h_pattern[i];
        for (int b = 0; b < 4; ++b) {
            h ^= (uint8_t)(v >> (8 * b));
            h *= 0x100000001b3ull;
        }
    }
    return h;
}

int trig_fixup_count() { return XA_TRIG_FIXUPS; }

__global__ void k_select(const OrbImage* __restrict__, const CandKey* __restrict__,
                         const xa_kp* __restrict__, const Cand* __restrict__, Cand* __restrict__,
                         int* __restrict__, ImgCounters* __restrict__,
                         xa_kp* __restrict__, DescKp* __restrict__, xa_kp* __restrict__,
                         SelState* __restrict__, const CandKey* __restrict__,
                         const uint2* __restrict__);
__global__ void k_describe(const OrbImage* __restrict__, const float* __restrict__,
                           const ImgCounters* __restrict__, const DescKp* __restrict__,
                           uint64_t* __restrict__);
constexpr int DESC_WARPS = 4;
constexpr int WIN = 49, HALF = 24, PAT = 37, PHALF = 18;
constexpr int WS = 52;               // window row stride (16-byte rows, +3 pad columns)
constexpr int TS = 40, TR = 52;      // H-pass buffer: row stride, rows (49 + 3 pad)
constexpr int DESC_SMEM = (2 * WIN * WS + TR * TS) * 4;  // two windows + H-pass buffer

// Host-side constant setup (called once per device by the engine).
int orb_init_constants() {
    float ls[kLevels];
    for (int i = 0; i < kLevels; ++i) ls[i] = (float)pow(kLevelRatio, i);
    int umax[kOrientR + 1] = {0};
    {
        const int r = kOrientR;
        const int vmax = (int)floor(r * sqrt(2.0) / 2 + 1);
        const int vmin = (int)ceil(r * sqrt(2.0) / 2);
        for (int v = 0; v <= vmax; ++v) umax[v] = (int)round(sqrt((double)r * r - v * v));
        int v0 = 0;
        for (int v = r; v >= vmin; --v) {
            while (umax[v0] == umax[v0 + 1]) ++v0;
            umax[v] = v0;
            ++v0;
        }
    }
    float k[13];
    {
        double sum = 0;
        for (int i = -6; i <= 6; ++i) {
            const double v = exp(-0.5 * i * i / (2.0 * 2.0));
            k[i + 6] = (float)v;
            sum += v;
        }
        for (int i = 0; i < 13; ++i) k[i] = (float)(k[i] / sum);
    }
    const double lr = log(kLevelRatio);
    if (cudaMemcpyToSymbol(c_level_scale, ls, sizeof ls) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(c_umax, umax, sizeof umax) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(c_blur2, k, sizeof k) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(c_log_ratio, &lr, sizeof lr) != cudaSuccess) return -1;
    // opt-in shared memory (per device; called once per engine)
    if (cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSortCap * (int)sizeof(CandKey) + kListCap * (int)sizeof(uint2)) != cudaSuccess)
        return -1;
    if (cudaFuncSetAttribute(k_describe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DESC_SMEM) != cudaSuccess)
        return -1;
    return 0;
}

__device__ __forceinline__ int find_seg(const LevelSeg* __restrict__ segs, int n, int blk) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].blk_start <= blk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------------------ FAST + NMS

constexpr int TW = kFastTileW, TH = kFastTileH;  // NMS tile (core pixels per tile): 60 x 30
constexpr int SH = TH + 8;                  // staged rows (FAST+NMS halo 4): 38
constexpr int FWV = TW + 2;                 // valid FAST positions per row (NMS halo 1): 62
constexpr int FW = 64, FH = TH + 2;         // position grid stride 64 (62 valid) x 32
constexpr int NF = FW * FH;                 // 2048 FAST positions per tile

// Warp-cooperative 32-ary search: last segment with blk_start <= blk
// (two dependent loads for up to 1024 segments instead of a serial bisection).
__device__ __forceinline__ int find_seg_warp(const LevelSeg* __restrict__ segs, int n, int blk) {
    const int lane = threadIdx.x & 31;
    int base = 0, span = n;
    while (span > 1) {
        const int stride = (span + 31) >> 5;
        const int off = lane * stride;
        const bool ok = off < span && segs[base + off].blk_start <= blk;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        const int k = 31 - __clz(m);
        base += k * stride;
        span = min(stride, span - k * stride);
    }
    return base;
}

// ------------------------------------------------------------------ pyramid

// build_pyramid (orb.cpp:130-141): level 0 copied, level i resized directly
// from level 0 (image.cpp:51-70, exact rounding). One CTA = a 128-column x
// kPyrRows-row block of one level; thread -> one column, half the rows. The
// column's x interpolation (double, exact) is computed once, the rows' y
// interpolation once per CTA (as source-row offsets). Coarse views arrive
// with level 0 already written by the view resampler (XA_PIX_PYR0): their
// level-0 blocks are not planned and levels 1.. read the float level 0
// (row stride spitch = its pitch) instead of the uint8 view.
template <class T>
__device__ __forceinline__ void pyr_rows(const T* __restrict__ src, int spitch, int w0, int h0, int w,
                                         int h, int pitch, int L, int y, int y1, int xb,
                                         float* __restrict__ out, int* s_ra, int* s_rb, float* s_wy) {
    const int x = xb + (threadIdx.x & 127);
    const int r0 = y + (threadIdx.x >> 7) * (kPyrRows / 2);
    const int r1 = min(y1, r0 + kPyrRows / 2);
    if (L == 0) {
        if (x < w)
#pragma unroll 4
            for (int yy = r0; yy < r1; ++yy) out[(size_t)yy * pitch + x] = ld_px(src, (size_t)yy * spitch + x);
        return;
    }
    if ((int)threadIdx.x < y1 - y) {  // per-row y interpolation, once per CTA
        const double fy = dsub(dmul(dadd((double)(y + threadIdx.x), 0.5), (double)h0 / h), 0.5);
        const int y0 = (int)floor(fy);
        s_ra[threadIdx.x] = clampi(y0, 0, h0 - 1) * spitch;
        s_rb[threadIdx.x] = clampi(y0 + 1, 0, h0 - 1) * spitch;
        s_wy[threadIdx.x] = (float)dsub(fy, (double)y0);
    }
    __syncthreads();
    if (x >= w) return;
    const double fx = dsub(dmul(dadd((double)x, 0.5), (double)w0 / w), 0.5);
    const int x0 = (int)floor(fx);
    const float wx = (float)dsub(fx, (double)x0), iwx = fsub(1.f, wx);
    const T* ca = src + clampi(x0, 0, w0 - 1);
    const T* cc = src + clampi(x0 + 1, 0, w0 - 1);
    float* o = out + (size_t)r0 * pitch + x;
#pragma unroll 4
    for (int yy = r0; yy < r1; ++yy, o += pitch) {
        const int ra = s_ra[yy - y], rb = s_rb[yy - y];
        const float wy = s_wy[yy - y], iwy = fsub(1.f, wy);
        const float v00 = ld_px(ca, ra), v10 = ld_px(cc, ra), v01 = ld_px(ca, rb), v11 = ld_px(cc, rb);
        *o = fadd(fmul(iwy, fadd(fmul(iwx, v00), fmul(wx, v10))), fmul(wy, fadd(fmul(iwx, v01), fmul(wx, v11))));
    }
}

// ZERO: the block is in the zero background of a coarse view (every 2x2
// source is 0.f outside the content), written as 0.f without the gather.
template <bool ZERO>
__global__ void __launch_bounds__(256) k_pyramid(const OrbImage* __restrict__ imgs,
                                                 const LevelSeg* __restrict__ segs, int nsegs,
                                                 float* __restrict__ pyr) {
    __shared__ int s_i[8];
    __shared__ const void* s_src;
    __shared__ long long s_off;
    __shared__ int s_ra[kPyrRows], s_rb[kPyrRows];
    __shared__ float s_wy[kPyrRows];
    if (threadIdx.x < 32) {
        const int k = find_seg_warp(segs, nsegs, blockIdx.x);
        if (threadIdx.x == 0) {
            const LevelSeg sg = segs[k];
            const OrbImage& im = imgs[sg.img];
            const int lb = blockIdx.x - sg.blk_start;
            s_i[0] = sg.level;
            s_i[1] = sg.r0 + (lb / sg.tiles_x) * kPyrRows;   // first row
            s_i[2] = (sg.c0 + lb % sg.tiles_x) * 128;        // first column
            s_i[3] = im.w[sg.level] | (im.h[sg.level] << 16);
            s_i[4] = im.w[0] | (im.h[0] << 16);
            s_i[5] = im.src_type;
            s_i[6] = im.pitch[sg.level];
            s_i[7] = im.src_type == XA_PIX_PYR0 ? im.pitch[0] : im.w[0];
            s_src = im.src_type == XA_PIX_PYR0 ? (const void*)(pyr + im.poff[0]) : im.src;
            s_off = im.poff[sg.level];
        }
    }
    __syncthreads();
    const int L = s_i[0], y = s_i[1], xb = s_i[2];
    const int w = s_i[3] & 0xFFFF, h = s_i[3] >> 16, w0 = s_i[4] & 0xFFFF, h0 = s_i[4] >> 16;
    float* out = pyr + s_off;
    const int y1 = min(h, y + kPyrRows);
    if (ZERO) {
        // 16-byte zero stores: the pitch and xb are multiples of 4 floats; the
        // last column group may run into the pitch padding (no reader takes
        // it as pixels)
        const int x = xb + 4 * (threadIdx.x & 31);
        if (x >= w) return;
        for (int yy = y + (threadIdx.x >> 5); yy < y1; yy += 8)
            *reinterpret_cast<float4*>(out + (size_t)yy * s_i[6] + x) = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    if (s_i[5] == XA_PIX_U8)
        pyr_rows((const uint8_t*)s_src, s_i[7], w0, h0, w, h, s_i[6], L, y, y1, xb, out, s_ra, s_rb, s_wy);
    else
        pyr_rows((const float*)s_src, s_i[7], w0, h0, w, h, s_i[6], L, y, y1, xb, out, s_ra, s_rb, s_wy);
}

// 3-input min / max (FMNMX3 on sm_100a); exact like any min/max.
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// Segment test via order statistics (exact): a run of 9 ring pixels all
// brighter than hi exists iff A = max_i min_{j<9} v[i+j] > hi, all darker than
// lo iff B = min_i max_{j<9} v[i+j] < lo (orb.cpp:43-72). One pass answers both
// thresholds (20 and the auto-relax 7).
__device__ __forceinline__ void ring_extrema(const float* v, float& A, float& B) {
    float mn3[16], mx3[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        mn3[i] = fmin3(v[i], v[(i + 1) & 15], v[(i + 2) & 15]);
        mx3[i] = fmax3(v[i], v[(i + 1) & 15], v[(i + 2) & 15]);
    }
    float a[16], b[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        a[i] = fmin3(mn3[i], mn3[(i + 3) & 15], mn3[(i + 6) & 15]);
        b[i] = fmax3(mx3[i], mx3[(i + 3) & 15], mx3[(i + 6) & 15]);
    }
    float a5[6], b5[6];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        a5[k] = fmax3(a[3 * k], a[3 * k + 1], a[3 * k + 2]);
        b5[k] = fmin3(b[3 * k], b[3 * k + 1], b[3 * k + 2]);
    }
    A = fmax3(fmax3(a5[0], a5[1], a5[2]), fmax3(a5[3], a5[4], a[15]), -INFINITY);
    B = fmin3(fmin3(b5[0], b5[1], b5[2]), fmin3(b5[3], b5[4], b[15]), INFINITY);
}


// Stage the level window of a tile with 16-byte cp.async: pyramid rows are
// 16-byte aligned (pitch % 4 == 0) and (ox-4) % 4 == 1 for every tile, so each
// row copies 72 floats from the aligned column ox-5: level column ox-4+c sits
// at buffer column c+1, FAST position fx (level column ox-1+fx) at fx+4. No
// column clamp is needed: only positions of the scan region [17, w-17) are
// evaluated and their ring stays inside the level; extra columns read the
// pitch padding / next row (the pyramid buffer has tail slack). Rows clamp at
// the bottom.
constexpr int SWA = 72;
constexpr int kTileFloats = SH * SWA + 16;  // staging buffer, padded to a 128-byte multiple
static_assert((kTileFloats * 4) % 128 == 0, "TMA destinations stay 128-byte aligned");
// One 2-D tensor TMA per tile: the 72 x 38 box at (ox-5, oy-4) of the level
// (tensor map of width = pitch; rows past the level's end are zero-filled and
// never evaluated), completion counted on the buffer's mbarrier.
__device__ __forceinline__ void fast_stage(float* dst, const void* map, int ox, int oy, uint64_t* bar) {
    if (threadIdx.x == 0) {
        mbar_arrive_tx(bar, SH * SWA * (unsigned)sizeof(float));
        tma_load_2d(dst, map, ox - 5, oy - 4, bar);
    }
}

// FAST-9 (both thresholds) + sum-abs score + 3x3 NMS. One CTA walks one row of
// 60x30 tiles of one pyramid level (the next tile's window is prefetched by
// TMA while the current one is processed). Per tile (62x32 positions
// including the 1-px NMS halo, on a 64-wide grid):
//   A    compass test at thr 7 in min/max form (a 9-run always covers two
//        adjacent compass points), 4 positions per thread from 16-byte
//        loads -> queue (~1-15% of positions)
//   B    full segment test + score for the queue (order statistics, FMNMX3);
//        corners set bits in two 2048-bit maps (thr 7, thr 20) -> corner queue
//   NMS  raster tie rule (orb.cpp:152-169) for both sets, only at corners;
//        survivors appended with one global atomic per warp-iteration.
// MODE 0: threshold 20 only (every image). MODE 1: the auto-relax pass at
// threshold 7 (with the threshold-20 flags needed by nothing but kept for the
// candidate record), run only for images whose threshold-20 survivors fell
// below max_points / 4 (orb.cpp:187-188) - most images never need it, and the
// compass test at 7 lets ~4x more positions into the full test than at 20.
template <int MODE>
__device__ __forceinline__ void fast_nms_row(int blk, const OrbImage* __restrict__ imgs,
                                             const LevelSeg* __restrict__ segs, int nsegs,
                                             const TileRange* __restrict__ rng,
                                             const float* __restrict__ pyr, const char* __restrict__ maps,
                                             Cand* __restrict__ cand, ImgCounters* __restrict__ cnt,
                                             uint64_t* s_bar, unsigned& phase) {
    __shared__ __align__(128) float s_px[2][kTileFloats];
    __shared__ __align__(16) __half s_hx[SH][SWA];  // half copy of the tile for the compass test
    __shared__ float s_sc[NF];
    __shared__ __align__(16) uint8_t s_flag[NF];
    __shared__ uint16_t s_q[NF];   // 8 per-warp queues of NF/8 entries
    __shared__ int s_seg[4];        // img, level, tile row, tiles_x
    __shared__ int s_dim[3];        // w, h, pitch
    __shared__ long long s_lvoff, s_candoff;
    __shared__ int s_candcap;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const TileRange tr = rng[blk];  // tiles of this row that can see view content
    if (tr.lo >= tr.hi) return;
    // auto-relax pass: images that kept enough threshold-20 corners skip it
    if (MODE == 1 && cnt[tr.img].n20 >= imgs[tr.img].max_points / 4) return;
    if (wid == 0) {
        const int k = find_seg_warp(segs, nsegs, blk);
        if (lane == 0) {
            const LevelSeg sg = segs[k];
            const OrbImage& im = imgs[sg.img];
            s_seg[0] = sg.img;
            s_seg[1] = sg.level;
            s_seg[2] = blk - sg.blk_start;
            s_seg[3] = sg.tiles_x;
            s_dim[0] = im.w[sg.level];
            s_dim[1] = im.h[sg.level];
            s_dim[2] = im.pitch[sg.level];
            s_lvoff = im.poff[sg.level];
            s_candoff = im.cand_off;
            s_candcap = im.cand_cap;
        }
    }
    __syncthreads();
    const int img = s_seg[0], L = s_seg[1];
    constexpr int kThrA = MODE == 0 ? kFastThr : kFastThrRelaxed;  // compass / corner threshold
    const int w = s_dim[0], h = s_dim[1], pitch = s_dim[2];
    const float* lv = pyr + s_lvoff;
    const int oy = kDetectBorder + s_seg[2] * TH;
    const int xe = w - kDetectBorder, ye = h - kDetectBorder;
    const uint32_t lt = (1u << lane) - 1u;
    const int fx0 = 4 * (tid & 15), fy0 = tid >> 4;  // phase A: 4 positions, rows fy0, fy0+16
    // valid-column mask of this thread's 4 positions in a tile clear of both
    // scan borders (almost all): every position of the 62-wide row
    const unsigned colm_full = fx0 + 4 <= FWV ? 0xFu : (1u << (FWV - fx0)) - 1u;
    int n20 = 0, n7 = 0;

    const char* map = maps + (size_t)(img * kLevels + L) * 128;
    fast_stage(s_px[tr.lo & 1], map, kDetectBorder + tr.lo * TW, oy, &s_bar[tr.lo & 1]);
    for (int tx = tr.lo; tx < tr.hi; ++tx) {
        const int ox = kDetectBorder + tx * TW, b = tx & 1;
        float(*px)[SWA] = reinterpret_cast<float(*)[SWA]>(s_px[b]);
        // the other buffer was released by the previous tile's closing barrier
        if (tx + 1 < tr.hi) fast_stage(s_px[b ^ 1], map, ox + TW, oy, &s_bar[b ^ 1]);
        if (tid < NF / 16) reinterpret_cast<uint4*>(s_flag)[tid] = make_uint4(0, 0, 0, 0);
        mbar_wait(&s_bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
        __syncthreads();
        // half copy of the window for the compass pre-test (2 positions per
        // HMNMX2 / HSET2 instead of one per float min/max/compare)
        for (int i = tid; i < SH * SWA / 4; i += 256) {
            const float4 f = reinterpret_cast<const float4*>(&px[0][0])[i];
            const __half2 lo = __floats2half2_rn(f.x, f.y), hi = __floats2half2_rn(f.z, f.w);
            reinterpret_cast<uint2*>(&s_hx[0][0])[i] =
                make_uint2(*reinterpret_cast<const unsigned*>(&lo), *reinterpret_cast<const unsigned*>(&hi));
        }
        __syncthreads();

        // A: compass pre-test on 4 adjacent positions per thread from five
        // 8-byte loads of the half copy -> this warp's own queue (no atomics).
        // The test in half precision is a superset of the float test: with the
        // threshold lowered by one it passes whenever the exact test passes
        // (conversions and the add each round by <= 0.125 on [0, 512)), and
        // phase B redoes the exact float segment test.
        // valid columns of this thread's 4 positions: j in [jlo, jhi)
        // (tiles clear of both scan borders -- almost all -- take every
        // position of the 62-wide row: a full mask except the last group)
        unsigned colm = colm_full;
        if (!(ox - 1 >= kDetectBorder && ox - 1 + FWV <= xe)) {
            const int jlo = min(max(kDetectBorder - (ox - 1) - fx0, 0), 4);
            const int jhi = min(max(min(FWV, xe - (ox - 1)) - fx0, 0), 4);
            colm = ((1u << jhi) - 1u) & ~((1u << jlo) - 1u);
        }
        uint16_t* q = s_q + wid * (NF / 8);
        int qn = 0;
        unsigned pm = 0;  // pass bits: 4 positions x 2 rows
        const __half2 thr2 = __float2half2_rn((float)(kThrA - 1));
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int fy = fy0 + 16 * k, gy = oy - 1 + fy;
            if (colm && gy >= kDetectBorder && gy < ye) {
                const int c = fx0 + 4, cy = fy + 3;
                const uint2 Ph = *reinterpret_cast<const uint2*>(&s_hx[cy][c]);
                const uint2 Nh = *reinterpret_cast<const uint2*>(&s_hx[cy - 3][c]);
                const uint2 Sh = *reinterpret_cast<const uint2*>(&s_hx[cy + 3][c]);
                const uint2 Wq = *reinterpret_cast<const uint2*>(&s_hx[cy][c - 4]);
                const uint2 Eq = *reinterpret_cast<const uint2*>(&s_hx[cy][c + 4]);
                // W of position j is column c+j-3, E is c+j+3 (pairs of halves)
                const unsigned wp[2] = {__byte_perm(Wq.x, Wq.y, 0x5432), __byte_perm(Wq.y, Ph.x, 0x5432)};
                const unsigned ep[2] = {__byte_perm(Ph.y, Eq.x, 0x5432), __byte_perm(Eq.x, Eq.y, 0x5432)};
                const unsigned pp[2] = {Ph.x, Ph.y}, np[2] = {Nh.x, Nh.y}, sp[2] = {Sh.x, Sh.y};
                unsigned m[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const __half2 P = *reinterpret_cast<const __half2*>(&pp[j]);
                    const __half2 N = *reinterpret_cast<const __half2*>(&np[j]);
                    const __half2 S = *reinterpret_cast<const __half2*>(&sp[j]);
                    const __half2 E = *reinterpret_cast<const __half2*>(&ep[j]);
                    const __half2 W = *reinterpret_cast<const __half2*>(&wp[j]);
                    const __half2 A = __hmin2(__hmax2(N, S), __hmax2(E, W));
                    const __half2 B = __hmax2(__hmin2(N, S), __hmin2(E, W));
                    m[j] = __hgt2_mask(A, __hadd2(P, thr2)) | __hlt2_mask(B, __hsub2(P, thr2));
                }
                const unsigned pk = (m[0] & 1u) | ((m[0] >> 15) & 2u) | ((m[1] & 1u) << 2) | ((m[1] >> 13) & 8u);
                pm |= (pk & colm) << (4 * k);
            }
        }
        if (__any_sync(0xffffffffu, pm != 0)) {  // append: warp exclusive scan of the per-lane pass counts
            const int c = __popc(pm);
            int incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += t;
            }
            int pos = incl - c;
            const int base = fy0 * FW + fx0;  // bit b -> position base + (b & 3) + (b >> 2) * 16 * FW
            static_assert(16 * FW == 1024, "row-block stride");
            while (pm) {
                const int b = __ffs(pm) - 1;
                pm &= pm - 1;
                q[pos++] = (uint16_t)(base + ((b & 3) | ((b & 4) << 8)));
            }
            qn = __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();

        // B: full segment test + score for this warp's queue; corners flag
        // bit0 = thr 7, bit1 = thr 20 and go to the warp's corner queue
        // the corner queue reuses the warp's compass queue: corners are appended
        // only after every lane read its entry of the current chunk, so the
        // write position never passes the read position
        uint16_t* cq = q;
        int cqn = 0;
        for (int q0 = 0; q0 < qn; q0 += 32) {
            bool corner = false;
            int i = 0;
            if (q0 + lane < qn) {
                i = q[q0 + lane];
                const int cx = (i & 63) + 4, cy = (i >> 6) + 3;
                const float p = px[cy][cx];
                float v[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = px[cy + ring_dy(r)][cx + ring_dx(r)];
                float A, B;
                ring_extrema(v, A, B);
                if (A > fadd(p, (float)kThrA) || B < fsub(p, (float)kThrA)) {
                    float sc = 0.f;
#pragma unroll
                    for (int r = 0; r < 16; ++r) sc = fadd(sc, fabsf(fsub(v[r], p)));
                    s_sc[i] = sc;
                    s_flag[i] = (MODE == 0 || A > fadd(p, (float)kFastThr) || B < fsub(p, (float)kFastThr)) ? 3 : 1;
                    corner = true;
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, corner);
            if (corner) cq[cqn + __popc(m & lt)] = (uint16_t)i;
            cqn += __popc(m);
        }
        __syncthreads();  // every warp's flags are visible to every NMS

        // NMS at this warp's corners in the core region (both sets)
        for (int q0 = 0; q0 < cqn; q0 += 32) {
            uint32_t f = 0;
            int cgx = 0, cgy = 0;
            if (q0 + lane < cqn) {
                const int i = cq[q0 + lane];
                const int fx = i & 63, fy = i >> 6;
                cgx = ox - 1 + fx;
                cgy = oy - 1 + fy;
                if (fx >= 1 && fx <= TW && fy >= 1 && fy <= TH) {
                    const float sv = s_sc[i];
                    bool keep7 = true, keep20 = s_flag[i] == 3;
#pragma unroll
                    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (dx == 0 && dy == 0) continue;
                            const int nb = i + dy * FW + dx;
                            const int fl = s_flag[nb];
                            if (!fl) continue;
                            const float o = s_sc[nb];
                            const bool early = (dy < 0 || (dy == 0 && dx < 0));
                            if (o > sv || (o == sv && early)) {
                                keep7 = false;
                                if (fl == 3) keep20 = false;
                            }
                        }
                    f = (keep20 ? 1u : 0u) | (MODE == 1 && keep7 ? 2u : 0u);
                }
            }
            n20 += (f & 1u) ? 1 : 0;
            n7 += (f & 2u) ? 1 : 0;
            const unsigned m = __ballot_sync(0xffffffffu, f != 0);
            if (m) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&cnt[img].n_cand, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (f) {
                    const int pos = base + __popc(m & lt);
                    if (pos < s_candcap) {
                        Cand c;
                        c.xy = (uint32_t)cgx | ((uint32_t)cgy << 16);
                        c.lf = (uint32_t)L | (f << 8);
                        cand[s_candoff + pos] = c;
                    } else {
                        cnt[img].overflow = 1;
                    }
                }
            }
        }
        __syncthreads();  // buffers and maps are rewritten by the next tile
    }
    n20 = __reduce_add_sync(0xffffffffu, n20);
    n7 = __reduce_add_sync(0xffffffffu, n7);
    if (lane == 0) {
        if (MODE == 0 && n20) atomicAdd(&cnt[img].n20, n20);
        if (MODE == 1 && n7) atomicAdd(&cnt[img].n7, n7);
    }
}

// MODE 0: one CTA per FAST tile row. MODE 1 (auto-relax): a grid-stride loop,
// so the rows of the images that do not need the pass cost one table read each
// instead of a CTA launch each.
template <int MODE>
__global__ void __launch_bounds__(256, 5) k_fast_nms(const OrbImage* __restrict__ imgs,
                                                     const LevelSeg* __restrict__ segs, int nsegs,
                                                     int nblk, const TileRange* __restrict__ rng,
                                                     const float* __restrict__ pyr,
                                                     const char* __restrict__ maps,
                                                     Cand* __restrict__ cand,
                                                     ImgCounters* __restrict__ cnt, int nimg) {
    __shared__ __align__(8) uint64_t s_bar[2];  // one mbarrier per staging buffer
    if (MODE == 1) {
        // nothing to do unless some image kept fewer than max_points / 4
        // threshold-20 corners (the usual case): one pass over the counters
        __shared__ int s_any;
        if (threadIdx.x == 0) s_any = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < nimg; i += blockDim.x)
            if (cnt[i].n20 < imgs[i].max_points / 4) s_any = 1;
        __syncthreads();
        if (!s_any) return;
    }
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    unsigned phase = 0;  // bit b: parity of buffer b's next completion
    if (MODE == 0) {
        fast_nms_row<0>(blockIdx.x, imgs, segs, nsegs, rng, pyr, maps, cand, cnt, s_bar, phase);
        return;
    }
    for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        fast_nms_row<1>(b, imgs, segs, nsegs, rng, pyr, maps, cand, cnt, s_bar, phase);
        __syncthreads();  // shared buffers are reused by the next row
    }
}

// ------------------------------------------------------------------ measures

// harris_response (orb.cpp:82-104) in the reference's order and rounding.
// Candidates lie >= 17 px inside their level (orb.cpp:149-151), so the 9x9
// support never needs the clamp; rows slide through three 9-wide register
// arrays (81 loads instead of 392).
__device__ float harris_at(const float* __restrict__ lv, int w, int x, int y) {
    const float* p = lv + (size_t)(y - 4) * w + (x - 4);
    float r0[9], r1[9], r2[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        r0[j] = __ldg(p + j);
        r1[j] = __ldg(p + w + j);
    }
    p += 2 * (size_t)w;
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
    for (int dy = -3; dy <= 3; ++dy) {
#pragma unroll
        for (int j = 0; j < 9; ++j) r2[j] = __ldg(p + j);
        p += w;
#pragma unroll
        for (int j = 1; j <= 7; ++j) {
            const float gx = fadd(fadd(fsub(r0[j + 1], r0[j - 1]), fmul(2.f, fsub(r1[j + 1], r1[j - 1]))),
                                  fsub(r2[j + 1], r2[j - 1]));
            const float gy = fadd(fadd(fsub(r2[j - 1], r0[j - 1]), fmul(2.f, fsub(r2[j], r0[j]))),
                                  fsub(r2[j + 1], r0[j + 1]));
            const double ix = gx, iy = gy;
            a = dadd(a, dmul(ix, ix));
            b = dadd(b, dmul(iy, iy));
            c = dadd(c, dmul(ix, iy));
        }
#pragma unroll
        for (int j = 0; j < 9; ++j) {
            r0[j] = r1[j];
            r1[j] = r2[j];
        }
    }
    const double sc = 1.0 / (255.0 * 4 * 7);
    const double sc2 = dmul(sc, sc);
    a = dmul(a, sc2);
    b = dmul(b, sc2);
    c = dmul(c, sc2);
    const double ab = dadd(a, b);
    return (float)dsub(dsub(dmul(a, b), dmul(c, c)), dmul(dmul(0.04, ab), ab));
}

// Order-preserving map of the response to a key where ascending key means
// descending response; -0 is folded into +0 because the reference comparator
// (orb.cpp:204) treats them as equal.
__device__ __forceinline__ uint32_t resp_key(float r) {
    if (r == 0.f) r = 0.f;
    uint32_t u = __float_as_uint(r);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ~u;
}

__global__ void __launch_bounds__(128) k_measures(const OrbImage* __restrict__ imgs,
                                                  const float* __restrict__ pyr,
                                                  const Cand* __restrict__ cand,
                                                  const ImgCounters* __restrict__ cnt,
                                                  CandKey* __restrict__ keys,
                                                  xa_kp* __restrict__ kps) {
    const int img = blockIdx.y;
    const OrbImage& im = imgs[img];
    const int n = min(cnt[img].n_cand, im.cand_cap);
    // auto-relax (orb.cpp:187-188): thr-20 survivors < max_points/4 -> thr 7 set
    const uint32_t bit = (cnt[img].n20 < im.max_points / 4) ? 2u : 1u;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const Cand c = cand[im.cand_off + i];
        CandKey k;
        if (!((c.lf >> 8) & bit)) {
            k.k0 = k.k1 = k.k2 = k.idx = 0xFFFFFFFFu;
            keys[im.cand_off + i] = k;
            continue;
        }
        const int x = c.xy & 0xFFFF, y = c.xy >> 16, L = c.lf & 0xFF;
        const float* lv = pyr + im.poff[L];
        xa_kp kp;
        const float ls = c_level_scale[L];
        kp.x = fmul((float)x, ls);
        kp.y = fmul((float)y, ls);
        kp.octave_scale = ls;
        kp.response = harris_at(lv, im.pitch[L], x, y);
        kp.orientation = 0.f;  // computed for the selected top-N only (k_select)
        kps[im.cand_off + i] = kp;
        k.k0 = resp_key(kp.response);
        k.k1 = __float_as_uint(kp.y);
        k.k2 = __float_as_uint(kp.x);
        k.idx = (uint32_t)i;
        keys[im.cand_off + i] = k;
    }
}

// ------------------------------------------------------------------ select

__device__ __forceinline__ bool key_less(const CandKey& a, const CandKey& b) {
    if (a.k0 != b.k0) return a.k0 < b.k0;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    if (a.k2 != b.k2) return a.k2 < b.k2;
    return a.idx < b.idx;
}

// Block-wide exclusive scan of one int per thread (1024 threads).
__device__ int block_excl_scan(int v, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        s_warp[lane] = s;
    }
    __syncthreads();
    const int excl = x - v + (wid ? s_warp[wid - 1] : 0);
    *total = s_warp[31];
    __syncthreads();
    return excl;
}

// describe_binary's per-keypoint checks (orb.cpp:219-228) and, for views,
// filter_to_content (pipeline.cpp:28-40). Returns true if kept.
// glibc cosf/sinf of the keypoint angle: correctly rounded values plus the
// fixups where glibc differs in a way that moves a pattern coordinate
// (tools/gen_trig_table.c).
__device__ __forceinline__ void glibc_cossin(float th, float& c, float& s) {
    c = (float)cos((double)th);
    s = (float)sin((double)th);
    if (!(fabsf(th) <= XA_TRIG_RANGE)) return;
    const uint32_t key = __float_as_uint(th);
    int lo = 0, hi = XA_TRIG_FIXUPS - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const uint32_t k = c_trig[mid].x;
        if (k == key) {
            c = __uint_as_float(c_trig[mid].c);
            s = __uint_as_float(c_trig[mid].s);
            return;
        }
        if (k < key) lo = mid + 1; else hi = mid - 1;
    }
}

__device__ __forceinline__ bool describe_ok(const OrbImage& im, const xa_kp& kp, bool content,
                                            DescKp& d, bool trig) {
    if (content) {
        double sx, sy;
        map_pt(im.back, (double)kp.x, (double)kp.y, sx, sy);
        const double xmax = dsub((double)(im.src_w - 1), im.margin);
        const double ymax = dsub((double)(im.src_h - 1), im.margin);
        if (!(sx >= im.margin && sx <= xmax && sy >= im.margin && sy <= ymax)) return false;
    }
    const int L = (int)round((double)logf(kp.octave_scale) / c_log_ratio);
    if (L < 0 || L >= im.nlev) return false;
    const int lx = (int)roundf(__fdiv_rn(kp.x, kp.octave_scale));
    const int ly = (int)roundf(__fdiv_rn(kp.y, kp.octave_scale));
    if (lx < kDescribeBorder || ly < kDescribeBorder || lx >= im.w[L] - kDescribeBorder ||
        ly >= im.h[L] - kDescribeBorder)
        return false;
    d.lx = lx;
    d.ly = ly;
    d.level = L;
    d.orientation = kp.orientation;
    d.cs = d.sn = 0.f;
    if (trig) glibc_cossin(kp.orientation, d.cs, d.sn);
    return true;
}

// Order-preserving compaction of det[0..n) into the describe list (4 items per
// thread, 1024 threads). Appends after *io_count.
// trig: also fill the descriptor's cos/sin (the coarse path leaves them to
// k_orient, which computes the orientation after the selection).
__device__ void compact_describe(const OrbImage& im, const xa_kp* det, int n, bool content,
                                 DescKp* desc_in, xa_kp* desc_kp, int* s_warp, int* io_count,
                                 int* det_map, bool trig) {
    for (int base = 0; base < n; base += 4096) {
        const int i0 = base + threadIdx.x * 4;
        bool keep[4];
        DescKp d[4];
        int c = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            keep[k] = (i0 + k < n) && describe_ok(im, det[i0 + k], content, d[k], trig);
            c += keep[k];
        }
        int total;
        int pos = *io_count + block_excl_scan(c, s_warp, &total);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (det_map && i0 + k < n) det_map[im.kp_off + i0 + k] = keep[k] ? pos : -1;
            if (keep[k]) {
                desc_in[im.kp_off + pos] = d[k];
                desc_kp[im.kp_off + pos] = det[i0 + k];
                ++pos;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) *io_count += total;
        __syncthreads();
    }
}

// One CTA per image: top-N select + sort (orb.cpp:203-208), then the describe
// list. Dynamic smem: kSortCap CandKey entries.
// Warp 0 of the CTA: the bin of a histogram (nbins = 1024 or 2048) holding
// the target-th entry (1-based) in ascending bin order, and the rank of that
// entry within its bin. Callers synchronise before and after.
__device__ __forceinline__ void select_bin(const int* hist, int nbins, int target, int* s_bin,
                                           int* s_rank) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x, per = nbins >> 5;
    int sum = 0;
    for (int j = 0; j < per; ++j) sum += hist[per * lane + j];
    int incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, incl >= target);
    if (lane == __ffs(hit) - 1) {
        int acc = incl - sum, d = per * lane;
        for (; d < per * lane + per - 1; ++d) {
            if (acc + hist[d] >= target) break;
            acc += hist[d];
        }
        *s_bin = d;
        *s_rank = target - acc;
    }
}

// ---- top-N selection, split over the whole GPU: per image the N-th key sits
// in bin `lo` of an 11-bit histogram of the keys' top bits; keys of lower bins
// are kept outright, keys of bin lo are listed and radix-selected on their low
// 21 bits by k_select, which then sorts the ~N survivors. The histogram and the
// split run with many CTAs per image (the single-CTA version spent ~0.1 ms
// walking the largest images' keys).
constexpr int kSelChunk = 4096;  // keys per k_sel_hist / k_sel_split CTA

__global__ void __launch_bounds__(256) k_sel_hist(const OrbImage* __restrict__ imgs,
                                                  const CandKey* __restrict__ keys,
                                                  const ImgCounters* __restrict__ cnt,
                                                  SelState* __restrict__ sel) {
    __shared__ int h[2048];
    __shared__ int s_v;
    const int img = blockIdx.y;
    const OrbImage& im = imgs[img];
    const int M = min(cnt[img].n_cand, im.cand_cap);
    const int base = blockIdx.x * kSelChunk;
    if (base >= M) return;
    for (int i = threadIdx.x; i < 2048; i += 256) h[i] = 0;
    if (threadIdx.x == 0) s_v = 0;
    __syncthreads();
    const CandKey* K = keys + im.cand_off;
    int v = 0;
    for (int i = base + threadIdx.x; i < min(base + kSelChunk, M); i += 256) {
        const CandKey k = K[i];
        if (k.idx != 0xFFFFFFFFu) {
            ++v;
            atomicAdd(&h[k.k0 >> 21], 1);
        }
    }
    v = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_v, v);
    __syncthreads();
    for (int b = threadIdx.x; b < 2048; b += 256)
        if (h[b]) atomicAdd(&sel[img].hist[b], h[b]);
    if (threadIdx.x == 0 && s_v) atomicAdd(&sel[img].valid, s_v);
}

// One warp per image: the bin holding the N-th key (or take-all).
__global__ void k_sel_bin(const OrbImage* __restrict__ imgs, SelState* __restrict__ sel) {
    SelState& S = sel[blockIdx.x];
    const int N = imgs[blockIdx.x].max_points;
    if (S.valid <= N) {
        if (threadIdx.x == 0) {
            S.lo = 2048;
            S.need = 0;
        }
        return;
    }
    select_bin(S.hist, 2048, N, &S.lo, &S.need);
}

__global__ void __launch_bounds__(256) k_sel_split(const OrbImage* __restrict__ imgs,
                                                   const CandKey* __restrict__ keys,
                                                   const ImgCounters* __restrict__ cnt,
                                                   SelState* __restrict__ sel,
                                                   CandKey* __restrict__ sel_list,
                                                   uint2* __restrict__ bnd_list) {
    const int img = blockIdx.y;
    const OrbImage& im = imgs[img];
    const int M = min(cnt[img].n_cand, im.cand_cap);
    const int base = blockIdx.x * kSelChunk;
    if (base >= M) return;
    SelState& S = sel[img];
    const uint32_t lo = (uint32_t)S.lo;
    const CandKey* K = keys + im.cand_off;
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    for (int w0 = base + (threadIdx.x & ~31); w0 < min(base + kSelChunk, M); w0 += 256) {
        const int i = w0 + lane;
        CandKey k;
        k.idx = 0xFFFFFFFFu;
        if (i < M) k = K[i];
        const bool ok = k.idx != 0xFFFFFFFFu;
        const uint32_t bin = k.k0 >> 21;
        const bool take = ok && bin < lo, list = ok && bin == lo;
        const unsigned mt = __ballot_sync(0xffffffffu, take), ml = __ballot_sync(0xffffffffu, list);
        int bt = 0, bl = 0;
        if (lane == 0) {
            if (mt) bt = atomicAdd(&S.nsel, __popc(mt));
            if (ml) bl = atomicAdd(&S.nbnd, __popc(ml));
        }
        bt = __shfl_sync(0xffffffffu, bt, 0);
        bl = __shfl_sync(0xffffffffu, bl, 0);
        if (take) {
            const int p = bt + __popc(mt & lt);
            if (p < kSortCap) sel_list[(size_t)img * kSortCap + p] = k;
        } else if (list) {
            const int q = bl + __popc(ml & lt);
            if (q < kListCap) bnd_list[(size_t)img * kListCap + q] = make_uint2(k.k0, (uint32_t)i);
        }
    }
}

__global__ void __launch_bounds__(1024) k_select(const OrbImage* __restrict__ imgs,
                                                 const CandKey* __restrict__ keys,
                                                 const xa_kp* __restrict__ kps,
                                                 const Cand* __restrict__ cand,
                                                 Cand* __restrict__ det_cand,
                                                 int* __restrict__ det_map,
                                                 ImgCounters* __restrict__ cnt,
                                                 xa_kp* __restrict__ det_out,
                                                 DescKp* __restrict__ desc_in,
                                                 xa_kp* __restrict__ desc_kp,
                                                 SelState* __restrict__ sel,
                                                 const CandKey* __restrict__ sel_list,
                                                 const uint2* __restrict__ bnd_list) {
    // dynamic smem: kSortCap sort entries, then kListCap (k0, index) pairs of
    // the boundary bin
    extern __shared__ CandKey s_buf[];
    uint2* s_list = reinterpret_cast<uint2*>(s_buf + kSortCap);
    __shared__ int s_hist[2048];
    __shared__ int s_warp[32];
    __shared__ int s_n, s_sel, s_rem, s_count;
    const int img = blockIdx.x;
    const OrbImage& im = imgs[img];
    const int tid = threadIdx.x, lane = tid & 31;
    const int M = min(cnt[img].n_cand, im.cand_cap);
    const CandKey* K = keys + im.cand_off;
    SelState& S = sel[img];
    const uint32_t lo = (uint32_t)S.lo;
    const int G0 = min(S.nsel, kSortCap), ln = S.nbnd;
    if (tid == 0) s_n = S.nsel;
    for (int i = tid; i < G0; i += 1024) s_buf[i] = sel_list[(size_t)img * kSortCap + i];
    const bool listed = ln <= kListCap;
    if (lo < 2048u && listed)
        for (int q = tid; q < ln; q += 1024) s_list[q] = bnd_list[(size_t)img * kListCap + q];
    __syncthreads();
    if (lo < 2048u) {
        // radix-select the need-th smallest key of bin lo (bits 20..10, 9..0);
        // the list lives in shared memory unless the bin overflowed it, in
        // which case the image's keys are walked again (batched loads)
        constexpr int kU = 8;
        auto for_bin = [&](auto&& f) {
            if (listed) {
                for (int q = tid; q < ln; q += 1024) f(s_list[q].x, (int)s_list[q].y);
            } else {
                for (int w0 = tid & ~31; w0 < M; w0 += 1024 * kU) {
                    const int i0 = w0 + lane;
                    CandKey kb[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        kb[u].idx = 0xFFFFFFFFu;
                        if (i0 + u * 1024 < M) kb[u] = K[i0 + u * 1024];
                    }
#pragma unroll
                    for (int u = 0; u < kU; ++u)
                        if (kb[u].idx != 0xFFFFFFFFu && (kb[u].k0 >> 21) == lo) f(kb[u].k0, i0 + u * 1024);
                }
            }
        };
        uint32_t prefix = lo << 21;
        int rem = S.need;
        for (int pass = 0; pass < 2; ++pass) {
            const int shift = pass == 0 ? 10 : 0, nb = pass == 0 ? 2048 : 1024;
            const uint32_t hi_mask = pass == 0 ? 0xFFE00000u : 0xFFFFFC00u;
            for (int i = tid; i < nb; i += 1024) s_hist[i] = 0;
            __syncthreads();
            for_bin([&](uint32_t k0, int) {
                if ((k0 & hi_mask) == prefix) atomicAdd(&s_hist[(k0 >> shift) & (nb - 1)], 1);
            });
            __syncthreads();
            select_bin(s_hist, nb, rem, &s_sel, &s_rem);
            __syncthreads();
            prefix |= (uint32_t)s_sel << shift;
            rem = s_rem;
            __syncthreads();
        }
        const uint32_t thr = prefix;  // keys of bin lo with k0 <= thr join the sort
        for_bin([&](uint32_t k0, int i) {
            if (k0 <= thr) {
                const int p = atomicAdd(&s_n, 1);
                if (p < kSortCap) s_buf[p] = K[i];
            }
        });
        __syncthreads();
    }
    const int G = s_n;
    if (G > kSortCap) {  // large max_points or massive response ties: k_select_big
        if (tid == 0) {
            S.big = 1;
            cnt[img].n_det = 0;
            cnt[img].n_desc = 0;
        }
        return;
    }
    int P = 1;
    while (P < G) P <<= 1;
    for (int i = G + tid; i < P; i += 1024) {
        CandKey k;
        k.k0 = k.k1 = k.k2 = k.idx = 0xFFFFFFFFu;
        s_buf[i] = k;
    }
    __syncthreads();
    // bitonic sort ascending on (k0, k1, k2, idx)
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P / 2; i += 1024) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                CandKey a = s_buf[lo], b = s_buf[hi];
                if (key_less(b, a) == up) {
                    s_buf[lo] = b;
                    s_buf[hi] = a;
                }
            }
            __syncthreads();
        }
    const int nd = min(G, im.max_points);
    xa_kp* det = det_out + im.kp_off;
    // the orientation is filled in by k_orient for these nd keypoints only
    for (int i = tid; i < nd; i += 1024) {
        const uint32_t ci = s_buf[i].idx;
        det[i] = kps[im.cand_off + ci];
        det_cand[im.kp_off + i] = cand[im.cand_off + ci];
    }
    if (tid == 0) {
        cnt[img].n_det = nd;
        s_count = 0;
    }
    __threadfence_block();
    __syncthreads();
    compact_describe(im, det, nd, im.filter != 0, desc_in, desc_kp, s_warp, &s_count, det_map, false);
    if (tid == 0) cnt[img].n_desc = s_count;
}

// Top-N for the images whose selection does not fit k_select's shared-memory
// sort (max_points above kSortCap, or more than kSortCap keys tied at the N-th
// response): every valid key of the image is gathered into a global scratch
// buffer and bitonic-sorted there by one CTA on the same unique 128-bit key,
// so the kept set and its order equal the reference's full sort + truncate
// (orb.cpp:203-208). One CTA walks the flagged images in turn (the launch is
// part of every chain; without flagged images it costs a table scan).
__global__ void __launch_bounds__(1024) k_select_big(const OrbImage* __restrict__ imgs, int nimg,
                                                     const CandKey* __restrict__ keys,
                                                     const xa_kp* __restrict__ kps,
                                                     const Cand* __restrict__ cand,
                                                     Cand* __restrict__ det_cand, int* __restrict__ det_map,
                                                     ImgCounters* __restrict__ cnt,
                                                     xa_kp* __restrict__ det_out,
                                                     DescKp* __restrict__ desc_in,
                                                     xa_kp* __restrict__ desc_kp,
                                                     const SelState* __restrict__ sel,
                                                     CandKey* __restrict__ buf, int cap) {
    __shared__ int s_warp[32];
    __shared__ int s_n, s_count;
    __shared__ int s_nbig, s_big[1024];
    const int tid = threadIdx.x;
    // the images whose selection exceeded the shared-memory sort (rare): one
    // block-wide pass over the flags instead of a serial scan of every image
    for (int ib = 0; ib < nimg; ib += 1024) {
    if (tid == 0) s_nbig = 0;
    __syncthreads();
    if (ib + tid < nimg && sel[ib + tid].big) s_big[atomicAdd(&s_nbig, 1)] = ib + tid;
    __syncthreads();
    const int nbig = s_nbig;
    for (int bi = 0; bi < nbig; ++bi) {
        const int img = s_big[bi];
        const OrbImage& im = imgs[img];
        const int M = min(cnt[img].n_cand, im.cand_cap);
        const CandKey* K = keys + im.cand_off;
        if (tid == 0) s_n = 0;
        __syncthreads();
        for (int i = tid; i < M; i += 1024) {
            const CandKey k = K[i];
            if (k.idx != 0xFFFFFFFFu) {
                const int p = atomicAdd(&s_n, 1);
                if (p < cap) buf[p] = k;
            }
        }
        __syncthreads();
        const int G = s_n;
        if (G > cap) {
            if (tid == 0) cnt[img].overflow = 2;
            __syncthreads();
            continue;
        }
        int P = 1;
        while (P < G) P <<= 1;
        for (int i = G + tid; i < P; i += 1024) {
            CandKey k;
            k.k0 = k.k1 = k.k2 = k.idx = 0xFFFFFFFFu;
            buf[i] = k;
        }
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = tid; i < P / 2; i += 1024) {
                    const int a = 2 * i - (i & (stride - 1)), b = a + stride;
                    const bool up = (a & size) == 0;
                    const CandKey ka = buf[a], kb = buf[b];
                    if (key_less(kb, ka) == up) {
                        buf[a] = kb;
                        buf[b] = ka;
                    }
                }
                __syncthreads();
            }
        const int nd = min(G, im.max_points);
        xa_kp* det = det_out + im.kp_off;
        for (int i = tid; i < nd; i += 1024) {
            const uint32_t ci = buf[i].idx;
            det[i] = kps[im.cand_off + ci];
            det_cand[im.kp_off + i] = cand[im.cand_off + ci];
        }
        if (tid == 0) {
            cnt[img].n_det = nd;
            s_count = 0;
        }
        __threadfence_block();
        __syncthreads();
        compact_describe(im, det, nd, im.filter != 0, desc_in, desc_kp, s_warp, &s_count, det_map, false);
        if (tid == 0) cnt[img].n_desc = s_count;
        __syncthreads();
    }
    __syncthreads();  // s_big is rewritten by the next block of images
    }
}

// Intensity-centroid orientation (orb.cpp:106-123) for the selected top-N
// only: it is a pure function of the level pixels, so computing it after the
// cap gives the reference's values while skipping the ~95% of candidates the
// cap drops. Thread per keypoint, reference summation order.
// Intensity-centroid orientation (centroid_orientation, orb.cpp:106-123) of
// the kept keypoints, in the reference's summation order (serial double sums
// per keypoint: row 0, then the row pairs v = 1..15). A one-warp CTA owns 32
// keypoints, one per lane. Row step v+1's segments of all 32 keypoints are
// copied to shared memory with cp.async (one coalesced warp copy per keypoint
// row) while the lanes sum step v from shared memory, instead of 31
// scattered, latency-bound global loads per row and lane.
// Row v of the 32 keypoints' discs (up and down), each keypoint's segment
// fetched by the whole warp (coalesced); the keypoints' centre pointers and
// pitches come from shared memory (broadcast loads, no shuffles).
__device__ __forceinline__ void orient_fetch(float (*su)[33], float (*sd)[33], const long long* s_p0,
                                             const int* s_pitch, int nk, int v) {
    const int lane = threadIdx.x & 31;
    const int d = v == 0 ? kOrientR : c_umax[v];
    const bool on = lane <= 2 * d;
    for (int k = 0; k < nk; ++k) {
        const float* pk = reinterpret_cast<const float*>(s_p0[k]) + (lane - d);
        const int off = v * s_pitch[k];
        if (on) {
            cp_async4(&su[k][lane], pk + off);
            if (v) cp_async4(&sd[k][lane], pk - off);
        }
    }
    cp_async_commit();
}

__global__ void __launch_bounds__(32) k_orient(const OrbImage* __restrict__ imgs,
                                               const float* __restrict__ pyr,
                                               const ImgCounters* __restrict__ cnt,
                                               const Cand* __restrict__ det_cand,
                                               const int* __restrict__ det_map,
                                               xa_kp* __restrict__ det_out,
                                               DescKp* __restrict__ desc_in,
                                               xa_kp* __restrict__ desc_kp) {
    __shared__ float s_rows[2][2][32][33];  // [buffer][up/down][keypoint][column]
    const int img = blockIdx.y;
    const OrbImage& im = imgs[img];
    const int n = cnt[img].n_det;
    const int lane = threadIdx.x;
    const int base = blockIdx.x * 32;
    if (base >= n) return;
    const int i = base + lane, nk = min(32, n - base);
    const bool act = i < n;
    long long p0 = 0;  // level pointer of the lane's keypoint centre
    int pitch = 0;
    if (act) {
        const Cand c = det_cand[im.kp_off + i];
        const int L = c.lf & 0xFF;
        pitch = im.pitch[L];
        p0 = (long long)(pyr + im.poff[L] + (size_t)(c.xy >> 16) * pitch + (c.xy & 0xFFFF));
    }
    double m01 = 0.0, m10 = 0.0;
    __shared__ long long s_p0[32];
    __shared__ int s_pitch[32];
    s_p0[lane] = p0;
    s_pitch[lane] = pitch;
    __syncwarp();
    orient_fetch(s_rows[0][0], s_rows[0][1], s_p0, s_pitch, nk, 0);
    for (int v = 0; v <= kOrientR; ++v) {
        if (v < kOrientR) {
            orient_fetch(s_rows[(v + 1) & 1][0], s_rows[(v + 1) & 1][1], s_p0, s_pitch, nk, v + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        if (act) {
            const float* ru = s_rows[v & 1][0][lane];
            if (v == 0) {
                for (int u = -kOrientR; u <= kOrientR; ++u)
                    m10 = dadd(m10, (double)fmul((float)u, ru[u + kOrientR]));
            } else {
                const int d = c_umax[v];
                const float* rd = s_rows[v & 1][1][lane];
                double vs = 0.0;
                for (int u = -d; u <= d; ++u) {
                    const double up = ru[u + d], dn = rd[u + d];
                    vs = dadd(vs, dsub(up, dn));
                    m10 = dadd(m10, dmul((double)u, dadd(up, dn)));
                }
                m01 = dadd(m01, dmul((double)v, vs));
            }
        }
        __syncwarp();  // buffer v & 1 is refilled by the next iteration's fetch
    }
    if (act) {
        const float th = (float)atan2(m01, m10);
        det_out[im.kp_off + i].orientation = th;
        const int m = det_map[im.kp_off + i];
        if (m >= 0) {
            DescKp& dk = desc_in[im.kp_off + m];
            dk.orientation = th;
            glibc_cossin(th, dk.cs, dk.sn);
            desc_kp[im.kp_off + m].orientation = th;
        }
    }
}

// describe_binary entry with caller keypoints (one image, one CTA).
__global__ void __launch_bounds__(1024) k_describe_prep(const OrbImage* __restrict__ imgs,
                                                        const xa_kp* __restrict__ in, int n,
                                                        ImgCounters* __restrict__ cnt,
                                                        DescKp* __restrict__ desc_in,
                                                        xa_kp* __restrict__ desc_kp) {
    __shared__ int s_warp[32];
    __shared__ int s_count;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    compact_describe(imgs[0], in, n, false, desc_in, desc_kp, s_warp, &s_count, nullptr, true);
    if (threadIdx.x == 0) cnt[0].n_desc = s_count;
}

// ------------------------------------------------------------------ describe

// Window of keypoint d (clamp-to-edge, the blur's at_clamped, image.cpp:35,44)
// copied to shared memory with cp.async.
__device__ __forceinline__ void describe_fetch(const OrbImage& im, const float* __restrict__ pyr,
                                               const DescKp& d, float* win) {
    const int w = im.w[d.level], h = im.h[d.level], pitch = im.pitch[d.level];
    const float* lv = pyr + im.poff[d.level];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int x0 = d.lx - HALF, y0 = d.ly - HALF;
    if (x0 >= 0 && y0 >= 0 && x0 + WIN <= w && y0 + WIN <= h) {  // interior: no clamps
        const float* p = lv + (size_t)y0 * pitch + x0;
        for (int r = wid; r < WIN; r += DESC_WARPS) {
            cp_async4(win + r * WS + lane, p + (size_t)r * pitch + lane);
            if (lane < WIN - 32) cp_async4(win + r * WS + 32 + lane, p + (size_t)r * pitch + 32 + lane);
        }
    } else {
        const int gx0 = clampi(x0 + lane, 0, w - 1), gx1 = clampi(x0 + 32 + lane, 0, w - 1);
        for (int r = wid; r < WIN; r += DESC_WARPS) {
            const float* row = lv + (size_t)clampi(y0 + r, 0, h - 1) * pitch;
            cp_async4(win + r * WS + lane, row + gx0);
            if (lane < WIN - 32) cp_async4(win + r * WS + 32 + lane, row + gx1);
        }
    }
    cp_async_commit();
}

__global__ void __launch_bounds__(32 * DESC_WARPS) k_describe(const OrbImage* __restrict__ imgs,
                                                              const float* __restrict__ pyr,
                                                              const ImgCounters* __restrict__ cnt,
                                                              const DescKp* __restrict__ desc_in,
                                                              uint64_t* __restrict__ desc) {
    // One CTA (4 warps) per keypoint at a time, the next keypoint's 49x49
    // window prefetched with cp.async: H pass (49x37, 4 adjacent outputs per
    // task from four 16-byte loads) -> V pass (37x37, 4 stacked outputs per
    // task) -> warp w produces descriptor word w (bits 64w..64w+63) with two
    // ballots. Both passes keep the reference's tap order and rounding.
    extern __shared__ __align__(16) float s_mem[];
    __shared__ int8_t s_pat[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_pat[i] = g_pattern[i];
    const int img = blockIdx.y;
    const OrbImage& im = imgs[img];
    const int n = cnt[img].n_desc;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NT = 32 * DESC_WARPS;
    float* tmp = s_mem + 2 * WIN * WS;
    int k = blockIdx.x;
    if (k >= n) return;
    DescKp d = desc_in[im.kp_off + k];
    describe_fetch(im, pyr, d, s_mem);
    for (int it = 0; k < n; k += gridDim.x, ++it) {
        float* win = s_mem + (it & 1) * WIN * WS;
        const int kn = k + gridDim.x;
        DescKp dn;
        if (kn < n) {
            dn = desc_in[im.kp_off + kn];
            describe_fetch(im, pyr, dn, s_mem + ((it + 1) & 1) * WIN * WS);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        // horizontal pass on all 49 rows, 37 centre columns (image.cpp:31-38)
        for (int task = tid; task < WIN * 10; task += NT) {
            const int r = task / 10, c0 = 4 * (task - r * 10);
            const float4* src = reinterpret_cast<const float4*>(win + r * WS + c0);
            float v[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 t4 = src[q];
                v[4 * q] = t4.x;
                v[4 * q + 1] = t4.y;
                v[4 * q + 2] = t4.z;
                v[4 * q + 3] = t4.w;
            }
            float o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                // 0.f + p == p bit for bit: the taps are positive and the pixels
                // non-negative, so the first product is never -0.f
                float acc = fmul(c_blur2[0], v[j]);
#pragma unroll
                for (int t = 1; t < 13; ++t) acc = fadd(acc, fmul(c_blur2[t], v[j + t]));
                o[j] = acc;
            }
            *reinterpret_cast<float4*>(tmp + r * TS + c0) = make_float4(o[0], o[1], o[2], o[3]);
        }
        __syncthreads();
        // vertical pass -> 37x37 blurred patch (image.cpp:40-47), into the
        // current window buffer (the next window goes to the other one)
        float* bl = win;
        for (int task = tid; task < PAT * 10; task += NT) {
            const int g = task / PAT, c = task - g * PAT, r0 = 4 * g;
            const float* src = tmp + r0 * TS + c;
            float v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = src[q * TS];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                // 0.f + p == p bit for bit: the taps are positive and the pixels
                // non-negative, so the first product is never -0.f
                float acc = fmul(c_blur2[0], v[j]);
#pragma unroll
                for (int t = 1; t < 13; ++t) acc = fadd(acc, fmul(c_blur2[t], v[j + t]));
                if (r0 + j < PAT) bl[(r0 + j) * PAT + c] = acc;
            }
        }
        __syncthreads();
        const float cs = d.cs, sn = d.sn;
        uint32_t words[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int j = 64 * wid + 32 * q + lane;
            const float px1 = s_pat[4 * j], py1 = s_pat[4 * j + 1];
            const float px2 = s_pat[4 * j + 2], py2 = s_pat[4 * j + 3];
            const int x1 = (int)roundf(fsub(fmul(cs, px1), fmul(sn, py1)));
            const int y1 = (int)roundf(fadd(fmul(sn, px1), fmul(cs, py1)));
            const int x2 = (int)roundf(fsub(fmul(cs, px2), fmul(sn, py2)));
            const int y2 = (int)roundf(fadd(fmul(sn, px2), fmul(cs, py2)));
            const float v1 = bl[(y1 + PHALF) * PAT + x1 + PHALF];
            const float v2 = bl[(y2 + PHALF) * PAT + x2 + PHALF];
            words[q] = __ballot_sync(0xffffffffu, v1 < v2);
        }
        if (lane == 0) desc[(im.kp_off + k) * 4 + wid] = (uint64_t)words[0] | ((uint64_t)words[1] << 32);
        __syncthreads();  // bl (= this window buffer) is refilled two keypoints on
        d = dn;
    }
}

// ------------------------------------------------------------------ launchers

int launch_pyramid(const OrbImage* d_imgs, const LevelSeg* d_segs, int nsegs, int total_blocks,
                   float* pyr, cudaStream_t st, bool zero) {
    if (total_blocks <= 0) return 0;
    if (zero)
        k_pyramid<true><<<total_blocks, 256, 0, st>>>(d_imgs, d_segs, nsegs, pyr);
    else
        k_pyramid<false><<<total_blocks, 256, 0, st>>>(d_imgs, d_segs, nsegs, pyr);
    return 1;
}

constexpr int kRelaxCtas = 148 * 5;  // one resident wave of the auto-relax pass

int launch_fast_nms(const OrbImage* d_imgs, const LevelSeg* d_segs, int nsegs, int total_blocks,
                    const TileRange* d_rng, const float* pyr, const void* maps, Cand* cand,
                    ImgCounters* cnt, cudaStream_t st, int nimg) {
    if (total_blocks <= 0) return 0;
    const char* m = static_cast<const char*>(maps);
    k_fast_nms<0><<<total_blocks, 256, 0, st>>>(d_imgs, d_segs, nsegs, total_blocks, d_rng, pyr, m,
                                                cand, cnt, nimg);
    // auto-relax pass; rows of images that kept enough threshold-20 corners are skipped
    k_fast_nms<1><<<std::min(total_blocks, kRelaxCtas), 256, 0, st>>>(d_imgs, d_segs, nsegs,
                                                                     total_blocks, d_rng, pyr, m, cand, cnt,
                                                                     nimg);
    return 2;
}

int launch_measures(const OrbImage* d_imgs, int nimg, const float* pyr, const Cand* cand,
                    const ImgCounters* cnt, CandKey* keys, xa_kp* kps, cudaStream_t st) {
    if (nimg <= 0) return 0;
    dim3 grid(64, nimg);
    k_measures<<<grid, 128, 0, st>>>(d_imgs, pyr, cand, cnt, keys, kps);
    return 1;
}

int launch_select(const OrbImage* d_imgs, int nimg, int max_points, const CandKey* keys,
                  const xa_kp* kps, const Cand* cand, const float* pyr, Cand* det_cand,
                  int* det_map, ImgCounters* cnt, xa_kp* det_out, DescKp* desc_in,
                  xa_kp* desc_kp_out, int max_cand, SelState* sel, CandKey* sel_list,
                  uint2* bnd_list, CandKey* big_scratch, int big_cap, cudaStream_t st) {
    if (nimg <= 0) return 0;
    // sel must be zeroed by the caller before (histograms and list counters)
    const dim3 gsel((max_cand + kSelChunk - 1) / kSelChunk, nimg);
    k_sel_hist<<<gsel, 256, 0, st>>>(d_imgs, keys, cnt, sel);
    k_sel_bin<<<nimg, 32, 0, st>>>(d_imgs, sel);
    k_sel_split<<<gsel, 256, 0, st>>>(d_imgs, keys, cnt, sel, sel_list, bnd_list);
    const int smem = kSortCap * (int)sizeof(CandKey) + kListCap * (int)sizeof(uint2);
    k_select<<<nimg, 1024, smem, st>>>(d_imgs, keys, kps, cand, det_cand, det_map, cnt, det_out,
                                       desc_in, desc_kp_out, sel, sel_list, bnd_list);
    k_select_big<<<1, 1024, 0, st>>>(d_imgs, nimg, keys, kps, cand, det_cand, det_map, cnt, det_out, desc_in,
                                     desc_kp_out, sel, big_scratch, big_cap);
    dim3 grid((max_points + 31) / 32, nimg);
    k_orient<<<grid, 32, 0, st>>>(d_imgs, pyr, cnt, det_cand, det_map, det_out, desc_in,
                                   desc_kp_out);
    return 6;
}

int launch_describe_prep(const OrbImage* d_imgs, const xa_kp* in, int n, ImgCounters* cnt,
                         DescKp* desc_in, xa_kp* desc_kp_out, cudaStream_t st) {
    k_describe_prep<<<1, 1024, 0, st>>>(d_imgs, in, n, cnt, desc_in, desc_kp_out);
    return 1;
}

int launch_describe(const OrbImage* d_imgs, int nimg, const float* pyr, const ImgCounters* cnt,
                    const DescKp* desc_in, uint64_t* desc, cudaStream_t st) {
    if (nimg <= 0) return 0;
    const int smem = DESC_SMEM;
    dim3 grid(128, nimg);
    k_describe<<<grid, 32 * DESC_WARPS, smem, st>>>(d_imgs, pyr, cnt, desc_in, desc);
    return 1;
}

}  // namespace xa
