// xa_orb.cu — ORB extraction on sm_100a, batched over images (target + views).
//
// Reference: proj/src/orb.cpp (detect_oriented_corners :182-210,
// describe_binary :212-248 and their helpers :25-172), proj/src/image.cpp
// (resize_bilinear, gaussian_blur), proj/src/pipeline.cpp:28-40
// (filter_to_content). Given identical level-0 pixels every output here is
// bit-identical to the reference (tests/test_gpu_orb.py):
//   k_pyramid    levels resized from level 0, exact float/double replay
//   k_fast_nms   FAST-9 at both thresholds (20 and the auto-relax 7) plus the
//                3x3 raster-tie NMS in one pass per 32x16 tile; survivors are
//                compacted with warp ballots. Running both thresholds at once
//                turns the reference's auto-relax re-run (orb.cpp:187-188)
//                into a per-image choice made on the device.
//   k_measures   Harris + intensity-centroid per candidate, reference order
//   k_select     per-image top-N: 32-bit radix select on the response key,
//                then a bitonic sort of the survivors on the exact 96-bit key
//                (response desc, y, x); fused with the content filter and the
//                describe-border drop (order preserving)
//   k_describe   one warp per keypoint: 49x49 window -> sigma=2 separable blur
//                in shared memory -> 256 steered comparisons -> 8 ballots
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

__constant__ int c_ring_dx[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
__constant__ int c_ring_dy[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};

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
                         const xa_kp* __restrict__, ImgCounters* __restrict__,
                         xa_kp* __restrict__, DescKp* __restrict__, xa_kp* __restrict__);
__global__ void k_describe(const OrbImage* __restrict__, const float* __restrict__,
                           const ImgCounters* __restrict__, const DescKp* __restrict__,
                           uint64_t* __restrict__);
constexpr int DESC_WARPS = 4;
constexpr int WIN = 49, HALF = 24, PAT = 37, PHALF = 18;
constexpr int DESC_SMEM_PER_WARP = (WIN * WIN + WIN * PAT) * 4;

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
                             kSortCap * (int)sizeof(CandKey)) != cudaSuccess)
        return -1;
    if (cudaFuncSetAttribute(k_describe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DESC_WARPS * DESC_SMEM_PER_WARP) != cudaSuccess)
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

// ------------------------------------------------------------------ pyramid

// build_pyramid (orb.cpp:130-141): level 0 copied, level i resized from level 0.
__global__ void __launch_bounds__(256) k_pyramid(const OrbImage* __restrict__ imgs,
                                                 const LevelSeg* __restrict__ segs, int nsegs,
                                                 float* __restrict__ pyr) {
    __shared__ LevelSeg s_seg;
    if (threadIdx.x == 0) s_seg = segs[find_seg(segs, nsegs, blockIdx.x)];
    __syncthreads();
    const OrbImage& im = imgs[s_seg.img];
    const int L = s_seg.level;
    const int w = im.w[L], h = im.h[L];
    float* out = pyr + im.poff[L];
    const long long base = (long long)(blockIdx.x - s_seg.blk_start) * 1024;
    const int w0 = im.w[0], h0 = im.h[0];
    const double sx = (double)w0 / w, sy = (double)h0 / h;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const long long i = base + threadIdx.x + 256 * k;
        if (i >= (long long)w * h) return;
        const int y = (int)(i / w), x = (int)(i - (long long)y * w);
        float v;
        if (L == 0)
            v = im.src_type == XA_PIX_U8 ? ld_px((const uint8_t*)im.src, (size_t)i)
                                         : ld_px((const float*)im.src, (size_t)i);
        else
            v = im.src_type == XA_PIX_U8 ? resize_px((const uint8_t*)im.src, w0, h0, sx, sy, x, y)
                                         : resize_px((const float*)im.src, w0, h0, sx, sy, x, y);
        out[i] = v;
    }
}

// ------------------------------------------------------------------ FAST + NMS

constexpr int TW = 32, TH = 16;             // NMS tile
constexpr int SW = TW + 8, SH = TH + 8;     // pixels with the FAST+NMS halo (4)
constexpr int FW = TW + 2, FH = TH + 2;     // FAST results with the NMS halo (1)

// 9 contiguous set bits in the circular 16-bit mask (orb.cpp:60-70).
__device__ __forceinline__ bool arc9(uint32_t m) {
    if (__popc(m) < 9) return false;
    uint32_t d = m | (m << 16);
    uint32_t a = d & (d >> 1);
    a &= a >> 2;
    a &= a >> 4;
    a &= d >> 8;
    return (a & 0xFFFFu) != 0;
}

__global__ void __launch_bounds__(256) k_fast_nms(const OrbImage* __restrict__ imgs,
                                                  const LevelSeg* __restrict__ segs, int nsegs,
                                                  const float* __restrict__ pyr,
                                                  Cand* __restrict__ cand,
                                                  ImgCounters* __restrict__ cnt) {
    __shared__ float s_px[SH][SW];
    __shared__ float s_sc[FH][FW];
    __shared__ uint8_t s_c20[FH][FW];
    __shared__ LevelSeg s_seg;
    __shared__ int s_wcnt[8][2], s_w20[8], s_w7[8];
    __shared__ int s_base;
    const int tid = threadIdx.x;
    if (tid == 0) s_seg = segs[find_seg(segs, nsegs, blockIdx.x)];
    __syncthreads();
    const int img = s_seg.img, L = s_seg.level;
    const OrbImage& im = imgs[img];
    const int w = im.w[L], h = im.h[L];
    const float* lv = pyr + im.poff[L];
    const int t = blockIdx.x - s_seg.blk_start;
    const int ox = kDetectBorder + (t % s_seg.tiles_x) * TW;
    const int oy = kDetectBorder + (t / s_seg.tiles_x) * TH;

    for (int i = tid; i < SW * SH; i += 256) {
        const int sx = i % SW, sy = i / SW;
        const int gx = clampi(ox - 4 + sx, 0, w - 1), gy = clampi(oy - 4 + sy, 0, h - 1);
        s_px[sy][sx] = __ldg(lv + (size_t)gy * w + gx);
    }
    __syncthreads();

    // FAST at both thresholds + sum-abs score (orb.cpp:43-80)
    const int xe = w - kDetectBorder, ye = h - kDetectBorder;
    for (int i = tid; i < FW * FH; i += 256) {
        const int fx = i % FW, fy = i / FW;
        const int gx = ox - 1 + fx, gy = oy - 1 + fy;
        float sc = -1.f;
        uint8_t c20 = 0;
        if (gx >= kDetectBorder && gx < xe && gy >= kDetectBorder && gy < ye) {
            const int cx = fx + 3, cy = fy + 3;
            const float p = s_px[cy][cx];
            const float hi20 = fadd(p, (float)kFastThr), lo20 = fsub(p, (float)kFastThr);
            const float hi7 = fadd(p, (float)kFastThrRelaxed), lo7 = fsub(p, (float)kFastThrRelaxed);
            uint32_t b20 = 0, d20 = 0, b7 = 0, d7 = 0;
            float s = 0.f;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const float v = s_px[cy + c_ring_dy[r]][cx + c_ring_dx[r]];
                b20 |= (uint32_t)(v > hi20) << r;
                d20 |= (uint32_t)(v < lo20) << r;
                b7 |= (uint32_t)(v > hi7) << r;
                d7 |= (uint32_t)(v < lo7) << r;
                s = fadd(s, fabsf(fsub(v, p)));
            }
            const bool k7 = arc9(b7) || arc9(d7);
            if (k7) {
                sc = s;
                c20 = (arc9(b20) || arc9(d20)) ? 1 : 0;
            }
        }
        s_sc[fy][fx] = sc;
        s_c20[fy][fx] = c20;
    }
    __syncthreads();

    // 3x3 NMS with the raster-order tie rule (orb.cpp:152-169), both sets
    const int lane = tid & 31, wid = tid >> 5;
    uint32_t flags[2];
    int px_[2], py_[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int tx = lane, ty = wid + 8 * r;
        const int gx = ox + tx, gy = oy + ty;
        px_[r] = gx;
        py_[r] = gy;
        uint32_t f = 0;
        const float s = s_sc[ty + 1][tx + 1];
        if (s >= 0.f && gx < xe && gy < ye) {
            const bool is20 = s_c20[ty + 1][tx + 1];
            bool keep7 = true, keep20 = is20;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (dx == 0 && dy == 0) continue;
                    const float o = s_sc[ty + 1 + dy][tx + 1 + dx];
                    const bool early = (dy < 0 || (dy == 0 && dx < 0));
                    if (o > s || (o == s && early)) keep7 = false;
                    const float o20 = s_c20[ty + 1 + dy][tx + 1 + dx] ? o : -1.f;
                    if (o20 > s || (o20 == s && early)) keep20 = false;
                }
            f = (keep20 ? 1u : 0u) | (keep7 ? 2u : 0u);
        }
        flags[r] = f;
    }
    uint32_t bal[2], b20[2], b7[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        bal[r] = __ballot_sync(0xffffffffu, flags[r] != 0);
        b20[r] = __ballot_sync(0xffffffffu, flags[r] & 1u);
        b7[r] = __ballot_sync(0xffffffffu, flags[r] & 2u);
    }
    if (lane == 0) {
        s_wcnt[wid][0] = __popc(bal[0]);
        s_wcnt[wid][1] = __popc(bal[1]);
        s_w20[wid] = __popc(b20[0]) + __popc(b20[1]);
        s_w7[wid] = __popc(b7[0]) + __popc(b7[1]);
    }
    __syncthreads();
    if (tid == 0) {
        int tot = 0, t20 = 0, t7 = 0;
        for (int k = 0; k < 8; ++k) {
            tot += s_wcnt[k][0] + s_wcnt[k][1];
            t20 += s_w20[k];
            t7 += s_w7[k];
        }
        s_base = tot ? atomicAdd(&cnt[img].n_cand, tot) : 0;
        if (t20) atomicAdd(&cnt[img].n20, t20);
        if (t7) atomicAdd(&cnt[img].n7, t7);
    }
    __syncthreads();
    if (!(bal[0] | bal[1])) return;
    int off = s_base;
    for (int k = 0; k < wid; ++k) off += s_wcnt[k][0] + s_wcnt[k][1];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        if (flags[r]) {
            const int pos = off + __popc(bal[r] & lt);
            if (pos < im.cand_cap) {
                Cand c;
                c.xy = (uint32_t)px_[r] | ((uint32_t)py_[r] << 16);
                c.lf = (uint32_t)L | (flags[r] << 8);
                cand[im.cand_off + pos] = c;
            } else {
                cnt[img].overflow = 1;
            }
        }
        off += __popc(bal[r]);
    }
}

// ------------------------------------------------------------------ measures

// harris_response (orb.cpp:82-104) in the reference's order and rounding.
__device__ float harris_at(const float* __restrict__ lv, int w, int h, int x, int y) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int dy = -3; dy <= 3; ++dy) {
        const int v = y + dy;
        const size_t rm = (size_t)clampi(v - 1, 0, h - 1) * w;
        const size_t r0 = (size_t)clampi(v, 0, h - 1) * w;
        const size_t rp = (size_t)clampi(v + 1, 0, h - 1) * w;
        for (int dx = -3; dx <= 3; ++dx) {
            const int u = x + dx;
            const int um = clampi(u - 1, 0, w - 1), u0 = clampi(u, 0, w - 1), up = clampi(u + 1, 0, w - 1);
            const float gx = fadd(fadd(fsub(__ldg(lv + rm + up), __ldg(lv + rm + um)),
                                       fmul(2.f, fsub(__ldg(lv + r0 + up), __ldg(lv + r0 + um)))),
                                  fsub(__ldg(lv + rp + up), __ldg(lv + rp + um)));
            const float gy = fadd(fadd(fsub(__ldg(lv + rp + um), __ldg(lv + rm + um)),
                                       fmul(2.f, fsub(__ldg(lv + rp + u0), __ldg(lv + rm + u0)))),
                                  fsub(__ldg(lv + rp + up), __ldg(lv + rm + up)));
            const double ix = gx, iy = gy;
            a = dadd(a, dmul(ix, ix));
            b = dadd(b, dmul(iy, iy));
            c = dadd(c, dmul(ix, iy));
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

// centroid_orientation (orb.cpp:106-123) in the reference's order and rounding.
__device__ float centroid_at(const float* __restrict__ lv, int w, int x, int y) {
    double m01 = 0.0, m10 = 0.0;
    const float* row = lv + (size_t)y * w + x;
    for (int u = -kOrientR; u <= kOrientR; ++u) m10 = dadd(m10, (double)fmul((float)u, __ldg(row + u)));
    for (int v = 1; v <= kOrientR; ++v) {
        const int d = c_umax[v];
        const float* rup = row + (size_t)v * w;
        const float* rdn = row - (size_t)v * w;
        double vs = 0.0;
        for (int u = -d; u <= d; ++u) {
            const double up = __ldg(rup + u), dn = __ldg(rdn + u);
            vs = dadd(vs, dsub(up, dn));
            m10 = dadd(m10, dmul((double)u, dadd(up, dn)));
        }
        m01 = dadd(m01, dmul((double)v, vs));
    }
    return (float)atan2(m01, m10);
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
        const int w = im.w[L], h = im.h[L];
        xa_kp kp;
        const float ls = c_level_scale[L];
        kp.x = fmul((float)x, ls);
        kp.y = fmul((float)y, ls);
        kp.octave_scale = ls;
        kp.response = harris_at(lv, w, h, x, y);
        kp.orientation = centroid_at(lv, w, x, y);
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
__device__ __forceinline__ bool describe_ok(const OrbImage& im, const xa_kp& kp, bool content,
                                            DescKp& d) {
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
    return true;
}

// Order-preserving compaction of det[0..n) into the describe list (4 items per
// thread, 1024 threads). Appends after *io_count.
__device__ void compact_describe(const OrbImage& im, const xa_kp* det, int n, bool content,
                                 DescKp* desc_in, xa_kp* desc_kp, int* s_warp, int* io_count) {
    for (int base = 0; base < n; base += 4096) {
        const int i0 = base + threadIdx.x * 4;
        bool keep[4];
        DescKp d[4];
        int c = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            keep[k] = (i0 + k < n) && describe_ok(im, det[i0 + k], content, d[k]);
            c += keep[k];
        }
        int total;
        int pos = *io_count + block_excl_scan(c, s_warp, &total);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (keep[k]) {
                desc_in[im.kp_off + pos] = d[k];
                desc_kp[im.kp_off + pos] = det[i0 + k];
                ++pos;
            }
        __syncthreads();
        if (threadIdx.x == 0) *io_count += total;
        __syncthreads();
    }
}

// One CTA per image: top-N select + sort (orb.cpp:203-208), then the describe
// list. Dynamic smem: kSortCap CandKey entries.
__global__ void __launch_bounds__(1024) k_select(const OrbImage* __restrict__ imgs,
                                                 const CandKey* __restrict__ keys,
                                                 const xa_kp* __restrict__ kps,
                                                 ImgCounters* __restrict__ cnt,
                                                 xa_kp* __restrict__ det_out,
                                                 DescKp* __restrict__ desc_in,
                                                 xa_kp* __restrict__ desc_kp) {
    extern __shared__ CandKey s_buf[];
    __shared__ int s_hist[256];
    __shared__ int s_warp[32];
    __shared__ int s_n, s_valid, s_prefix_sel, s_remaining, s_count;
    const int img = blockIdx.x;
    const OrbImage& im = imgs[img];
    const int tid = threadIdx.x;
    const int M = min(cnt[img].n_cand, im.cand_cap);
    const int N = im.max_points;
    const CandKey* K = keys + im.cand_off;
    if (tid == 0) {
        s_n = 0;
        s_valid = 0;
    }
    __syncthreads();
    // count valid
    {
        int v = 0;
        for (int i = tid; i < M; i += 1024) v += K[i].idx != 0xFFFFFFFFu;
        atomicAdd(&s_valid, v);
    }
    __syncthreads();
    const int V = s_valid;
    uint32_t thr = 0xFFFFFFFFu;  // gather entries with k0 <= thr
    if (V > kSortCap) {
        // radix select the N-th smallest k0 among valid entries
        uint32_t prefix = 0, mask = 0;
        int remaining = N;
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += 1024) s_hist[i] = 0;
            __syncthreads();
            for (int i = tid; i < M; i += 1024) {
                const CandKey k = K[i];
                if (k.idx != 0xFFFFFFFFu && (k.k0 & mask) == prefix)
                    atomicAdd(&s_hist[(k.k0 >> shift) & 255], 1);
            }
            __syncthreads();
            if (tid == 0) {
                int acc = 0, d = 0;
                for (; d < 256; ++d) {
                    if (acc + s_hist[d] >= remaining) break;
                    acc += s_hist[d];
                }
                s_prefix_sel = d;
                s_remaining = remaining - acc;
            }
            __syncthreads();
            prefix |= (uint32_t)s_prefix_sel << shift;
            mask |= 0xFFu << shift;
            remaining = s_remaining;
            __syncthreads();
        }
        thr = prefix;
    }
    // gather
    for (int i = tid; i < M; i += 1024) {
        const CandKey k = K[i];
        if (k.idx != 0xFFFFFFFFu && k.k0 <= thr) {
            const int p = atomicAdd(&s_n, 1);
            if (p < kSortCap) s_buf[p] = k;
        }
    }
    __syncthreads();
    const int G = s_n;
    if (G > kSortCap) {
        if (tid == 0) {
            cnt[img].overflow = 2;
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
    const int nd = min(G, N);
    xa_kp* det = det_out + im.kp_off;
    for (int i = tid; i < nd; i += 1024) det[i] = kps[im.cand_off + s_buf[i].idx];
    if (tid == 0) {
        cnt[img].n_det = nd;
        s_count = 0;
    }
    __threadfence_block();
    __syncthreads();
    compact_describe(im, det, nd, im.filter != 0, desc_in, desc_kp, s_warp, &s_count);
    if (tid == 0) cnt[img].n_desc = s_count;
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
    compact_describe(imgs[0], in, n, false, desc_in, desc_kp, s_warp, &s_count);
    if (threadIdx.x == 0) cnt[0].n_desc = s_count;
}

// ------------------------------------------------------------------ describe

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

__global__ void __launch_bounds__(32 * DESC_WARPS) k_describe(const OrbImage* __restrict__ imgs,
                                                              const float* __restrict__ pyr,
                                                              const ImgCounters* __restrict__ cnt,
                                                              const DescKp* __restrict__ desc_in,
                                                              uint64_t* __restrict__ desc) {
    extern __shared__ float s_mem[];
    __shared__ int8_t s_pat[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_pat[i] = g_pattern[i];
    __syncthreads();
    const int img = blockIdx.y;
    const OrbImage& im = imgs[img];
    const int n = cnt[img].n_desc;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float* win = s_mem + wid * (WIN * WIN + WIN * PAT);  // later reused for the blurred patch
    float* tmp = win + WIN * WIN;
    for (int k = blockIdx.x * DESC_WARPS + wid; k < n; k += gridDim.x * DESC_WARPS) {
        const DescKp d = desc_in[im.kp_off + k];
        const int w = im.w[d.level], h = im.h[d.level];
        const float* lv = pyr + im.poff[d.level];
        // window with clamp-to-edge (the blur's at_clamped, image.cpp:35,44)
        for (int i = lane; i < WIN * WIN; i += 32) {
            const int r = i / WIN, c = i - r * WIN;
            const int gy = clampi(d.ly - HALF + r, 0, h - 1), gx = clampi(d.lx - HALF + c, 0, w - 1);
            win[i] = __ldg(lv + (size_t)gy * w + gx);
        }
        __syncwarp();
        // horizontal pass on all 49 rows, 37 centre columns
        for (int i = lane; i < WIN * PAT; i += 32) {
            const int r = i / PAT, c = i - r * PAT;
            const float* src = win + r * WIN + c;
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < 13; ++t) acc = fadd(acc, fmul(c_blur2[t], src[t]));
            tmp[i] = acc;
        }
        __syncwarp();
        // vertical pass -> 37x37 blurred patch (stored over the window)
        float* bl = win;
        for (int i = lane; i < PAT * PAT; i += 32) {
            const int r = i / PAT, c = i - r * PAT;
            const float* src = tmp + r * PAT + c;
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < 13; ++t) acc = fadd(acc, fmul(c_blur2[t], src[t * PAT]));
            bl[i] = acc;
        }
        __syncwarp();
        float cs, sn;
        glibc_cossin(d.orientation, cs, sn);
        uint32_t words[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int j = lane + 32 * q;
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
        if (lane < 4) {
            uint64_t wv = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q == lane) wv = (uint64_t)words[2 * q] | ((uint64_t)words[2 * q + 1] << 32);
            desc[(im.kp_off + k) * 4 + lane] = wv;
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ launchers

int launch_pyramid(const OrbImage* d_imgs, const LevelSeg* d_segs, int nsegs, int total_blocks,
                   float* pyr, cudaStream_t st) {
    if (total_blocks <= 0) return 0;
    k_pyramid<<<total_blocks, 256, 0, st>>>(d_imgs, d_segs, nsegs, pyr);
    return 1;
}

int launch_fast_nms(const OrbImage* d_imgs, const LevelSeg* d_segs, int nsegs, int total_blocks,
                    const float* pyr, Cand* cand, ImgCounters* cnt, cudaStream_t st) {
    if (total_blocks <= 0) return 0;
    k_fast_nms<<<total_blocks, 256, 0, st>>>(d_imgs, d_segs, nsegs, pyr, cand, cnt);
    return 1;
}

int launch_measures(const OrbImage* d_imgs, int nimg, const float* pyr, const Cand* cand,
                    const ImgCounters* cnt, CandKey* keys, xa_kp* kps, cudaStream_t st) {
    if (nimg <= 0) return 0;
    dim3 grid(64, nimg);
    k_measures<<<grid, 128, 0, st>>>(d_imgs, pyr, cand, cnt, keys, kps);
    return 1;
}

int launch_select(const OrbImage* d_imgs, int nimg, const CandKey* keys, const xa_kp* kps,
                  ImgCounters* cnt, xa_kp* det_out, DescKp* desc_in, xa_kp* desc_kp_out,
                  cudaStream_t st) {
    if (nimg <= 0) return 0;
    const int smem = kSortCap * (int)sizeof(CandKey);
    k_select<<<nimg, 1024, smem, st>>>(d_imgs, keys, kps, cnt, det_out, desc_in, desc_kp_out);
    return 1;
}

int launch_describe_prep(const OrbImage* d_imgs, const xa_kp* in, int n, ImgCounters* cnt,
                         DescKp* desc_in, xa_kp* desc_kp_out, cudaStream_t st) {
    k_describe_prep<<<1, 1024, 0, st>>>(d_imgs, in, n, cnt, desc_in, desc_kp_out);
    return 1;
}

int launch_describe(const OrbImage* d_imgs, int nimg, const float* pyr, const ImgCounters* cnt,
                    const DescKp* desc_in, uint64_t* desc, cudaStream_t st) {
    if (nimg <= 0) return 0;
    const int smem = DESC_WARPS * DESC_SMEM_PER_WARP;
    dim3 grid(32, nimg);
    k_describe<<<grid, 32 * DESC_WARPS, smem, st>>>(d_imgs, pyr, cnt, desc_in, desc);
    return 1;
}

}  // namespace xa
