// xa_warp.cu — view simulation on sm_100a: directional anti-alias blur and
// nearest / Lanczos-4 affine resampling, batched over views.
//
// Reference: proj/src/warp.cpp:86-158 (warp_nearest, warp_lanczos,
// antialias_tilt), proj/src/image.cpp:25-70 (gaussian_blur, resize_bilinear).
//
// One launch covers every view of a batch: views are flattened into a tile
// list (host-built prefix table, binary-searched per CTA), so wildly unequal
// view sizes (SURVEY.md §7 hard part 5) still fill all 148 SMs.
#include "xa_common.cuh"
#include "xa_kernels.h"

namespace xa {

// ----------------------------------------------------------------- blur

// Directional Gaussian along (cos phi, -sin phi) (warp.cpp:128-158), in the
// reference's arithmetic: per pixel and tap the sample point is x + i*dx,
// y + i*dy in double (i*dx precomputed on the host with the same rounding),
// its floor and (float) fraction give the float bilinear_clamped expression
// (warp.cpp:44-51), and acc += k * sample is a separately rounded double
// multiply and add in tap order -- bit-identical to the reference.
template <class Tin>
__device__ __forceinline__ float bilerp_tap(const Tin* src, int w, int h, int x, int y,
                                            const BlurTap& t) {
    const double X = dadd((double)x, t.px), Y = dadd((double)y, t.py);
    const double fx = floor(X), fy = floor(Y);
    const int x0 = (int)fx, y0 = (int)fy;
    const float wx = (float)dsub(X, fx), wy = (float)dsub(Y, fy);
    const int xa = clampi(x0, 0, w - 1), xb = clampi(x0 + 1, 0, w - 1);
    const int ya = clampi(y0, 0, h - 1), yb = clampi(y0 + 1, 0, h - 1);
    const float v00 = ld_px(src, (size_t)ya * w + xa), v10 = ld_px(src, (size_t)ya * w + xb);
    const float v01 = ld_px(src, (size_t)yb * w + xa), v11 = ld_px(src, (size_t)yb * w + xb);
    const float iwx = fsub(1.f, wx), iwy = fsub(1.f, wy);
    const float top = fadd(fmul(iwx, v00), fmul(wx, v10));
    const float bot = fadd(fmul(iwx, v01), fmul(wx, v11));
    return fadd(fmul(iwy, top), fmul(wy, bot));
}

template <class Tin>
__global__ void __launch_bounds__(256) k_antialias(const BlurView* __restrict__ views,
                                                   const BlurTap* __restrict__ taps,
                                                   const Tin* __restrict__ src, int w, int h,
                                                   float* __restrict__ out) {
    const BlurView v = views[blockIdx.z];
    __shared__ BlurTap s_taps[kMaxBlurTaps];
    for (int i = threadIdx.x + threadIdx.y * 32; i < v.ntaps; i += 256) s_taps[i] = taps[v.tap_off + i];
    __syncthreads();
    const int x = blockIdx.x * 32 + threadIdx.x;
    const int y0 = blockIdx.y * 32 + threadIdx.y;
    if (x >= w) return;
    float* o = out + v.out_off;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int y = y0 + 8 * r;
        if (y >= h) break;
        double acc = 0.0;
        if (v.aligned) {
            const size_t row = (size_t)y * w;
            for (int i = 0; i < v.ntaps; ++i)
                acc = dadd(acc, dmul(s_taps[i].k, (double)ld_px(src, row + clampi(x + s_taps[i].ox, 0, w - 1))));
        } else {
            for (int i = 0; i < v.ntaps; ++i)
                acc = dadd(acc, dmul(s_taps[i].k, (double)bilerp_tap(src, w, h, x, y, s_taps[i])));
        }
        o[(size_t)y * w + x] = (float)acc;
    }
}

// Pipeline blur: the same directional Gaussian folded on the host into one
// 2-D stencil per view (each tap's bilinear cell weights summed per integer
// offset, ~2 cells per tap instead of 4 loads + lerp per tap). A CTA stages its
// 64x64 tile plus the stencil footprint in shared memory (converted to float
// once; interior tiles with 4-pixel vector loads from a 4-aligned start
// column) twice: as loaded (A) and shifted left by one float (B), so that the
// pixel pair (c, c+1) of any stencil offset is one aligned 8-byte load (from A
// when the offset's column parity is even, else from B). Each thread owns two
// adjacent columns x 4 rows (512 threads: 16 warps hide the shared-load
// latency): every stencil entry is one broadcast read + 4 (LDS.64, FFMA2)
// pairs on the packed f32x2 pipe. Float accumulation; parity
// with the reference's double sum is by tolerance (tests/test_gpu_views.py).
__host__ __device__ inline int blur_row_stride(int bx0, int bx1) {
    return (kBlurTW + (bx1 - bx0) + 3 + 3) & ~3;  // + up to 3 alignment columns, 16-byte rows
}

template <class Tin>
__device__ __forceinline__ float4 ld4_px(const Tin* p);
template <>
__device__ __forceinline__ float4 ld4_px<uint8_t>(const uint8_t* p) {
    const uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(p));
    return make_float4((float)(u & 0xFF), (float)((u >> 8) & 0xFF), (float)((u >> 16) & 0xFF),
                       (float)(u >> 24));
}
template <>
__device__ __forceinline__ float4 ld4_px<float>(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

template <class Tin>
__global__ void __launch_bounds__(512) k_blur_stencil(const BlurView* __restrict__ views,
                                                      const BlurCell* __restrict__ cells,
                                                      const Tin* __restrict__ src, int w, int h,
                                                      float* __restrict__ out) {
    extern __shared__ __align__(16) float s_tile[];
    __shared__ int2 s_cell[kMaxBlurCells];
    const BlurView v = views[blockIdx.z];
    const int tid = threadIdx.x + threadIdx.y * 32;
    constexpr int NT = 512;
    const int x0 = blockIdx.x * kBlurTW, y0 = blockIdx.y * kBlurTH;
    // staged columns start at the 4-aligned ax <= x0 + bx0; shift = x0 + bx0 - ax
    const int gx0 = x0 + v.bx0, ax = gx0 & ~3, shift = gx0 - ax;
    const int SW = blur_row_stride(v.bx0, v.bx1), SHd = kBlurTH + v.by1 - v.by0;
    const int gy0 = y0 + v.by0;
    const int nB = SHd * SW;  // copy B (shifted by one float) follows copy A
    for (int i = tid; i < v.ncells; i += NT) {
        const BlurCell c = cells[v.cell_off + i];
        const int a = (c.oy - v.by0) * SW + (c.ox - v.bx0) + shift;  // SW is even
        s_cell[i] = make_int2((a & 1) ? nB + a - 1 : a, __float_as_int(c.w));
    }
    const int nq = SW >> 2;  // 4-pixel groups per staged row
    const bool vec = (w & 3) == 0 && ((size_t)src & (4 * sizeof(Tin) - 1)) == 0;  // aligned 4-px groups
    if (vec && ax >= 0 && ax + SW <= w && gy0 >= 0 && gy0 + SHd <= h) {
        for (int i = tid; i < SHd * nq; i += NT) {
            const int r = i / nq, q = i - r * nq;
            *reinterpret_cast<float4*>(s_tile + r * SW + 4 * q) =
                ld4_px(src + (size_t)(gy0 + r) * w + ax + 4 * q);
        }
    } else {  // image border: clamp per element (at_clamped)
        for (int i = tid; i < SHd * SW; i += NT) {
            const int r = i / SW, c = i - r * SW;
            const int gx = clampi(ax + c, 0, w - 1), gy = clampi(gy0 + r, 0, h - 1);
            s_tile[i] = ld_px(src, (size_t)gy * w + gx);
        }
    }
    __syncthreads();
    for (int i = tid; i < nB - 1; i += NT) s_tile[nB + i] = s_tile[i + 1];
    __syncthreads();
    const int tx = threadIdx.x, ty = threadIdx.y;
    float2 acc[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[r] = make_float2(0.f, 0.f);
    const float* base = s_tile + ty * SW + 2 * tx;
    for (int c = 0; c < v.ncells; ++c) {
        const int2 cl = s_cell[c];
        const float wgt = __int_as_float(cl.y);
        const float2 wv = make_float2(wgt, wgt);
        const float2* p = reinterpret_cast<const float2*>(base + cl.x);
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] = __ffma2_rn(wv, p[r * 8 * SW], acc[r]);
    }
    const int x = x0 + 2 * tx;
    if (x >= w) return;
    float* o = out + v.out_off;
    const bool pair = x + 1 < w && ((v.out_off + x) & 1) == 0 && (w & 1) == 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int y = y0 + ty + 16 * r;
        if (y >= h) break;
        float* q = o + (size_t)y * w + x;
        if (pair) {
            *reinterpret_cast<float2*>(q) = acc[r];
        } else {
            q[0] = acc[r].x;
            if (x + 1 < w) q[1] = acc[r].y;
        }
    }
}


// Directional blur as runs (k_blur_runs): the folded stencil (blur_stencil)
// grouped into runs along its long axis -- rowmode (|dx| >= |dy|): cells of
// one row oy, contiguous in ox; else cells of one column. A warp owns an
// 8-pixel block along the run axis and 32 (+32) lanes across it (lanes on
// different rows / columns: conflict-free scalar shared loads, odd row
// stride); each lane keeps an 11-value sliding window in registers, so a
// staged pixel is loaded once per run and feeds 8 outputs x 4 weights per
// block (the stencil kernel loads it once per cell). Every output pixel
// accumulates its cells in (run, offset) order with FMA; zero-padded weights
// add exact zeros. Output tile 64 x 64, 256 threads.
int blur_runs_tile_floats(const BlurView& v) {
    int SW, SH;
    blur_runs_geometry(v, SW, SH);
    return SW * SH;
}

template <class Tin>
__global__ void __launch_bounds__(256) k_blur_runs(const BlurView* __restrict__ views, const BlurRun* __restrict__ runs,
                                                   const float* __restrict__ rw, const Tin* __restrict__ src, int w,
                                                   int h, float* __restrict__ out) {
    extern __shared__ __align__(16) float s_tile[];
    __shared__ BlurRun s_run[kMaxBlurRuns];
    __shared__ __align__(16) float s_w[kMaxBlurRunW];
    const BlurView v = views[blockIdx.z];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int x0 = blockIdx.x * 64, y0 = blockIdx.y * 64;
    int SW, SH;
    blur_runs_geometry(v, SW, SH);
    const int gx0 = x0 + v.bx0, gy0 = y0 + v.by0;
    const int ax = gx0 & ~3;
    if (sizeof(Tin) == 1 && (w & 3) == 0 && ((size_t)src & 3) == 0 && ax >= 0 && ax + SW + 4 <= w && gy0 >= 0 &&
        gy0 + SH <= h) {
        // interior uint8 tile: aligned 4-pixel words, each lane's word spread to 4 floats
        const int nq = (gx0 - ax + SW + 3) >> 2;
        for (int r = wid; r < SH; r += 8) {
            const uint32_t* row = reinterpret_cast<const uint32_t*>(src + (size_t)(gy0 + r) * w + ax);
            float* d = s_tile + r * SW - (gx0 - ax);
            for (int q = lane; q < nq; q += 32) {
                const uint32_t u = __ldg(row + q);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int c = 4 * q + i - (gx0 - ax);
                    if (c >= 0 && c < SW) d[4 * q + i] = (float)((u >> (8 * i)) & 0xFFu);
                }
            }
        }
    } else if (gx0 >= 0 && gx0 + SW <= w && gy0 >= 0 && gy0 + SH <= h) {
        for (int r = wid; r < SH; r += 8) {
            const Tin* row = src + (size_t)(gy0 + r) * w + gx0;
            for (int c = lane; c < SW; c += 32) s_tile[r * SW + c] = ld_px(row, c);
        }
    } else {  // image border: clamp per element (at_clamped)
        for (int r = wid; r < SH; r += 8) {
            const Tin* row = src + (size_t)clampi(gy0 + r, 0, h - 1) * w;
            for (int c = lane; c < SW; c += 32) s_tile[r * SW + c] = ld_px(row, clampi(gx0 + c, 0, w - 1));
        }
    }
    for (int i = tid; i < v.nruns; i += 256) s_run[i] = runs[v.run_off + i];
    for (int i = tid; i < v.nrw; i += 256) s_w[i] = rw[v.rw_off + i];
    __syncthreads();
    // the lane's two outputs rows / columns (hh = 0, 1) ride in one packed
    // pair: FFMA2 with the run weight as the scalar operand
    float2 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float2(0.f, 0.f);
    // rowmode: window along x (step 1), lanes along y (step SW); else transposed
    const int ws = v.rowmode ? 1 : SW, hs = 32 * (v.rowmode ? SW : 1);
    const float* cbase = v.rowmode ? s_tile + lane * SW + 8 * wid : s_tile + 8 * wid * SW + lane;
    for (int ri = 0; ri < v.nruns; ++ri) {
        const BlurRun R = s_run[ri];
        const float* p = cbase + R.major;  // host-resolved tile offset of the run start
        float2 win[11];
#pragma unroll
        for (int k = 0; k < 7; ++k) win[k] = make_float2(p[k * ws], p[k * ws + hs]);
        const float* wp = s_w + R.woff;
        for (int b = 0; b < R.nblk; ++b) {
            const float* pb = p + (7 + 4 * b) * ws;
#pragma unroll
            for (int k = 0; k < 4; ++k) win[7 + k] = make_float2(pb[k * ws], pb[k * ws + hs]);
            const float4 wt = *reinterpret_cast<const float4*>(wp + 4 * b);
            const float wj[4] = {wt.x, wt.y, wt.z, wt.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(make_float2(wj[j], wj[j]), win[k + j], acc[k]);
#pragma unroll
            for (int k = 0; k < 7; ++k) win[k] = win[k + 4];
        }
    }
    float* o = out + v.out_off;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        if (v.rowmode) {
            const int y = y0 + lane + 32 * hh, x = x0 + 8 * wid;
            if (y >= h) continue;
            float* d = o + (size_t)y * w + x;
            if (x + 8 <= w && (((size_t)(v.out_off + (size_t)y * w + x)) & 3) == 0) {
                const float a0 = hh ? acc[0].y : acc[0].x, a1 = hh ? acc[1].y : acc[1].x, a2 = hh ? acc[2].y : acc[2].x,
                            a3 = hh ? acc[3].y : acc[3].x, a4 = hh ? acc[4].y : acc[4].x, a5 = hh ? acc[5].y : acc[5].x,
                            a6 = hh ? acc[6].y : acc[6].x, a7 = hh ? acc[7].y : acc[7].x;
                reinterpret_cast<float4*>(d)[0] = make_float4(a0, a1, a2, a3);
                reinterpret_cast<float4*>(d)[1] = make_float4(a4, a5, a6, a7);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (x + k < w) d[k] = hh ? acc[k].y : acc[k].x;
            }
        } else {
            const int x = x0 + lane + 32 * hh, y = y0 + 8 * wid;
            if (x >= w) continue;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (y + k < h) o[(size_t)(y + k) * w + x] = hh ? acc[k].y : acc[k].x;
        }
    }
}

// ----------------------------------------------------------------- resample

__device__ __forceinline__ int find_view_warp(const WarpView* __restrict__ views, int n, int tile) {
    const int lane = threadIdx.x & 31;
    int base = 0, span = n;
    while (span > 1) {
        const int stride = (span + 31) >> 5;
        const int off = lane * stride;
        const bool ok = off < span && views[base + off].tile_start <= tile;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        const int k = 31 - __clz(m);
        base += k * stride;
        span = min(stride, span - k * stride);
    }
    return base;
}

// sin and cos of theta = pi*r/4, r in [0,1] (theta <= pi/4): Taylor to degree 9 / 10.
__device__ __forceinline__ void sincos_q(float r, float& s, float& c) {
    const float x = 0.785398163397448f * r, x2 = x * x;
    float ps = 2.7557319e-6f;
    ps = fmaf(ps, x2, -1.9841270e-4f);
    ps = fmaf(ps, x2, 8.3333333e-3f);
    ps = fmaf(ps, x2, -1.6666667e-1f);
    s = fmaf(ps * x2, x, x);
    float pc = -2.7557319e-7f;
    pc = fmaf(pc, x2, 2.4801587e-5f);
    pc = fmaf(pc, x2, -1.3888889e-3f);
    pc = fmaf(pc, x2, 4.1666667e-2f);
    pc = fmaf(pc, x2, -0.5f);
    c = fmaf(pc, x2, 1.f);
}

// Lanczos-4 weights for taps i = -3..4 at fractional offset r in [0,1), up to
// the common factor pi^2/4 that sample_lanczos's acc/wsum normalisation cancels
// (warp.cpp:55-84): L(t) ~ sin(pi t) sin(pi t/4) / t^2 with
// sin(pi(i-r)) = -(-1)^i sin(pi r) and sin(pi(i-r)/4) by angle addition.
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void lanczos_w(float r, float* wt) {
    // r in [1e-12, 1 - 2^-24] keeps t*t normal for the taps at t = -r and
    // t = 1 - r (r arrives as (float)(sx - floor(sx)), which can round to 1);
    // at the ends the weights tend to a single pi^2/4 tap (relative change
    // <= 1e-7), matching the reference's t == 0 case.
    r = fminf(fmaxf(r, 1e-12f), 0.99999994f);
    float s4, c4;
    sincos_q(r, s4, c4);
    // numerator_j = sign_j * sin(pi r) * (sin(pi i/4) c4 - cos(pi i/4) s4), signs
    // folded: with (-(-1)^i) sin(pi i/4), (-(-1)^i) cos(pi i/4) for i = -3..4
    // the numerators are (a, p, -b, q, -a, -p, b, -q), a = k(q - p), b = k(p + q).
    // sin(pi r) is common to all eight taps and cancels in the normalisation,
    // so p = c4, q = s4 (at r -> 0 the t = -r tap still dominates as ~1/r).
    const float p = c4, q = s4;
    const float k = 0.70710678118654752f;
    const float a = k * (q - p), b = k * (p + q);
    const float num[8] = {a, p, -b, q, -a, -p, b, -q};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float t = (float)(j - 3) - r;
        wt[j] = num[j] * rcp_approx(t * t);
    }
}

// lanczos_w for both axes at once on the packed f32x2 pipe: (wx_j, wy_j) per
// tap pair j, and the two weight sums (same formula, same rounding per op).
__device__ __forceinline__ float2 f2s(float v) { return make_float2(v, v); }

__device__ __forceinline__ void lanczos_wxy(float2 r, float2* w, float2& sum) {
    r.x = fminf(fmaxf(r.x, 1e-12f), 0.99999994f);
    r.y = fminf(fmaxf(r.y, 1e-12f), 0.99999994f);
    const float2 x = __fmul2_rn(f2s(0.785398163397448f), r), x2 = __fmul2_rn(x, x);
    float2 ps = __ffma2_rn(f2s(2.7557319e-6f), x2, f2s(-1.9841270e-4f));
    ps = __ffma2_rn(ps, x2, f2s(8.3333333e-3f));
    ps = __ffma2_rn(ps, x2, f2s(-1.6666667e-1f));
    const float2 q = __ffma2_rn(__fmul2_rn(ps, x2), x, x);
    float2 pc = __ffma2_rn(f2s(-2.7557319e-7f), x2, f2s(2.4801587e-5f));
    pc = __ffma2_rn(pc, x2, f2s(-1.3888889e-3f));
    pc = __ffma2_rn(pc, x2, f2s(4.1666667e-2f));
    pc = __ffma2_rn(pc, x2, f2s(-0.5f));
    const float2 p = __ffma2_rn(pc, x2, f2s(1.f));
    const float2 k = f2s(0.70710678118654752f);
    const float2 a = __fmul2_rn(k, __fadd2_rn(q, make_float2(-p.x, -p.y)));
    const float2 b = __fmul2_rn(k, __fadd2_rn(p, q));
    const float2 num[8] = {a, p, make_float2(-b.x, -b.y), q, make_float2(-a.x, -a.y),
                           make_float2(-p.x, -p.y), b, make_float2(-q.x, -q.y)};
    const float2 nr = make_float2(-r.x, -r.y);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float2 t = __fadd2_rn(f2s((float)(j - 3)), nr);
        const float2 u = __fmul2_rn(t, t);
        w[j] = __fmul2_rn(num[j], make_float2(rcp_approx(u.x), rcp_approx(u.y)));
    }
    sum = w[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) sum = __fadd2_rn(sum, w[j]);
}

template <class Tin>
__device__ __forceinline__ float lanczos_px(const Tin* __restrict__ src, int w, int h, double sx,
                                            double sy) {
    const double fxd = floor(sx), fyd = floor(sy);
    const int fx = (int)fxd, fy = (int)fyd;
    float wx[8], wy[8];
    lanczos_w((float)(sx - fxd), wx);
    lanczos_w((float)(sy - fyd), wy);
    float sw = wx[0], sh = wy[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        sw += wx[i];
        sh += wy[i];
    }
    float acc = 0.f;
    if (fx >= 3 && fx + 4 < w && fy >= 3 && fy + 4 < h) {
        // interior: one base pointer, constant offsets per tap
        const Tin* p = src + (size_t)(fy - 3) * w + (fx - 3);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float rs = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) rs = fmaf(wx[i], ld_px(p, i), rs);
            acc = fmaf(wy[j], rs, acc);
            p += w;
        }
    } else {
        int xs[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xs[i] = clampi(fx + i - 3, 0, w - 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const size_t row = (size_t)clampi(fy + j - 3, 0, h - 1) * w;
            float rs = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) rs = fmaf(wx[i], ld_px(src, row + xs[i]), rs);
            acc = fmaf(wy[j], rs, acc);
        }
    }
    const float v = __fdividef(acc, sw * sh);
    return fminf(fmaxf(v, 0.f), 255.f);
}

// View value as stored: uint8 views use the lround + clamp quantisation of
// image_io.cpp:17-20.
template <class Tout>
__device__ __forceinline__ float quant_px(float v) {
    return sizeof(Tout) == 1 ? fminf(fmaxf(roundf(v), 0.f), 255.f) : v;
}

// Store one view pixel to the view buffer (if any) and, for coarse batches,
// as ORB pyramid level 0 (float, pitched) so k_pyramid never re-reads it.
// IN_RANGE: val is already clamped to [0, 255] (the Lanczos paths), so the
// quantisation needs only the rounding
template <class Tout, bool IN_RANGE = false>
__device__ __forceinline__ void store_view(const WarpView& v, Tout* out, float* pyr, int x, int y,
                                           float val) {
    const float q = IN_RANGE && sizeof(Tout) == 1 ? roundf(val) : quant_px<Tout>(val);
    if (out) out[v.out_off + (size_t)y * v.W + x] = (Tout)q;
    if (pyr) pyr[v.pyr_off + (size_t)y * v.pyr_pitch + x] = q;
}

template <class Tin, class Tout, int MODE>
__device__ __forceinline__ void warp_tile(const WarpView& v, int tile, Tout* out, float* pyr) {
    const int t = tile - v.tile_start;
    const int tx = t % v.tiles_x, ty = t / v.tiles_x;
    const int x = tx * 32 + (threadIdx.x & 31);
    const int yb = ty * 32 + (threadIdx.x >> 5);
    if (x >= v.W) return;
    const Tin* src = static_cast<const Tin*>(v.src);
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
        const int y = yb + 8 * r;
        if (y >= v.H) return;
        double sx, sy;
        map_pt(v.back, (double)x, (double)y, sx, sy);
        float val = 0.f;
        if (MODE == 0) {
            // warp_nearest (warp.cpp:96-103): lround, copy if inside
            const double rx = round(sx), ry = round(sy);
            if (rx >= 0.0 && rx < (double)v.sw && ry >= 0.0 && ry < (double)v.sh)
                val = ld_px(src, (size_t)(int)ry * v.sw + (int)rx);
        } else {
            // warp_lanczos (warp.cpp:116-124): outside the content domain stays 0
            if (!(sx < 0.0 || sx > v.sw - 1.0 || sy < 0.0 || sy > v.sh - 1.0))
                val = lanczos_px(src, v.sw, v.sh, sx, sy);
        }
        store_view(v, out, pyr, x, y, val);
    }
}

template <class Tout, int MODE>
__global__ void __launch_bounds__(256, 3) k_warp(const WarpView* __restrict__ views, int nviews,
                                                 Tout* __restrict__ out, float* __restrict__ pyr) {
    __shared__ WarpView s_v;
    if (threadIdx.x < 32) {
        const int k = find_view_warp(views, nviews, blockIdx.x);
        if (threadIdx.x == 0) s_v = views[k];
    }
    __syncthreads();
    const WarpView& v = s_v;
    if (v.src_type == XA_PIX_U8)
        warp_tile<uint8_t, Tout, MODE>(v, blockIdx.x, out, pyr);
    else
        warp_tile<float, Tout, MODE>(v, blockIdx.x, out, pyr);
}

// Lanczos views with the source footprint staged in shared memory. A CTA owns
// a T x TH output tile (64x64 ... 8x8 per view, chosen on the host so the
// footprint fits); it back-maps the tile corners, loads the bounding box plus
// the 8-tap support once (clamped = at_clamped, coalesced rows, padded stride
// against bank conflicts), then every pixel's 64 taps are shared-memory reads.
// Without this, a warp's 32 pixels of a rotated view touch ~32 different
// source rows per load (L1 wavefront-bound, profiles/r01_*).
template <class Tin, class Tout>
__device__ __forceinline__ void lanczos_tile(const WarpView& v, int tile, float* s_src, Tout* out,
                                             float* pyr, uint64_t* bar, const char* maps, int zpass) {
    const int T = v.tile, TH = v.tile_h;
    const int t = tile - v.tile_start;
    const int x0 = (t % v.tiles_x) * T, y0 = (t / v.tiles_x) * TH;
    __shared__ int s_box[5];
    if (threadIdx.x == 0) {
        const int xm = min(x0 + T, v.W) - 1, ym = min(y0 + TH, v.H) - 1;
        double mnx = 1e300, mny = 1e300, mxx = -1e300, mxy = -1e300;
        const int cx[4] = {x0, xm, x0, xm}, cy[4] = {y0, y0, ym, ym};
        for (int k = 0; k < 4; ++k) {
            double sx, sy;
            map_pt(v.back, (double)cx[k], (double)cy[k], sx, sy);
            mnx = fmin(mnx, sx);
            mxx = fmax(mxx, sx);
            mny = fmin(mny, sy);
            mxy = fmax(mxy, sy);
        }
        // tile entirely outside the content domain (by a margin far above the
        // rounding of the per-pixel back-mapping): every pixel is 0
        const double eps = 1e-6;
        const bool outside = mnx > v.sw - 1.0 + eps || mxx < -eps || mny > v.sh - 1.0 + eps || mxy < -eps;
        // clip to the content domain [0, w-1] x [0, h-1] (outside pixels stay 0);
        // one column/row of slack beyond the 8-tap support on each side
        mnx = fmax(mnx, 0.0);
        mny = fmax(mny, 0.0);
        mxx = fmin(mxx, v.sw - 1.0);
        mxy = fmin(mxy, v.sh - 1.0);
        const int bx0 = (int)floor(mnx) - 4, by0 = (int)floor(mny) - 4;
        s_box[0] = bx0;
        s_box[1] = by0;
        s_box[2] = outside ? 0 : (int)floor(mxx) + 6 - bx0;
        s_box[3] = outside ? 0 : (int)floor(mxy) + 6 - by0;
        s_box[4] = outside;
    }
    __syncthreads();
    const int bx0 = s_box[0], by0 = s_box[1], bw = s_box[2], bh = s_box[3];
    // zpass 1: only the tiles outside the content (their zeros); zpass 2: those
    // tiles were zeroed by a zpass-1 launch of the same tile table and are skipped
    if (zpass == 1 && !s_box[4]) return;
    if (s_box[4]) {
        if (zpass == 2) return;
        if (!out && pyr && T >= 4) {
            // level 0 only (coarse chain): 16-byte zero stores (pitch and x0 are
            // multiples of 4 floats; the last column group may run into the
            // pitch padding, which no reader takes as pixels)
            const int cols = (min(T, v.W - x0) + 3) >> 2, rows = min(TH, v.H - y0);
            const int lq = 29 - __clz(T);  // log2(T / 4)
            float* base = pyr + v.pyr_off + (size_t)y0 * v.pyr_pitch + x0;
            for (int i = threadIdx.x; i < (rows << lq); i += blockDim.x) {
                const int c = i & ((1 << lq) - 1), r = i >> lq;
                if (c < cols)
                    *reinterpret_cast<float4*>(base + (size_t)r * v.pyr_pitch + 4 * c) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            return;
        }
        const int lt = 31 - __clz(T);  // T is a power of two
        for (int i = threadIdx.x; i < T * TH; i += blockDim.x) {
            const int x = x0 + (i & (T - 1)), y = y0 + (i >> lt);
            if (x < v.W && y < v.H) store_view(v, out, pyr, x, y, 0.f);
        }
        return;
    }
    // One copy of the footprint, staged from ax = the 16-byte aligned column
    // at or left of bx0: interior tiles copy whole 16-byte chunks (cp.async,
    // no clamps), tiles touching the image border copy clamped floats.
    const int ax = bx0 & ~3;
    int stride = lanczos_stride(bw, v.lz_res);
    const Tin* src = static_cast<const Tin*>(v.src);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (sizeof(Tin) == 4) {  // float source (blurred views): async copies, no register round trip
        const float* fsrc = reinterpret_cast<const float*>(src);
        if (maps && v.tmap_idx >= 0 && ax >= 0 && ax + v.lz_stride <= v.sw && by0 >= 0 &&
            by0 + v.lz_box_h <= v.sh && bh <= v.lz_box_h) {
            // interior footprint: one 2-D tensor TMA of the view's box
            // (lz_stride x lz_box_h floats at (ax, by0)) into rows of lz_stride
            stride = v.lz_stride;
            if (threadIdx.x == 0) {
                mbar_arrive_tx(bar, (unsigned)(v.lz_box_h * stride) * (unsigned)sizeof(float));
                tma_load_2d(s_src, maps + (size_t)v.tmap_idx * 128, ax, by0, bar);
            }
            mbar_wait(bar, 0);
        } else if (ax >= 0 && ax + stride <= v.sw && by0 >= 0 && by0 + bh <= v.sh && (v.sw & 3) == 0 &&
                   bh <= (int)blockDim.x) {
            // interior footprint without a tensor map: one bulk copy per row
            if (threadIdx.x == 0) mbar_arrive_tx(bar, (unsigned)(bh * stride) * (unsigned)sizeof(float));
            if ((int)threadIdx.x < bh)
                bulk_g2s(s_src + threadIdx.x * stride, fsrc + (size_t)(by0 + threadIdx.x) * v.sw + ax,
                         (unsigned)stride * (unsigned)sizeof(float), bar);
            mbar_wait(bar, 0);
        } else {
            for (int r = wid; r < bh; r += nw) {
                const float* row = fsrc + (size_t)clampi(by0 + r, 0, v.sh - 1) * v.sw;
                for (int c = lane; c < stride; c += 32)
                    cp_async4(s_src + r * stride + c, row + clampi(ax + c, 0, v.sw - 1));
            }
            cp_async_commit();
            cp_async_wait<0>();
        }
    } else {
        for (int r = wid; r < bh; r += nw) {
            const size_t row = (size_t)clampi(by0 + r, 0, v.sh - 1) * v.sw;
            for (int c = lane; c < stride; c += 32)
                s_src[r * stride + c] = ld_px(src, row + clampi(ax + c, 0, v.sw - 1));
        }
    }
    __syncthreads();
    // each warp takes (1 << pw) x (32 >> pw) output patches, the shape and the
    // stride residue planned per view so the 32 tap windows of a load fall in
    // distinct banks (lanczos_bank_plan)
    const int pw = v.lz_pw, ph = 5 - pw;
    const int wsh = (31 - __clz(T)) - pw;  // log2 patches per patch row
    const int npatch = (T * TH) >> 5;
    for (int pt = wid; pt < npatch; pt += nw) {
        const int x = x0 + ((pt & ((1 << wsh) - 1)) << pw) + (lane & ((1 << pw) - 1));
        const int y = y0 + ((pt >> wsh) << ph) + (lane >> pw);
        if (x >= v.W || y >= v.H) continue;
        double sx, sy;
        map_pt(v.back, (double)x, (double)y, sx, sy);
        float val = 0.f;
        if (!(sx < 0.0 || sx > v.sw - 1.0 || sy < 0.0 || sy > v.sh - 1.0)) {
            const double fxd = floor(sx), fyd = floor(sy);
            // both axes' weights at once on the packed f32x2 pipe (bit-identical
            // to two lanczos_w calls: the same operations, each rounded once)
            float wx[8], wy[8];
            float2 wxy[8], s2;
            lanczos_wxy(make_float2((float)(sx - fxd), (float)(sy - fyd)), wxy, s2);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                wx[i] = wxy[i].x;
                wy[i] = wxy[i].y;
            }
            const float sw = s2.x, sh = s2.y;
            // 8 taps from an 8-byte aligned 10-float window: an odd start
            // column shifts the weights by one (a zero weight first instead of
            // last), which leaves every partial sum unchanged
            const int col = (int)fxd - 3 - ax;
            const bool odd = col & 1;
            float w9[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) w9[i] = odd ? (i ? wx[i - 1] : 0.f) : (i < 8 ? wx[i] : 0.f);
            const float2* p = reinterpret_cast<const float2*>(s_src + ((int)fyd - 3 - by0) * stride + (col & ~1));
            const int st2 = stride >> 1;
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float rs = 0.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 q = p[i];
                    rs = fmaf(w9[2 * i], q.x, rs);
                    rs = fmaf(w9[2 * i + 1], q.y, rs);
                }
                rs = fmaf(w9[8], p[4].x, rs);
                acc = fmaf(wy[j], rs, acc);
                p += st2;
            }
            val = fminf(fmaxf(__fdividef(acc, sw * sh), 0.f), 255.f);
        }
        store_view<Tout, true>(v, out, pyr, x, y, val);
    }
}

template <class Tout>
__global__ void __launch_bounds__(256, 4) k_lanczos_smem(const WarpView* __restrict__ views,
                                                         int nviews, Tout* __restrict__ out,
                                                         float* __restrict__ pyr,
                                                         const char* __restrict__ maps, int zpass) {
    extern __shared__ __align__(128) float s_src[];
    __shared__ WarpView s_v;
    __shared__ __align__(8) uint64_t s_bar;  // footprint bulk-copy completion (one use per CTA)
    if (threadIdx.x < 32) {
        const int k = find_view_warp(views, nviews, blockIdx.x);
        // the view record copied by the warp's lanes, one word each
        static_assert(sizeof(WarpView) % 4 == 0, "word copy");
        const unsigned* gv = reinterpret_cast<const unsigned*>(views + k);
        unsigned* sv = reinterpret_cast<unsigned*>(&s_v);
        for (int i = threadIdx.x; i < (int)(sizeof(WarpView) / 4); i += 32) sv[i] = gv[i];
        if (threadIdx.x == 0) {
            mbar_init(&s_bar, 1);
            fence_mbar_init();
        }
    }
    __syncthreads();
    if (s_v.src_type == XA_PIX_U8)
        lanczos_tile<uint8_t, Tout>(s_v, blockIdx.x, s_src, out, pyr, &s_bar, maps, zpass);
    else
        lanczos_tile<float, Tout>(s_v, blockIdx.x, s_src, out, pyr, &s_bar, maps, zpass);
}


// Separable Lanczos for views whose back-map is diagonal (phi = 0 grid entries,
// including the identity view t = 1: b1 = b3 = 0 exactly, so sx depends on x
// only and sy on y only). sample_lanczos (warp.cpp:62-84) is then a horizontal
// pass per (source row, output column) followed by a vertical pass per output
// pixel: each row sum rs_j = sum_i wx_i S[fy + j - 3][fx + i - 3] is shared by
// every output row that reads source row fy + j - 3, so a 64 x 64 tile costs
// (64 / s + 8) x 64 x 8 + 64 x 64 x 8 MACs instead of 64 x 64 x 64. Weights,
// tap order (fmaf chains from 0 over the 8 taps, then over the 8 row sums),
// the wsum product and the division are those of k_lanczos_smem, so the
// values are bit-identical. Out-of-range taps clamp (at_clamped).
// staged source rows / columns of a 64 x 64 tile: |b4| 63 + 10 and |b0| 63 + 10
// must fit (the host routes a diagonal view here only then)
constexpr int kSepRows = 76, kSepCols = 136, kSepSW = kSepCols + 1;
constexpr int kSepSmemBytes = (kSepRows * kSepSW + kSepRows * 65) * 4;

struct SepShared {
    float wx[64][9], wy[64][9];  // 8 weights + their sum, per column / row
    int fx[64], fy[64];
    unsigned char inx[64], iny[64];
    int r0, c0, nr, nc;
};

template <class Tin, class Tout>
__device__ __forceinline__ void lanczos_sep_tile(const WarpView& v, int tile, Tout* out, float* pyr,
                                                 SepShared& S, float* s_dyn) {
    float(*s_wx)[9] = S.wx;
    float(*s_wy)[9] = S.wy;
    int* s_fx = S.fx;
    int* s_fy = S.fy;
    unsigned char* s_inx = S.inx;
    unsigned char* s_iny = S.iny;
    int &s_r0 = S.r0, &s_c0 = S.c0, &s_nr = S.nr, &s_nc = S.nc;
    float(*s_src)[kSepSW] = reinterpret_cast<float(*)[kSepSW]>(s_dyn);
    float(*s_h)[65] = reinterpret_cast<float(*)[65]>(s_dyn + kSepRows * kSepSW);
    const int T = 64;
    const int t = tile - v.tile_start;
    const int x0 = (t % v.tiles_x) * T, y0 = (t / v.tiles_x) * T;
    const int tid = threadIdx.x;
    if (tid < 128) {  // per column (tid < 64) / per row (64..127): floor, fractional weights, inside
        const int k = tid & 63;
        const bool col = tid < 64;
        const int xy = (col ? x0 : y0) + k;
        double sxy;
        if (col) sxy = dadd(dadd(dmul(v.back[0], (double)xy), dmul(v.back[1], (double)y0)), v.back[2]);
        else sxy = dadd(dadd(dmul(v.back[3], (double)x0), dmul(v.back[4], (double)xy)), v.back[5]);
        const double f = floor(sxy);
        float2 w2[8], s2;
        const float r = (float)(sxy - f);
        lanczos_wxy(make_float2(r, r), w2, s2);
        float* wrow = col ? s_wx[k] : s_wy[k];
#pragma unroll
        for (int i = 0; i < 8; ++i) wrow[i] = w2[i].x;
        wrow[8] = s2.x;
        const int lim = col ? v.sw : v.sh;
        if (col) {
            s_fx[k] = (int)f;
            s_inx[k] = !(sxy < 0.0 || sxy > lim - 1.0);
        } else {
            s_fy[k] = (int)f;
            s_iny[k] = !(sxy < 0.0 || sxy > lim - 1.0);
        }
    }
    __syncthreads();
    if (tid == 0) {
        const int nyv = min(T, v.H - y0), nxv = min(T, v.W - x0);
        s_r0 = s_fy[0] - 3;
        s_c0 = s_fx[0] - 3;
        s_nr = s_fy[nyv - 1] + 5 - s_r0;
        s_nc = s_fx[nxv - 1] + 5 - s_c0;
    }
    __syncthreads();
    const int r0 = s_r0, c0 = s_c0, nr = s_nr, nc = s_nc;
    // stage the source region (clamped) once; interior float tiles as 16-byte
    // async copies from the 4-aligned column at or left of c0
    const Tin* src = static_cast<const Tin*>(v.src);
    const int ca = c0 & ~3, sh4 = c0 - ca;
    if (sizeof(Tin) == 4 && (v.sw & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && ca >= 0 &&
        ca + nc + sh4 + 3 <= v.sw && r0 >= 0 && r0 + nr <= v.sh) {
        const int nq = (nc + sh4 + 3) >> 2;
        for (int r = tid >> 5; r < nr; r += 8) {
            const float* row = reinterpret_cast<const float*>(src) + (size_t)(r0 + r) * v.sw + ca;
            for (int q = tid & 31; q < nq; q += 32) {
                const float4 f = __ldg(reinterpret_cast<const float4*>(row) + q);
                const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int c = 4 * q + i - sh4;
                    if (c >= 0 && c < nc) s_src[r][c] = fv[i];
                }
            }
        }
    } else {
        for (int r = tid >> 5; r < nr; r += 8) {
            const size_t row = (size_t)clampi(r0 + r, 0, v.sh - 1) * v.sw;
            for (int c = tid & 31; c < nc; c += 32) s_src[r][c] = ld_px(src, row + clampi(c0 + c, 0, v.sw - 1));
        }
    }
    __syncthreads();
    // horizontal pass: H[r][x] = sum_i wx_i(x) S[r][fx(x) - 3 + i]; lanes own
    // columns x and x + 32 (weights in registers), warps rows r = w, w + 8, ...
    const int nxv = min(T, v.W - x0), nyv = min(T, v.H - y0);
    const int lane = tid & 31, wid = tid >> 5;
    float wa[8], wb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        wa[k] = s_wx[lane][k];
        wb[k] = s_wx[lane + 32][k];
    }
    const int fa = s_fx[lane] - 3 - c0, fb = s_fx[lane + 32] - 3 - c0;
    const bool va = lane < nxv, vb = lane + 32 < nxv;
    for (int r = wid; r < nr; r += 8) {
        const float* row = s_src[r];
        float ra = 0.f, rb = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (va) ra = fmaf(wa[k], row[fa + k], ra);
            if (vb) rb = fmaf(wb[k], row[fb + k], rb);
        }
        s_h[r][lane] = ra;
        s_h[r][lane + 32] = rb;
    }
    __syncthreads();
    // vertical pass per output pixel (same lanes / columns, warps own rows)
    const float swa = s_wx[lane][8], swb = s_wx[lane + 32][8];
    const bool ia = s_inx[lane], ib = s_inx[lane + 32];
    for (int y = wid; y < nyv; y += 8) {
        float wy[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) wy[j] = s_wy[y][j];
        const float sh = s_wy[y][8];
        const bool iy = s_iny[y];
        const int rbase = s_fy[y] - 3 - r0;
        float acc_a = 0.f, acc_b = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc_a = fmaf(wy[j], s_h[rbase + j][lane], acc_a);
            acc_b = fmaf(wy[j], s_h[rbase + j][lane + 32], acc_b);
        }
        const float vla = iy && ia ? fminf(fmaxf(__fdividef(acc_a, swa * sh), 0.f), 255.f) : 0.f;
        const float vlb = iy && ib ? fminf(fmaxf(__fdividef(acc_b, swb * sh), 0.f), 255.f) : 0.f;
        if (va) store_view<Tout, true>(v, out, pyr, x0 + lane, y0 + y, vla);
        if (vb) store_view<Tout, true>(v, out, pyr, x0 + lane + 32, y0 + y, vlb);
    }
}

template <class Tout>
__global__ void __launch_bounds__(256) k_lanczos_sep(const WarpView* __restrict__ views, int nviews, int tile0,
                                                     Tout* __restrict__ out, float* __restrict__ pyr) {
    __shared__ WarpView s_v;
    __shared__ SepShared s_sep;
    extern __shared__ __align__(16) float s_dyn[];
    const int tile = tile0 + blockIdx.x;
    if (threadIdx.x < 32) {
        const int k = find_view_warp(views, nviews, tile);
        if (threadIdx.x == 0) s_v = views[k];
    }
    __syncthreads();
    if (s_v.src_type == XA_PIX_U8)
        lanczos_sep_tile<uint8_t, Tout>(s_v, tile, out, pyr, s_sep, s_dyn);
    else
        lanczos_sep_tile<float, Tout>(s_v, tile, out, pyr, s_sep, s_dyn);
}

// ----------------------------------------------------------------- API blur/resize

// gaussian_blur passes (image.cpp:31-47), float accumulation in tap order.
__global__ void k_gauss_h(const float* __restrict__ in, float* __restrict__ out, int w, int h,
                          const float* __restrict__ k, int r) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    float acc = 0.f;
    for (int i = -r; i <= r; ++i)
        acc = fadd(acc, fmul(__ldg(k + i + r), __ldg(in + (size_t)y * w + clampi(x + i, 0, w - 1))));
    out[(size_t)y * w + x] = acc;
}

__global__ void k_gauss_v(const float* __restrict__ in, float* __restrict__ out, int w, int h,
                          const float* __restrict__ k, int r) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    float acc = 0.f;
    for (int i = -r; i <= r; ++i)
        acc = fadd(acc, fmul(__ldg(k + i + r), __ldg(in + (size_t)clampi(y + i, 0, h - 1) * w + x)));
    out[(size_t)y * w + x] = acc;
}

__global__ void k_resize(const float* __restrict__ in, int w, int h, float* __restrict__ out,
                         int nw, int nh) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= nw) return;
    out[(size_t)y * nw + x] = resize_px(in, w, h, (double)w / nw, (double)h / nh, x, y);
}

// ----------------------------------------------------------------- launchers

int launch_antialias(const BlurView* d_views, const BlurTap* d_taps, int nviews, const void* src,
                     int src_type, int w, int h, float* out, cudaStream_t st) {
    if (nviews <= 0) return 0;
    dim3 grid((w + 31) / 32, (h + 31) / 32, nviews), block(32, 8);
    if (src_type == XA_PIX_U8)
        k_antialias<uint8_t><<<grid, block, 0, st>>>(d_views, d_taps, (const uint8_t*)src, w, h, out);
    else
        k_antialias<float><<<grid, block, 0, st>>>(d_views, d_taps, (const float*)src, w, h, out);
    return 1;
}

int launch_blur_stencil(const BlurView* d_views, const BlurCell* d_cells, int nviews, int max_smem,
                        const void* src, int src_type, int w, int h, float* out, cudaStream_t st,
                        const BlurRun* d_runs, const float* d_rw, int runs_smem) {
    if (nviews <= 0) return 0;
    if (d_runs && runs_smem > 0) {
        dim3 grid((w + 63) / 64, (h + 63) / 64, nviews);
        const size_t smem = sizeof(float) * (size_t)runs_smem;
        if (src_type == XA_PIX_U8)
            k_blur_runs<uint8_t><<<grid, 256, smem, st>>>(d_views, d_runs, d_rw, (const uint8_t*)src, w, h, out);
        else
            k_blur_runs<float><<<grid, 256, smem, st>>>(d_views, d_runs, d_rw, (const float*)src, w, h, out);
        return 1;
    }
    dim3 grid((w + kBlurTW - 1) / kBlurTW, (h + kBlurTH - 1) / kBlurTH, nviews), block(32, 16);
    const size_t smem = sizeof(float) * (size_t)max_smem;
    if (src_type == XA_PIX_U8)
        k_blur_stencil<uint8_t><<<grid, block, smem, st>>>(d_views, d_cells, (const uint8_t*)src, w, h, out);
    else
        k_blur_stencil<float><<<grid, block, smem, st>>>(d_views, d_cells, (const float*)src, w, h, out);
    return 1;
}

int warp_init_attributes() {
    const int smem = kBlurSmemFloats * (int)sizeof(float);
    // k_blur_runs: up to (64 + 2 reach + 4) x (64 + 2 reach + 3) floats + run tables
    const int rsm = ((64 + 2 * kMaxBlurReach + 4) | 1) * (64 + 2 * kMaxBlurReach + 3) * (int)sizeof(float);
    if (cudaFuncSetAttribute(k_blur_runs<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, rsm) != cudaSuccess) return -1;
    if (cudaFuncSetAttribute(k_blur_runs<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, rsm) != cudaSuccess) return -1;
    if (cudaFuncSetAttribute(k_blur_stencil<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
    if (cudaFuncSetAttribute(k_blur_stencil<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
    const int ls = kLanczosSmemFloats * (int)sizeof(float);
    if (cudaFuncSetAttribute(k_lanczos_smem<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, ls) != cudaSuccess) return -1;
    if (cudaFuncSetAttribute(k_lanczos_sep<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemBytes) != cudaSuccess) return -1;
    if (cudaFuncSetAttribute(k_lanczos_sep<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemBytes) != cudaSuccess) return -1;
    if (cudaFuncSetAttribute(k_lanczos_smem<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, ls) != cudaSuccess) return -1;
    return 0;
}

int launch_warp(const WarpView* d_views, int nviews, int total_tiles, int mode, int out_type,
                void* out, float* pyr, int smem_floats, cudaStream_t st, const void* maps, int sep_tile0,
                int zpass) {
    const char* m = static_cast<const char*>(maps);
    if (nviews <= 0 || total_tiles <= 0) return 0;
    size_t smem = sizeof(float) * (size_t)smem_floats;
    // Lanczos: tiles [0, sep_tile0) general views, [sep_tile0, total) diagonal back-maps
    const int t0 = mode == 0 || sep_tile0 < 0 ? total_tiles : std::min(sep_tile0, total_tiles);
    if (zpass == 1) {  // zero background of the general Lanczos views only
        if (mode == 0 || t0 <= 0) return 0;
        if (out_type == XA_PIX_U8) k_lanczos_smem<uint8_t><<<t0, 256, 0, st>>>(d_views, nviews, (uint8_t*)out, pyr, m, 1);
        else k_lanczos_smem<float><<<t0, 256, 0, st>>>(d_views, nviews, (float*)out, pyr, m, 1);
        return 1;
    }
    int L = 0;
    if (out_type == XA_PIX_U8) {
        if (mode == 0) k_warp<uint8_t, 0><<<total_tiles, 256, 0, st>>>(d_views, nviews, (uint8_t*)out, pyr);
        else if (t0 > 0) k_lanczos_smem<uint8_t><<<t0, 256, smem, st>>>(d_views, nviews, (uint8_t*)out, pyr, m, zpass);
        if (mode != 0 && t0 < total_tiles)
            k_lanczos_sep<uint8_t><<<total_tiles - t0, 256, kSepSmemBytes, st>>>(d_views, nviews, t0, (uint8_t*)out, pyr), ++L;
    } else {
        if (mode == 0) k_warp<float, 0><<<total_tiles, 256, 0, st>>>(d_views, nviews, (float*)out, pyr);
        else if (t0 > 0) k_lanczos_smem<float><<<t0, 256, smem, st>>>(d_views, nviews, (float*)out, pyr, m, zpass);
        if (mode != 0 && t0 < total_tiles)
            k_lanczos_sep<float><<<total_tiles - t0, 256, kSepSmemBytes, st>>>(d_views, nviews, t0, (float*)out, pyr), ++L;
    }
    return 1 + L;
}

// synth_warp_case (eval.cpp:101-141): the evaluation harness's projective
// renderer. Per output pixel the framed homography's inverse maps (x, y) back
// with map_point_projective (geometry.cpp:84-88: numerators and w in double,
// source order, IEEE division); pixels outside [0, w-1] x [0, h-1] stay 0,
// the rest take sample_lanczos (a = 4, clamp-to-edge) clamped to [0, 255].
// U8 output applies the lround + clamp of save_image (image_io.cpp:17-20).
template <class Tout>
__global__ void __launch_bounds__(256) k_warp_projective(const float* __restrict__ src, int w, int h,
                                                         ProjView pv, Tout* __restrict__ out) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (x >= pv.W || y >= pv.H) return;
    const double* m = pv.back;
    const double xd = (double)x, yd = (double)y;
    const double wd = dadd(dadd(dmul(m[6], xd), dmul(m[7], yd)), m[8]);
    const double sx = __ddiv_rn(dadd(dadd(dmul(m[0], xd), dmul(m[1], yd)), m[2]), wd);
    const double sy = __ddiv_rn(dadd(dadd(dmul(m[3], xd), dmul(m[4], yd)), m[5]), wd);
    float val = 0.f;
    if (!(sx < 0.0 || sx > w - 1.0 || sy < 0.0 || sy > h - 1.0)) val = lanczos_px(src, w, h, sx, sy);
    out[(size_t)y * pv.W + x] = (Tout)quant_px<Tout>(val);
}

int launch_warp_projective(const float* src, int w, int h, const ProjView& pv, int out_type, void* out,
                           cudaStream_t st) {
    if (pv.W <= 0 || pv.H <= 0) return 0;
    dim3 grid((pv.W + 31) / 32, (pv.H + 7) / 8);
    if (out_type == XA_PIX_U8) k_warp_projective<uint8_t><<<grid, 256, 0, st>>>(src, w, h, pv, (uint8_t*)out);
    else k_warp_projective<float><<<grid, 256, 0, st>>>(src, w, h, pv, (float*)out);
    return 1;
}

int launch_gauss(const float* in, float* tmp, float* out, int w, int h, const float* d_k, int r,
                 cudaStream_t st) {
    dim3 grid((w + 127) / 128, h);
    k_gauss_h<<<grid, 128, 0, st>>>(in, tmp, w, h, d_k, r);
    k_gauss_v<<<grid, 128, 0, st>>>(tmp, out, w, h, d_k, r);
    return 2;
}

int launch_resize(const float* in, int w, int h, float* out, int nw, int nh, cudaStream_t st) {
    dim3 grid((nw + 127) / 128, nh);
    k_resize<<<grid, 128, 0, st>>>(in, w, h, out, nw, nh);
    return 1;
}

}  // namespace xa
