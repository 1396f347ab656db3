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

// Directional Gaussian along (cos phi, -sin phi) (warp.cpp:128-158). The tap
// geometry (integer offset + bilinear fraction) is the same for every pixel
// because pixel coordinates are integers, so the host precomputes it per view.
// Accumulation is double (DFMA) like the reference's double acc; the bilinear
// sample is the reference's float expression with exact rounding.
template <class Tin>
__device__ __forceinline__ float bilerp_tap(const Tin* src, int w, int h, int x, int y,
                                            const BlurTap& t) {
    const int x0 = x + t.ox, y0 = y + t.oy;
    const int xa = clampi(x0, 0, w - 1), xb = clampi(x0 + 1, 0, w - 1);
    const int ya = clampi(y0, 0, h - 1), yb = clampi(y0 + 1, 0, h - 1);
    const float v00 = ld_px(src, (size_t)ya * w + xa), v10 = ld_px(src, (size_t)ya * w + xb);
    const float v01 = ld_px(src, (size_t)yb * w + xa), v11 = ld_px(src, (size_t)yb * w + xb);
    const float iwx = fsub(1.f, t.wx), iwy = fsub(1.f, t.wy);
    const float top = fadd(fmul(iwx, v00), fmul(t.wx, v10));
    const float bot = fadd(fmul(iwx, v01), fmul(t.wx, v11));
    return fadd(fmul(iwy, top), fmul(t.wy, bot));
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
                acc = fma(s_taps[i].k, (double)ld_px(src, row + clampi(x + s_taps[i].ox, 0, w - 1)), acc);
        } else {
            for (int i = 0; i < v.ntaps; ++i)
                acc = fma(s_taps[i].k, (double)bilerp_tap(src, w, h, x, y, s_taps[i]), acc);
        }
        o[(size_t)y * w + x] = (float)acc;
    }
}

// ----------------------------------------------------------------- resample

__device__ __forceinline__ int find_view(const WarpView* __restrict__ views, int n, int tile) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (views[mid].tile_start <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Lanczos-4 weights for the 8 taps i = -3..4 at fractional offset r in [0,1):
// L(i - r) up to a common factor (cancelled by the acc/wsum normalisation of
// sample_lanczos, warp.cpp:62-84). sin(pi(i-r)) = -(-1)^i sin(pi r) and
// sin(pi(i-r)/4) by angle addition, so one sincospi pair per axis.
__device__ __forceinline__ void lanczos_w(float r, float* wt) {
    float s1, c1, s4, c4;
    sincospif(r, &s1, &c1);
    sincospif(0.25f * r, &s4, &c4);
    const float k = 0.70710678118654752f;
    // sin(pi*i/4), cos(pi*i/4) for i = -3..4
    const float si[8] = {-k, -1.f, -k, 0.f, k, 1.f, k, 0.f};
    const float ci[8] = {-k, 0.f, k, 1.f, k, 0.f, -k, -1.f};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = j - 3;
        const float t = (float)i - r;
        if (t == 0.f) {
            wt[j] = 2.4674011002723395f;  // pi^2/4: L(0)=1 in these units
        } else {
            const float a = (i & 1) ? s1 : -s1;
            const float b = si[j] * c4 - ci[j] * s4;
            wt[j] = a * b / (t * t);
        }
    }
}

template <class Tin>
__device__ __forceinline__ float lanczos_px(const Tin* src, int w, int h, double sx, double sy) {
    const double fxd = floor(sx), fyd = floor(sy);
    const int fx = (int)fxd, fy = (int)fyd;
    float wx[8], wy[8];
    lanczos_w((float)(sx - fxd), wx);
    lanczos_w((float)(sy - fyd), wy);
    int xs[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) xs[i] = clampi(fx + i - 3, 0, w - 1);
    float acc = 0.f, sw = 0.f, sh = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) sw += wx[i];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const size_t row = (size_t)clampi(fy + j - 3, 0, h - 1) * w;
        float rs = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) rs = fmaf(wx[i], ld_px(src, row + xs[i]), rs);
        acc = fmaf(wy[j], rs, acc);
        sh += wy[j];
    }
    float v = acc / (sw * sh);
    return fminf(fmaxf(v, 0.f), 255.f);
}

template <class Tout>
__device__ __forceinline__ void store_px(Tout* p, size_t i, float v);
template <>
__device__ __forceinline__ void store_px<float>(float* p, size_t i, float v) { p[i] = v; }
template <>
__device__ __forceinline__ void store_px<uint8_t>(uint8_t* p, size_t i, float v) {
    // lround + clamp quantisation (image_io.cpp:17-20)
    p[i] = (uint8_t)fminf(fmaxf(roundf(v), 0.f), 255.f);
}

template <class Tin, class Tout, int MODE>
__device__ __forceinline__ void warp_tile(const WarpView& v, int tile, Tout* out) {
    const int t = tile - v.tile_start;
    const int tx = t % v.tiles_x, ty = t / v.tiles_x;
    const int x = tx * 32 + (threadIdx.x & 31);
    const int yb = ty * 32 + (threadIdx.x >> 5);
    if (x >= v.W) return;
    const Tin* src = static_cast<const Tin*>(v.src);
    Tout* o = out + v.out_off;
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
        store_px(o, (size_t)y * v.W + x, val);
    }
}

template <class Tout, int MODE>
__global__ void __launch_bounds__(256) k_warp(const WarpView* __restrict__ views, int nviews,
                                              Tout* __restrict__ out) {
    __shared__ int s_view;
    if (threadIdx.x == 0) s_view = find_view(views, nviews, blockIdx.x);
    __syncthreads();
    const WarpView v = views[s_view];
    if (v.src_type == XA_PIX_U8)
        warp_tile<uint8_t, Tout, MODE>(v, blockIdx.x, out);
    else
        warp_tile<float, Tout, MODE>(v, blockIdx.x, out);
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

int launch_warp(const WarpView* d_views, int nviews, int total_tiles, int mode, int out_type,
                void* out, cudaStream_t st) {
    if (nviews <= 0 || total_tiles <= 0) return 0;
    if (out_type == XA_PIX_U8) {
        if (mode == 0) k_warp<uint8_t, 0><<<total_tiles, 256, 0, st>>>(d_views, nviews, (uint8_t*)out);
        else k_warp<uint8_t, 1><<<total_tiles, 256, 0, st>>>(d_views, nviews, (uint8_t*)out);
    } else {
        if (mode == 0) k_warp<float, 0><<<total_tiles, 256, 0, st>>>(d_views, nviews, (float*)out);
        else k_warp<float, 1><<<total_tiles, 256, 0, st>>>(d_views, nviews, (float*)out);
    }
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
