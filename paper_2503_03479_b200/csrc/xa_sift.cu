// xa_sift.cu — the fine stage's SIFT on sm_100a:
// detect_dog_keypoints (sift.cpp:290-358) and describe_gradient
// (sift.cpp:360-386).
//
// This file is compiled with --fmad=false: every float expression below is
// evaluated with one rounding per operation in the reference's order, so the
// Gaussian/DoG pyramid, the extremum test, the sub-pixel refinement and the
// descriptor arithmetic replay the reference exactly. What cannot be replayed
// bit for bit are the transcendentals: CUDA's double atan2/exp/pow (orientation
// histogram, keypoint scale) and float atan2f/expf/cosf/sinf (descriptor) may
// differ from glibc by an ulp. tests/test_gpu_sift.py states the resulting
// tolerance.
//
// Work split: the pyramid uses the exact resize / separable-blur kernels of
// xa_warp.cu plus k_halve / k_dog here; extrema are one thread per DoG pixel
// (appended with a warp-aggregated atomic); refinement + orientation run one
// thread per candidate, and descriptors one thread per keypoint, each in the
// reference's serial order (per-keypoint float accumulation order matters).
#include <math.h>

#include <algorithm>

#include "xa_common.cuh"
#include "xa_kernels.h"

namespace xa {

namespace {

__global__ void k_halve(const float* __restrict__ in, int w, float* __restrict__ out, int ow, int oh) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x < ow && y < oh) out[(size_t)y * ow + x] = in[(size_t)(2 * y) * w + 2 * x];
}

__global__ void k_dog(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ d,
                      size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        d[i] = b[i] - a[i];
}

// 26-neighbour strict extremum above the preliminary contrast threshold
// (sift.cpp:299-321), one thread per interior pixel of DoG layer `layer`.
__global__ void k_dog_extrema(const float* __restrict__ base, SiftImg prv, SiftImg cur, SiftImg nxt,
                              float prelim, int o, int layer, SiftCand* __restrict__ cand,
                              int* __restrict__ count, int cap) {
    const int c = 5 + blockIdx.x * blockDim.x + threadIdx.x, r = 5 + blockIdx.y;
    bool ext = false;
    if (c < cur.w - 5 && r < cur.h - 5) {
        const float* P = base + prv.off;
        const float* C = base + cur.off;
        const float* N = base + nxt.off;
        const int w = cur.w;
        const float v = C[(size_t)r * w + c];
        if (fabsf(v) > prelim) {
            bool is_max = true, is_min = true;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    const size_t i = (size_t)(r + dy) * w + (c + dx);
                    const float a = P[i], b = C[i], n = N[i];
                    if (a >= v || n >= v || (b >= v && (dx || dy))) is_max = false;
                    if (a <= v || n <= v || (b <= v && (dx || dy))) is_min = false;
                }
            ext = is_max || is_min;
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, ext);
    if (!m) return;
    int base_i = 0;
    if ((threadIdx.x & 31) == __ffs(m) - 1) base_i = atomicAdd(count, __popc(m));
    base_i = __shfl_sync(0xffffffffu, base_i, __ffs(m) - 1);
    if (ext) {
        const int p = base_i + __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
        if (p < cap) cand[p] = SiftCand{o, layer, r, c};
    }
}

__device__ __forceinline__ float at(const float* base, const SiftImg& im, int x, int y) {
    return base[im.off + (size_t)y * im.w + x];
}

__device__ __forceinline__ double det3(const double M[3][3]) {
    return M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
           M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
           M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
}

// refine_extremum (sift.cpp:136-195); dog = the octave's 5 DoG layers.
__device__ bool refine(const float* base, const SiftImg* dog, int& layer, int& r, int& c, float& xr,
                       float& xc, float& xs, float& contrast) {
    const float sc = 1.f / 255.f;
    for (int step = 0;; ++step) {
        if (step >= 5) return false;
        const SiftImg& cu = dog[layer];
        const SiftImg& pv = dog[layer - 1];
        const SiftImg& nx = dog[layer + 1];
        const float dx = (at(base, cu, c + 1, r) - at(base, cu, c - 1, r)) * 0.5f * sc;
        const float dy = (at(base, cu, c, r + 1) - at(base, cu, c, r - 1)) * 0.5f * sc;
        const float ds = (at(base, nx, c, r) - at(base, pv, c, r)) * 0.5f * sc;
        const float v2 = at(base, cu, c, r) * 2 * sc;
        const float dxx = (at(base, cu, c + 1, r) + at(base, cu, c - 1, r)) * sc - v2;
        const float dyy = (at(base, cu, c, r + 1) + at(base, cu, c, r - 1)) * sc - v2;
        const float dss = (at(base, nx, c, r) + at(base, pv, c, r)) * sc - v2;
        const float dxy = (at(base, cu, c + 1, r + 1) - at(base, cu, c - 1, r + 1) -
                           at(base, cu, c + 1, r - 1) + at(base, cu, c - 1, r - 1)) * 0.25f * sc;
        const float dxs = (at(base, nx, c + 1, r) - at(base, nx, c - 1, r) - at(base, pv, c + 1, r) +
                           at(base, pv, c - 1, r)) * 0.25f * sc;
        const float dys = (at(base, nx, c, r + 1) - at(base, nx, c, r - 1) - at(base, pv, c, r + 1) +
                           at(base, pv, c, r - 1)) * 0.25f * sc;
        const double H[3][3] = {{dxx, dxy, dxs}, {dxy, dyy, dys}, {dxs, dys, dss}};
        const double det = det3(H);
        if (fabs(det) < 1e-20) return false;
        double sol[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double M[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) M[a][b] = H[a][b];
            M[0][i] = -dx;
            M[1][i] = -dy;
            M[2][i] = -ds;
            sol[i] = det3(M) / det;
        }
        xc = (float)sol[0];
        xr = (float)sol[1];
        xs = (float)sol[2];
        if (fabsf(xc) < 0.5f && fabsf(xr) < 0.5f && fabsf(xs) < 0.5f) {
            contrast = at(base, cu, c, r) * sc + 0.5f * (dx * xc + dy * xr + ds * xs);
            const float tr = dxx + dyy;
            const float det2 = dxx * dyy - dxy * dxy;
            if (det2 <= 0) return false;
            if (tr * tr * 10.0 >= (10.0 + 1) * (10.0 + 1) * det2) return false;
            return fabsf(contrast) * 3 >= 0.03;
        }
        if (fabsf(xc) > 1e6f || fabsf(xr) > 1e6f || fabsf(xs) > 1e6f) return false;
        c += (int)lroundf(xc);
        r += (int)lroundf(xr);
        layer += (int)lroundf(xs);
        if (layer < 1 || layer > 3 || c < 5 || c >= cu.w - 5 || r < 5 || r >= cu.h - 5) return false;
    }
}

// orientation_histogram_peak (sift.cpp:93-125) for one candidate, one warp:
// the lanes compute the window samples (double gradient, angle and weight,
// as the reference) a chunk at a time into shared memory; then lane b owns
// raw bins b and b + 32 and scans the chunk in sample order, adding only its
// bins' values. Every bin therefore sums exactly the reference's sequence in
// the reference's order (skipped samples contribute nothing), so the raw and
// smoothed histograms equal the serial ones bit for bit.
constexpr int kOriChunk = 256;
constexpr int kKpWarps = 4;

struct OriScratch {
    float val[kOriChunk];
    int8_t bin[kOriChunk];
    float raw[36];
};

__device__ float ori_hist_warp(const float* base, const SiftImg& im, int x, int y, double s,
                               float* hist, OriScratch& sc) {
    const int lane = threadIdx.x & 31;
    const int radius = (int)round(4.5 * s);
    const double wf = -1.0 / (2.0 * (1.5 * s) * (1.5 * s));
    const float* p = base + im.off;
    const int side = 2 * radius + 1, nsamp = side * side;
    float acc0 = 0.f, acc1 = 0.f;  // raw[lane], raw[lane + 32]
    for (int c0 = 0; c0 < nsamp; c0 += kOriChunk) {
        for (int k = lane; k < kOriChunk; k += 32) {
            const int s_i = c0 + k;
            int bin = -1;
            float v = 0.f;
            if (s_i < nsamp) {
                const int dy = s_i / side - radius, dx = s_i - (s_i / side) * side - radius;
                const int py = y + dy, px = x + dx;
                if (py > 0 && py < im.h - 1 && px > 0 && px < im.w - 1) {
                    const double gx = p[(size_t)py * im.w + px + 1] - p[(size_t)py * im.w + px - 1];
                    const double gy = p[(size_t)(py - 1) * im.w + px] - p[(size_t)(py + 1) * im.w + px];
                    const double mag = sqrt(gx * gx + gy * gy);
                    const double ang = atan2(gy, gx);
                    const double w = exp(wf * (dx * dx + dy * dy));
                    bin = (int)round(36 * (ang + M_PI) / (2 * M_PI));
                    if (bin >= 36) bin -= 36;
                    if (bin < 0) bin += 36;
                    v = (float)(w * mag);
                }
            }
            sc.val[k] = v;
            sc.bin[k] = (int8_t)bin;
        }
        __syncwarp();
        const int n = min(kOriChunk, nsamp - c0);
        for (int k = 0; k < n; ++k) {
            const int b = sc.bin[k];
            const float v = sc.val[k];
            if (b == lane) acc0 += v;
            if (b == lane + 32) acc1 += v;
        }
        __syncwarp();
    }
    sc.raw[lane] = acc0;
    if (lane < 4) sc.raw[lane + 32] = acc1;
    __syncwarp();
    float peak = 0.f;
    const float* raw = sc.raw;
    for (int i = 0; i < 36; ++i) {
        hist[i] = (raw[(i - 2 + 36) % 36] + raw[(i + 2) % 36]) * (1.f / 16) +
                  (raw[(i - 1 + 36) % 36] + raw[(i + 1) % 36]) * (4.f / 16) + raw[i] * (6.f / 16);
        peak = peak < hist[i] ? hist[i] : peak;
    }
    return peak;
}

// One warp per candidate: refinement (every lane, identical), keypoint
// fields, orientation peaks (sift.cpp:323-354); lane 0 appends the surviving
// orientations to `out`.
__global__ void __launch_bounds__(32 * kKpWarps) k_sift_keypoints(const float* __restrict__ base,
                                                                 const SiftImg* __restrict__ gauss,
                                                                 const SiftImg* __restrict__ dog,
                                                                 const SiftCand* __restrict__ cand,
                                                                 const int* __restrict__ ncand_p,
                                                                 int cand_cap, xa_kp* __restrict__ out,
                                                                 int* __restrict__ nout, int out_cap) {
    __shared__ OriScratch s_sc[kKpWarps];
    const int wid = threadIdx.x >> 5;
    const int i = blockIdx.x * kKpWarps + wid;
    if (i >= min(*ncand_p, cand_cap)) return;
    const SiftCand cd = cand[i];
    const int o = cd.o;
    int ll = cd.layer, rr = cd.r, cc = cd.c;
    float xr, xc, xs, contrast;
    if (!refine(base, dog + 5 * o, ll, rr, cc, xr, xc, xs, contrast)) return;
    const double scl = 1.6 * pow(2.0, (ll + xs) / 3);
    const double of = pow(2.0, o);
    xa_kp kp;
    kp.x = (float)((cc + xc) * of * 0.5);
    kp.y = (float)((rr + xr) * of * 0.5);
    kp.octave_scale = (float)(scl * of * 0.5);
    kp.response = fabsf(contrast);
    float hist[36];
    const float peak = ori_hist_warp(base, gauss[6 * o + ll], cc, rr, scl, hist, s_sc[wid]);
    if ((threadIdx.x & 31) || peak <= 0) return;
    const float thr = peak * 0.8f;
    for (int bin = 0; bin < 36; ++bin) {
        const int l = (bin - 1 + 36) % 36, rb = (bin + 1) % 36;
        if (hist[bin] < thr || hist[bin] <= hist[l] || hist[bin] <= hist[rb]) continue;
        float fbin = bin + 0.5f * (hist[l] - hist[rb]) / (hist[l] - 2 * hist[bin] + hist[rb]);
        if (fbin < 0) fbin += 36;
        if (fbin >= 36) fbin -= 36;
        kp.orientation = (float)(fbin * 2 * M_PI / 36 - M_PI);
        const int p = atomicAdd(nout, 1);
        if (p < out_cap) out[p] = kp;
    }
}

// append_descriptor (sift.cpp:197-277), one warp per keypoint; the host
// resolved the pyramid image and the border filter (sift.cpp:367-379). The
// lanes stride over the window samples and accumulate into private
// histograms in shared memory (only the 4x4 cells the descriptor keeps; the
// reference's border cells are never read), which are then summed in lane
// order: deterministic, and equal to the reference's serial sums up to float
// reassociation (far below the glibc/CUDA atan2f/expf ulp differences).
constexpr int kDescWarps = 2;
constexpr int kHistStride = 16 * 10 + 1;  // 16 cells x 10 orientation slots, +1 against bank conflicts

__global__ void __launch_bounds__(32 * kDescWarps) k_sift_describe(const float* __restrict__ base,
                                                                  const SiftImg* __restrict__ gauss,
                                                                  const SiftJob* __restrict__ jobs, int n,
                                                                  float* __restrict__ desc) {
    extern __shared__ float s_hist[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int k = blockIdx.x * kDescWarps + wid;
    if (k >= n) return;
    float* hist = s_hist + (size_t)wid * 32 * kHistStride;
    float* mine = hist + lane * kHistStride;
    for (int i = 0; i < 160; ++i) mine[i] = 0.f;
    const SiftJob J = jobs[k];
    const SiftImg im = gauss[J.img];
    const float* p = base + im.off;
    // glibc cosf/sinf differ from the correctly rounded value by an ulp on
    // ~0.2% of angles (tools/gen_trig_table.c); here that is within tolerance
    const float cos_t = (float)cos((double)J.angle), sin_t = (float)sin((double)J.angle);
    const float bpr = 8 / (2 * (float)M_PI);
    const float es = -1.f / (4 * 4 * 0.5f);
    const float hw = 3.f * (float)J.scl;
    int radius = (int)roundf(hw * sqrtf(2.f) * (4 + 1) * 0.5f);
    radius = min(radius, (int)sqrt((double)im.w * im.w + (double)im.h * im.h));
    const float ct = cos_t / hw, st = sin_t / hw;
    const int icol = (int)roundf(J.col), irow = (int)roundf(J.row);
    const int side = 2 * radius + 1, nsamp = side * side;
    int i = lane / side, j = lane - (lane / side) * side;  // sample s = i * side + j
    const int di = 32 / side, dj = 32 - di * side;
    for (int s = lane; s < nsamp; s += 32) {
        const int ii = i - radius, jj = j - radius;
        j += dj;
        i += di;
        if (j >= side) {
            j -= side;
            ++i;
        }
        const float c_rot = jj * ct - ii * st;
        const float r_rot = jj * st + ii * ct;
        const float rbin = r_rot + 4 / 2 - 0.5f;
        const float cbin = c_rot + 4 / 2 - 0.5f;
        const int py = irow + ii, px = icol + jj;
        if (rbin <= -1 || rbin >= 4 || cbin <= -1 || cbin >= 4 || px <= 0 || px >= im.w - 1 ||
            py <= 0 || py >= im.h - 1)
            continue;
        const float gx = p[(size_t)py * im.w + px + 1] - p[(size_t)py * im.w + px - 1];
        const float gy = p[(size_t)(py - 1) * im.w + px] - p[(size_t)(py + 1) * im.w + px];
        const float mag = sqrtf(gx * gx + gy * gy);
        float theta = atan2f(gy, gx) - J.angle;
        while (theta < 0) theta += 2 * (float)M_PI;
        while (theta >= 2 * (float)M_PI) theta -= 2 * (float)M_PI;
        const float obin = theta * bpr;
        const float w = expf((c_rot * c_rot + r_rot * r_rot) * es) * mag;
        const int r0 = (int)floorf(rbin), c0 = (int)floorf(cbin);
        int o0 = (int)floorf(obin);
        const float rb = rbin - r0, cb = cbin - c0, ob = obin - o0;
        if (o0 >= 8) o0 -= 8;
#pragma unroll
        for (int dr = 0; dr <= 1; ++dr) {
            const int rr = r0 + dr;  // kept cells: rr, cc in 0..3 (reference rows 1..4)
            if (rr < 0 || rr >= 4) continue;
            const float wr = w * (dr ? rb : 1 - rb);
#pragma unroll
            for (int dc = 0; dc <= 1; ++dc) {
                const int cc = c0 + dc;
                if (cc < 0 || cc >= 4) continue;
                const float wc = wr * (dc ? cb : 1 - cb);
                float* h = mine + (rr * 4 + cc) * 10 + o0;
                h[0] += wc * (1 - ob);
                h[1] += wc * ob;
            }
        }
    }
    __syncwarp();
    // lane-ordered sum of the 32 private histograms into lane 0's copy
    for (int b = lane; b < 160; b += 32) {
        float t = hist[b];
        for (int l = 1; l < 32; ++l) t += hist[l * kHistStride + b];
        hist[b] = t;
    }
    __syncwarp();
    float* v = desc + (size_t)k * 128;
    if (lane == 0) {
        double norm = 0;
        for (int c = 0; c < 16; ++c) {
            float* cell = hist + c * 10;
            cell[0] += cell[8];
            cell[1] += cell[9];
            for (int q = 0; q < 8; ++q) norm += (double)cell[q] * cell[q];
        }
        const float thr = (float)sqrt(norm) * 0.2f;
        norm = 0;
        for (int c = 0; c < 16; ++c)
            for (int q = 0; q < 8; ++q) {
                float* x = hist + c * 10 + q;
                *x = thr < *x ? thr : *x;
                norm += (double)*x * *x;
            }
        const double sn = sqrt(norm);
        hist[kHistStride - 1] = 512.f / (float)(sn < 1e-12 ? 1e-12 : sn);
    }
    __syncwarp();
    const float scale = hist[kHistStride - 1];
    for (int q = lane; q < 128; q += 32) v[q] = hist[(q >> 3) * 10 + (q & 7)] * scale;
}

}  // namespace

int launch_halve(const float* in, int w, float* out, int ow, int oh, cudaStream_t st) {
    dim3 grid((ow + 127) / 128, oh);
    k_halve<<<grid, 128, 0, st>>>(in, w, out, ow, oh);
    return 1;
}

int launch_dog(const float* a, const float* b, float* d, size_t n, cudaStream_t st) {
    const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    k_dog<<<grid, 256, 0, st>>>(a, b, d, n);
    return 1;
}

int launch_dog_extrema(const float* base, SiftImg prv, SiftImg cur, SiftImg nxt, float prelim, int o,
                       int layer, SiftCand* cand, int* count, int cap, cudaStream_t st) {
    if (cur.w <= 10 || cur.h <= 10) return 0;
    dim3 grid((cur.w - 10 + 127) / 128, cur.h - 10);
    k_dog_extrema<<<grid, 128, 0, st>>>(base, prv, cur, nxt, prelim, o, layer, cand, count, cap);
    return 1;
}

int launch_sift_keypoints(const float* base, const SiftImg* gauss, const SiftImg* dog,
                          const SiftCand* cand, const int* ncand, int cand_cap, xa_kp* out, int* nout,
                          int out_cap, cudaStream_t st) {
    if (cand_cap <= 0) return 0;
    k_sift_keypoints<<<(cand_cap + kKpWarps - 1) / kKpWarps, 32 * kKpWarps, 0, st>>>(
        base, gauss, dog, cand, ncand, cand_cap, out, nout, out_cap);
    return 1;
}

int launch_sift_describe(const float* base, const SiftImg* gauss, const SiftJob* jobs, int n,
                         float* desc, cudaStream_t st) {
    if (n <= 0) return 0;
    const size_t smem = sizeof(float) * kDescWarps * 32 * kHistStride;
    k_sift_describe<<<(n + kDescWarps - 1) / kDescWarps, 32 * kDescWarps, smem, st>>>(base, gauss, jobs, n, desc);
    return 1;
}

}  // namespace xa
