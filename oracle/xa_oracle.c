/* oracle/xa_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU parity checker.
 *
 * A plain-C restatement of the reference algorithm for the coarse hot path.
 * Every function cites the reference file:line whose arithmetic it follows
 * (paths relative to /root/reference/proj). Arithmetic is IEEE-754 in source
 * order: this file must be compiled with -ffp-contract=off (oracle/Makefile),
 * matching the flags the reference oracle is built with.
 *
 * Pinned by tests/test_oracle.py against oracle/_ref/libxaref.so (the
 * reference compiled from its own sources) and tests/golden/ fixtures.
 * Known, documented divergence: the final keypoint sort uses qsort where the
 * reference uses std::sort; both are unstable, so keypoints that tie on all
 * three keys (response, y, x) may come out in a different relative order.
 */
#define _GNU_SOURCE
#include "xa_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
static int g_threads = 0;

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}

const char* orc_last_error(void) { return g_err; }
void orc_free(void* p) { free(p); }
const char* orc_kind(void) { return "port"; }
int orc_set_threads(int n) {
    g_threads = n;
    return 0;
}

/* ------------------------------------------------------------------ pattern */

static const int8_t k_pattern[1024] = {
#include "../paper_2503_03479_b200/csrc/orb_pattern.inc"
};

/* FNV-1a over little-endian int32 quadruples (orb_pattern.cpp:270-285). */
uint64_t orc_pattern_checksum(void) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int i = 0; i < 1024; ++i) {
        const int32_t v = k_pattern[i];
        for (int b = 0; b < 4; ++b) {
            h ^= (uint8_t)(v >> (8 * b));
            h *= 0x100000001b3ull;
        }
    }
    return h;
}

void orc_pattern(int8_t* out) { memcpy(out, k_pattern, 1024); }

/* ------------------------------------------------------------------ raster */

typedef struct {
    int w, h;
    float* d;
} img_t;

static img_t img_new(int w, int h, float fill) {
    img_t r = {w, h, (float*)malloc(sizeof(float) * (size_t)(w > 0 ? w : 1) * (h > 0 ? h : 1))};
    for (size_t i = 0; i < (size_t)w * h; ++i) r.d[i] = fill;
    return r;
}

static img_t img_wrap(const float* p, int w, int h) {
    img_t r = {w, h, (float*)p};
    return r;
}

static inline float px(const img_t* im, int x, int y) { return im->d[(size_t)y * im->w + x]; }

/* clamp-to-edge fetch (image.hpp:25-31) */
static inline float pxc(const img_t* im, int x, int y) {
    if (x < 0) x = 0;
    if (x >= im->w) x = im->w - 1;
    if (y < 0) y = 0;
    if (y >= im->h) y = im->h - 1;
    return im->d[(size_t)y * im->w + x];
}

/* normalised float taps; weights from double exp (image.cpp:10-21) */
static int blur_taps(double sigma, float* k) {
    int r = (int)ceil(3.0 * sigma);
    if (r < 1) r = 1;
    double sum = 0;
    for (int i = -r; i <= r; ++i) {
        const double v = exp(-0.5 * i * i / (sigma * sigma));
        k[i + r] = (float)v;
        sum += v;
    }
    for (int i = 0; i < 2 * r + 1; ++i) k[i] = (float)(k[i] / sum);
    return r;
}

/* separable blur, float accumulation, H then V (image.cpp:25-49) */
static void blur_into(const img_t* src, double sigma, img_t* out) {
    if (sigma <= 0) {
        memcpy(out->d, src->d, sizeof(float) * (size_t)src->w * src->h);
        return;
    }
    float k[512];
    const int r = blur_taps(sigma, k);
    img_t tmp = img_new(src->w, src->h, 0.f);
    for (int y = 0; y < src->h; ++y)
        for (int x = 0; x < src->w; ++x) {
            float acc = 0;
            for (int i = -r; i <= r; ++i) acc += k[i + r] * pxc(src, x + i, y);
            tmp.d[(size_t)y * src->w + x] = acc;
        }
    for (int y = 0; y < src->h; ++y)
        for (int x = 0; x < src->w; ++x) {
            float acc = 0;
            for (int i = -r; i <= r; ++i) acc += k[i + r] * pxc(&tmp, x, y + i);
            out->d[(size_t)y * src->w + x] = acc;
        }
    free(tmp.d);
}

/* half-pixel bilinear resize (image.cpp:51-70) */
static void resize_into(const img_t* src, int nw, int nh, img_t* out) {
    const double sx = (double)src->w / nw, sy = (double)src->h / nh;
    for (int y = 0; y < nh; ++y) {
        const double fy = (y + 0.5) * sy - 0.5;
        const int y0 = (int)floor(fy);
        const float wy = (float)(fy - y0);
        for (int x = 0; x < nw; ++x) {
            const double fx = (x + 0.5) * sx - 0.5;
            const int x0 = (int)floor(fx);
            const float wx = (float)(fx - x0);
            const float v00 = pxc(src, x0, y0), v10 = pxc(src, x0 + 1, y0);
            const float v01 = pxc(src, x0, y0 + 1), v11 = pxc(src, x0 + 1, y0 + 1);
            out->d[(size_t)y * nw + x] =
                (1 - wy) * ((1 - wx) * v00 + wx * v10) + wy * ((1 - wx) * v01 + wx * v11);
        }
    }
}

int orc_gaussian_blur(const float* p, int w, int h, double sigma, float* out) {
    img_t s = img_wrap(p, w, h), o = img_wrap(out, w, h);
    blur_into(&s, sigma, &o);
    return 0;
}

int orc_resize_bilinear(const float* p, int w, int h, int nw, int nh, float* out) {
    img_t s = img_wrap(p, w, h), o = img_wrap(out, nw, nh);
    resize_into(&s, nw, nh, &o);
    return 0;
}

/* ---------------------------------------------------------------- geometry */

typedef struct {
    double m[9];
} mat_t;

static mat_t mat_eye(void) {
    mat_t r = {{1, 0, 0, 0, 1, 0, 0, 0, 1}};
    return r;
}

static mat_t mat_shift(double tx, double ty) {
    mat_t r = mat_eye();
    r.m[2] = tx;
    r.m[5] = ty;
    return r;
}

/* geometry.cpp:18-26 */
static mat_t mat_rot(double a) {
    mat_t r = mat_eye();
    const double c = cos(a), s = sin(a);
    r.m[0] = c;
    r.m[1] = -s;
    r.m[3] = s;
    r.m[4] = c;
    return r;
}

static mat_t mat_scale(double s) {
    mat_t r = mat_eye();
    r.m[0] = s;
    r.m[4] = s;
    return r;
}

/* row-by-column, accumulator starts at +0 (geometry.cpp:35-44) */
static mat_t mat_mul(const mat_t* a, const mat_t* b) {
    mat_t r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0;
            for (int k = 0; k < 3; ++k) acc += a->m[i * 3 + k] * b->m[k * 3 + j];
            r.m[i * 3 + j] = acc;
        }
    return r;
}

static void params_of(const double* p, double* psi, double* t, double* phi, double* s, double* tx,
                      double* ty) {
    *psi = p[0];
    *t = p[1];
    *phi = p[2];
    *s = p[3];
    *tx = p[4];
    *ty = p[5];
}

/* T * R(psi) * S(s) * diag(tfac, 1) * R(phi), left-associated (geometry.cpp:42-58) */
static mat_t compose(const double* p, int simulate) {
    double psi, t, phi, s, tx, ty;
    params_of(p, &psi, &t, &phi, &s, &tx, &ty);
    mat_t tau = mat_eye();
    tau.m[0] = simulate ? 1.0 / t : t;
    mat_t a = mat_shift(tx, ty), b = mat_rot(psi), c = mat_scale(s), e = mat_rot(phi);
    mat_t r = mat_mul(&a, &b);
    r = mat_mul(&r, &c);
    r = mat_mul(&r, &tau);
    return mat_mul(&r, &e);
}

int orc_simulation_from_params(const double* p, double* m) {
    if (p[1] < 1.0) return fail("simulation_from_params: tilt must be >= 1");
    if (p[3] <= 0.0) return fail("simulation_from_params: scale must be > 0");
    mat_t r = compose(p, 1);
    memcpy(m, r.m, sizeof r.m);
    return 0;
}

int orc_affine_from_params(const double* p, double* m) {
    if (p[1] < 1.0) return fail("affine_from_params: tilt must be >= 1");
    if (p[3] <= 0.0) return fail("affine_from_params: scale must be > 0");
    mat_t r = compose(p, 0);
    memcpy(m, r.m, sizeof r.m);
    return 0;
}

/* cofactor inverse (geometry.cpp:65-78) */
static int mat_inv(const mat_t* a, mat_t* r) {
    const double* m = a->m;
    const double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                       m[2] * (m[3] * m[7] - m[4] * m[6]);
    if (fabs(det) < 1e-14) return fail("invert: singular matrix");
    r->m[0] = (m[4] * m[8] - m[5] * m[7]) / det;
    r->m[1] = (m[2] * m[7] - m[1] * m[8]) / det;
    r->m[2] = (m[1] * m[5] - m[2] * m[4]) / det;
    r->m[3] = (m[5] * m[6] - m[3] * m[8]) / det;
    r->m[4] = (m[0] * m[8] - m[2] * m[6]) / det;
    r->m[5] = (m[2] * m[3] - m[0] * m[5]) / det;
    r->m[6] = (m[3] * m[7] - m[4] * m[6]) / det;
    r->m[7] = (m[1] * m[6] - m[0] * m[7]) / det;
    r->m[8] = (m[0] * m[4] - m[1] * m[3]) / det;
    return 0;
}

int orc_invert(const double* m, double* out) {
    mat_t a, r;
    memcpy(a.m, m, sizeof a.m);
    if (mat_inv(&a, &r)) return -1;
    memcpy(out, r.m, sizeof r.m);
    return 0;
}

/* geometry.cpp:80-82 */
static inline void map_pt(const mat_t* m, double x, double y, double* ox, double* oy) {
    *ox = m->m[0] * x + m->m[1] * y + m->m[2];
    *oy = m->m[3] * x + m->m[4] * y + m->m[5];
}

/* viewpoint grid (geometry.cpp:90-112) */
int orc_build_grid(double a, int n, double b_deg, double delta_s, double** params, int* count) {
    if (a <= 1.0) return fail("build_param_grid: a must be > 1");
    if (n < 0) return fail("build_param_grid: n must be >= 0");
    int cap = 64, cnt = 0;
    double* out = (double*)malloc(sizeof(double) * 6 * cap);
    for (int k = 0; k <= n; ++k) {
        const double t = pow(a, k);
        const double s = 1.0 + k * delta_s;
        const double step = (k == 0) ? 0.0 : b_deg / t;
        for (int j = 0; k == 0 ? j < 1 : j * step < 180.0 - 1e-9; ++j) {
            if (cnt == cap) {
                cap *= 2;
                out = (double*)realloc(out, sizeof(double) * 6 * cap);
            }
            double* e = out + 6 * cnt++;
            e[0] = 0.0;
            e[1] = t;
            e[2] = (k == 0) ? 0.0 : j * step * M_PI / 180.0;
            e[3] = s;
            e[4] = 0.0;
            e[5] = 0.0;
        }
    }
    *params = out;
    *count = cnt;
    return 0;
}

/* -------------------------------------------------------------------- warp */

/* half-pixel conjugation (warp.cpp:13-15) */
static mat_t center_adj(const mat_t* m) {
    mat_t a = mat_shift(-0.5, -0.5), b = mat_shift(0.5, 0.5);
    mat_t r = mat_mul(&a, m);
    return mat_mul(&r, &b);
}

/* output bbox of the mapped corners with integer snapping (warp.cpp:24-42) */
static void frame_of(const mat_t* fwd, int w, int h, int* W, int* H, double* tx, double* ty) {
    const double cx[4] = {0.0, (double)(w - 1), 0.0, (double)(w - 1)};
    const double cy[4] = {0.0, 0.0, (double)(h - 1), (double)(h - 1)};
    double minx = 1e30, miny = 1e30, maxx = -1e30, maxy = -1e30;
    for (int i = 0; i < 4; ++i) {
        double x, y;
        map_pt(fwd, cx[i], cy[i], &x, &y);
        if (x < minx) minx = x;
        if (maxx < x) maxx = x;
        if (y < miny) miny = y;
        if (maxy < y) maxy = y;
    }
    *tx = -floor(minx + 1e-9);
    *ty = -floor(miny + 1e-9);
    *W = (int)(ceil(maxx - 1e-9) + *tx) + 1;
    *H = (int)(ceil(maxy - 1e-9) + *ty) + 1;
}

/* warp.cpp:55-60 */
double orc_lanczos_kernel(double x, int a) {
    if (x <= -a || x >= a) return 0.0;
    if (x == 0.0) return 1.0;
    const double t = M_PI * x;
    return (sin(t) / t) * (sin(t / a) * a / t);
}

/* row sums then weighted column sum, normalised (warp.cpp:62-84) */
static double lanczos_at(const img_t* im, double x, double y, int a) {
    const int fx = (int)floor(x), fy = (int)floor(y);
    const double rx = x - fx, ry = y - fy;
    double wx[16], wy[16];
    for (int i = -a + 1; i <= a; ++i) {
        wx[i + a - 1] = orc_lanczos_kernel(i - rx, a);
        wy[i + a - 1] = orc_lanczos_kernel(i - ry, a);
    }
    double acc = 0, wsum = 0;
    for (int j = 0; j < 2 * a; ++j) {
        const int yy = fy + j - a + 1;
        double row = 0, rw = 0;
        for (int i = 0; i < 2 * a; ++i) {
            row += wx[i] * pxc(im, fx + i - a + 1, yy);
            rw += wx[i];
        }
        acc += wy[j] * row;
        wsum += wy[j] * rw;
    }
    return acc / wsum;
}

double orc_sample_lanczos(const float* p, int w, int h, double x, double y, int a) {
    img_t im = img_wrap(p, w, h);
    return lanczos_at(&im, x, y, a);
}

/* warp_nearest (warp.cpp:86-105) and warp_lanczos (warp.cpp:107-126) */
int orc_warp(int mode, const float* p, int w, int h, const double* m, int a, float** out, int* W,
             int* H, double* tx, double* ty, double* fwd) {
    mat_t mm, adj, inv, f, back;
    memcpy(mm.m, m, sizeof mm.m);
    adj = center_adj(&mm);
    if (mode == 0 && mat_inv(&adj, &inv)) return -1;
    frame_of(&adj, w, h, W, H, tx, ty);
    mat_t sh = mat_shift(*tx, *ty);
    f = mat_mul(&sh, &adj);
    memcpy(fwd, f.m, sizeof f.m);
    if (mat_inv(&f, &back)) return -1;
    img_t src = img_wrap(p, w, h);
    img_t o = img_new(*W, *H, 0.f);
    for (int y = 0; y < *H; ++y)
        for (int x = 0; x < *W; ++x) {
            double sx, sy;
            map_pt(&back, x, y, &sx, &sy);
            if (mode == 0) {
                const int ix = (int)lround(sx), iy = (int)lround(sy);
                if (ix >= 0 && ix < w && iy >= 0 && iy < h) o.d[(size_t)y * *W + x] = px(&src, ix, iy);
            } else {
                if (sx < 0.0 || sx > w - 1.0 || sy < 0.0 || sy > h - 1.0) continue;
                double v = lanczos_at(&src, sx, sy, a);
                v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
                o.d[(size_t)y * *W + x] = (float)v;
            }
        }
    *out = o.d;
    return 0;
}

/* map_point_projective (geometry.cpp:84-88) */
static void map_pt_proj(const mat_t* m, double x, double y, double* ox, double* oy) {
    const double w = m->m[6] * x + m->m[7] * y + m->m[8];
    *ox = (m->m[0] * x + m->m[1] * y + m->m[2]) / w;
    *oy = (m->m[3] * x + m->m[4] * y + m->m[5]) / w;
}

/* synth_warp_case (eval.cpp:101-141): half-pixel framing of the homography
   (eval.cpp:104-128), inverse (:129-134), then per output pixel a projective
   back-map and sample_lanczos clamped to [0, 255]; outside pixels stay 0. */
int orc_synth_warp_case(const float* p, int w, int h, const double* hm, float** out, int* W, int* H,
                        double* composed) {
    mat_t mm, a0, a1, adj, f, back;
    memcpy(mm.m, hm, sizeof mm.m);
    a0 = mat_shift(-0.5, -0.5);
    a1 = mat_shift(0.5, 0.5);
    adj = mat_mul(&a0, &mm);
    adj = mat_mul(&adj, &a1);
    const double cx[4] = {0.0, (double)(w - 1), 0.0, (double)(w - 1)};
    const double cy[4] = {0.0, 0.0, (double)(h - 1), (double)(h - 1)};
    double minx = 1e30, miny = 1e30, maxx = -1e30, maxy = -1e30;
    for (int i = 0; i < 4; ++i) {
        const double wq = adj.m[6] * cx[i] + adj.m[7] * cy[i] + adj.m[8];
        if (fabs(wq) < 1e-9) return fail("degenerate homography for synthetic warp");
        double x, y;
        map_pt_proj(&adj, cx[i], cy[i], &x, &y);
        if (x < minx) minx = x;
        if (maxx < x) maxx = x;
        if (y < miny) miny = y;
        if (maxy < y) maxy = y;
    }
    if (maxx - minx > 20000 || maxy - miny > 20000)
        return fail("degenerate homography: unbounded warp target");
    const double tx = -floor(minx + 1e-9), ty = -floor(miny + 1e-9);
    *W = (int)(ceil(maxx - 1e-9) + tx) + 1;
    *H = (int)(ceil(maxy - 1e-9) + ty) + 1;
    mat_t sh = mat_shift(tx, ty);
    f = mat_mul(&sh, &adj);
    memcpy(composed, f.m, sizeof f.m);
    if (mat_inv(&f, &back)) return fail("degenerate homography: not invertible");
    img_t src = img_wrap(p, w, h);
    img_t o = img_new(*W, *H, 0.f);
    for (int y = 0; y < *H; ++y)
        for (int x = 0; x < *W; ++x) {
            double sx, sy;
            map_pt_proj(&back, x, y, &sx, &sy);
            if (sx < 0.0 || sx > w - 1.0 || sy < 0.0 || sy > h - 1.0) continue;
            double v = lanczos_at(&src, sx, sy, 4);
            v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            o.d[(size_t)y * *W + x] = (float)v;
        }
    *out = o.d;
    return 0;
}

/* float bilinear with clamp, double coordinates (warp.cpp:44-51) */
static inline float bilin_c(const img_t* im, double x, double y) {
    const int x0 = (int)floor(x), y0 = (int)floor(y);
    const float wx = (float)(x - x0), wy = (float)(y - y0);
    return (1 - wy) * ((1 - wx) * pxc(im, x0, y0) + wx * pxc(im, x0 + 1, y0)) +
           wy * ((1 - wx) * pxc(im, x0, y0 + 1) + wx * pxc(im, x0 + 1, y0 + 1));
}

/* directional anti-alias Gaussian (warp.cpp:128-158) */
int orc_antialias_tilt(const float* p, int w, int h, double t, double phi, float* out) {
    if (t < 1.0) return fail("antialias_tilt: tilt must be >= 1");
    if (t == 1.0) {
        memcpy(out, p, sizeof(float) * (size_t)w * h);
        return 0;
    }
    const double sigma = 0.8 * sqrt(t * t - 1.0);
    const double dx = cos(phi), dy = -sin(phi);
    int r = (int)ceil(3.0 * sigma);
    if (r < 1) r = 1;
    double* k = (double*)malloc(sizeof(double) * (2 * r + 1));
    double sum = 0;
    for (int i = -r; i <= r; ++i) {
        k[i + r] = exp(-0.5 * i * i / (sigma * sigma));
        sum += k[i + r];
    }
    for (int i = 0; i < 2 * r + 1; ++i) k[i] /= sum;
    img_t src = img_wrap(p, w, h);
    const int aligned = (dy == 0.0);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0;
            if (aligned)
                for (int i = -r; i <= r; ++i) acc += k[i + r] * pxc(&src, x + i, y);
            else
                for (int i = -r; i <= r; ++i) acc += k[i + r] * bilin_c(&src, x + i * dx, y + i * dy);
            out[(size_t)y * w + x] = (float)acc;
        }
    free(k);
    return 0;
}

/* --------------------------------------------------------------------- orb */

enum { LEVELS = 8, THR_MAIN = 20, THR_RELAXED = 7, ORIENT_R = 15, DETECT_BORDER = 17,
       DESCRIBE_BORDER = 20, MIN_SIDE = 32 };
static const double LEVEL_RATIO = 1.2;

/* Bresenham ring of radius 3, clockwise from 12 o'clock (orb.cpp:21-22) */
static const int ring_dx[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
static const int ring_dy[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};

/* half-width of the radius-15 orientation disc per row, mirrored across the
   diagonal (orb.cpp:25-41) */
static void disc_rows(int* umax) {
    const int r = ORIENT_R;
    const int vmax = (int)floor(r * sqrt(2.0) / 2 + 1);
    const int vmin = (int)ceil(r * sqrt(2.0) / 2);
    for (int v = 0; v <= r; ++v) umax[v] = 0;
    for (int v = 0; v <= vmax; ++v) umax[v] = (int)round(sqrt((double)r * r - v * v));
    int v0 = 0;
    for (int v = r; v >= vmin; --v) {
        while (umax[v0] == umax[v0 + 1]) ++v0;
        umax[v] = v0;
        ++v0;
    }
}

/* segment test: 9 contiguous ring pixels all brighter or all darker
   (orb.cpp:43-72) */
static int is_corner(const img_t* im, int x, int y, float thr) {
    const float p = px(im, x, y);
    const float hi = p + thr, lo = p - thr;
    int bright = 0, dark = 0, nb = 0, nd = 0;
    for (int i = 0; i < 16; ++i) {
        const float v = px(im, x + ring_dx[i], y + ring_dy[i]);
        if (v > hi) {
            bright |= 1 << i;
            ++nb;
        } else if (v < lo) {
            dark |= 1 << i;
            ++nd;
        }
    }
    if (nb < 9 && nd < 9) return 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int mask = pass == 0 ? bright : dark;
        int run = 0;
        for (int i = 0; i < 32; ++i) {
            if (mask >> (i & 15) & 1) {
                if (++run >= 9) return 1;
            } else {
                run = 0;
            }
        }
    }
    return 0;
}

/* sum of absolute ring differences in ring order (orb.cpp:74-80) */
static float seg_score(const img_t* im, int x, int y) {
    const float p = px(im, x, y);
    float s = 0;
    for (int i = 0; i < 16; ++i) s += fabsf(px(im, x + ring_dx[i], y + ring_dy[i]) - p);
    return s;
}

/* 7x7 Sobel structure tensor, k = 0.04 (orb.cpp:82-104) */
static float harris(const img_t* im, int x, int y) {
    double a = 0, b = 0, c = 0;
    for (int dy = -3; dy <= 3; ++dy)
        for (int dx = -3; dx <= 3; ++dx) {
            const int u = x + dx, v = y + dy;
            const float gx = (pxc(im, u + 1, v - 1) - pxc(im, u - 1, v - 1)) +
                             2 * (pxc(im, u + 1, v) - pxc(im, u - 1, v)) +
                             (pxc(im, u + 1, v + 1) - pxc(im, u - 1, v + 1));
            const float gy = (pxc(im, u - 1, v + 1) - pxc(im, u - 1, v - 1)) +
                             2 * (pxc(im, u, v + 1) - pxc(im, u, v - 1)) +
                             (pxc(im, u + 1, v + 1) - pxc(im, u + 1, v - 1));
            const double ix = gx, iy = gy;
            a += ix * ix;
            b += iy * iy;
            c += ix * iy;
        }
    const double sc = 1.0 / (255.0 * 4 * 7);
    a *= sc * sc;
    b *= sc * sc;
    c *= sc * sc;
    return (float)(a * b - c * c - 0.04 * (a + b) * (a + b));
}

/* intensity-centroid angle over the radius-15 disc (orb.cpp:106-123) */
static float centroid_angle(const img_t* im, int x, int y, const int* umax) {
    double m01 = 0, m10 = 0;
    for (int u = -ORIENT_R; u <= ORIENT_R; ++u) m10 += (float)u * px(im, x + u, y);
    for (int v = 1; v <= ORIENT_R; ++v) {
        const int d = umax[v];
        double vs = 0;
        for (int u = -d; u <= d; ++u) {
            const double up = px(im, x + u, y + v);
            const double dn = px(im, x + u, y - v);
            vs += up - dn;
            m10 += u * (up + dn);
        }
        m01 += v * vs;
    }
    return (float)atan2(m01, m10);
}

typedef struct {
    int n;
    img_t lv[LEVELS];
} pyr_t;

/* levels resized directly from level 0, stop below 32 px (orb.cpp:130-141) */
static void pyr_build(const img_t* im, pyr_t* p) {
    p->n = 1;
    p->lv[0] = img_new(im->w, im->h, 0.f);
    memcpy(p->lv[0].d, im->d, sizeof(float) * (size_t)im->w * im->h);
    for (int i = 1; i < LEVELS; ++i) {
        const double s = pow(LEVEL_RATIO, i);
        const int w = (int)round(im->w / s), h = (int)round(im->h / s);
        if (w < MIN_SIDE || h < MIN_SIDE) break;
        p->lv[i] = img_new(w, h, 0.f);
        resize_into(im, w, h, &p->lv[i]);
        p->n = i + 1;
    }
}

static void pyr_free(pyr_t* p) {
    for (int i = 0; i < p->n; ++i) free(p->lv[i].d);
}

typedef struct {
    int x, y, level;
    float score;
} cand_t;

typedef struct {
    cand_t* v;
    int n, cap;
} cands_t;

static void cands_push(cands_t* c, cand_t e) {
    if (c->n == c->cap) {
        c->cap = c->cap ? 2 * c->cap : 1024;
        c->v = (cand_t*)realloc(c->v, sizeof(cand_t) * c->cap);
    }
    c->v[c->n++] = e;
}

/* FAST + score map + 3x3 NMS with raster-order tie rule (orb.cpp:143-172) */
static void detect_levels(const pyr_t* p, float thr, cands_t* out) {
    out->n = 0;
    for (int L = 0; L < p->n; ++L) {
        const img_t* im = &p->lv[L];
        img_t sc = img_new(im->w, im->h, -1.f);
        for (int y = DETECT_BORDER; y < im->h - DETECT_BORDER; ++y)
            for (int x = DETECT_BORDER; x < im->w - DETECT_BORDER; ++x)
                if (is_corner(im, x, y, thr)) sc.d[(size_t)y * im->w + x] = seg_score(im, x, y);
        for (int y = DETECT_BORDER; y < im->h - DETECT_BORDER; ++y)
            for (int x = DETECT_BORDER; x < im->w - DETECT_BORDER; ++x) {
                const float s = px(&sc, x, y);
                if (s < 0) continue;
                int keep = 1;
                for (int dy = -1; dy <= 1 && keep; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        if (!dx && !dy) continue;
                        const float o = pxc(&sc, x + dx, y + dy);
                        if (o > s || (o == s && (dy < 0 || (dy == 0 && dx < 0)))) {
                            keep = 0;
                            break;
                        }
                    }
                if (keep) {
                    cand_t e = {x, y, L, s};
                    cands_push(out, e);
                }
            }
        free(sc.d);
    }
}

typedef struct {
    float x, y, response, orientation, octave_scale;
} kp_t;

/* response desc, then y asc, then x asc (orb.cpp:203-207) */
static int kp_order(const void* pa, const void* pb) {
    const kp_t* a = (const kp_t*)pa;
    const kp_t* b = (const kp_t*)pb;
    if (a->response != b->response) return a->response > b->response ? -1 : 1;
    if (a->y != b->y) return a->y < b->y ? -1 : 1;
    if (a->x != b->x) return a->x < b->x ? -1 : 1;
    return 0;
}

/* orb.cpp:182-210 */
int orc_detect(const float* p, int w, int h, int max_points, float** kps, int* n) {
    *n = 0;
    *kps = (float*)malloc(sizeof(kp_t));
    if (w < MIN_SIDE || h < MIN_SIDE || max_points <= 0) return 0;
    int umax[ORIENT_R + 1];
    disc_rows(umax);
    img_t im = img_wrap(p, w, h);
    pyr_t pyr;
    pyr_build(&im, &pyr);
    cands_t raw = {0, 0, 0};
    detect_levels(&pyr, (float)THR_MAIN, &raw);
    if (raw.n < max_points / 4) detect_levels(&pyr, (float)THR_RELAXED, &raw);
    kp_t* out = (kp_t*)malloc(sizeof(kp_t) * (raw.n ? raw.n : 1));
    for (int i = 0; i < raw.n; ++i) {
        const cand_t* c = &raw.v[i];
        const img_t* lv = &pyr.lv[c->level];
        const float ls = (float)pow(LEVEL_RATIO, c->level);
        out[i].x = c->x * ls;
        out[i].y = c->y * ls;
        out[i].octave_scale = ls;
        out[i].response = harris(lv, c->x, c->y);
        out[i].orientation = centroid_angle(lv, c->x, c->y, umax);
    }
    qsort(out, raw.n, sizeof(kp_t), kp_order);
    *n = raw.n < max_points ? raw.n : max_points;
    free(*kps);
    *kps = (float*)out;
    free(raw.v);
    pyr_free(&pyr);
    return 0;
}

int orc_detect_candidates(const float* p, int w, int h, float thr, int32_t** xyl, float** score,
                          int* n) {
    img_t im = img_wrap(p, w, h);
    pyr_t pyr;
    pyr_build(&im, &pyr);
    cands_t raw = {0, 0, 0};
    detect_levels(&pyr, thr, &raw);
    *xyl = (int32_t*)malloc(sizeof(int32_t) * 3 * (raw.n ? raw.n : 1));
    *score = (float*)malloc(sizeof(float) * (raw.n ? raw.n : 1));
    for (int i = 0; i < raw.n; ++i) {
        (*xyl)[3 * i] = raw.v[i].x;
        (*xyl)[3 * i + 1] = raw.v[i].y;
        (*xyl)[3 * i + 2] = raw.v[i].level;
        (*score)[i] = raw.v[i].score;
    }
    *n = raw.n;
    free(raw.v);
    pyr_free(&pyr);
    return 0;
}

int orc_corner_measures(const float* p, int w, int h, const int32_t* xy, int n, float* resp,
                        float* orient) {
    int umax[ORIENT_R + 1];
    disc_rows(umax);
    img_t im = img_wrap(p, w, h);
    for (int i = 0; i < n; ++i) {
        resp[i] = harris(&im, xy[2 * i], xy[2 * i + 1]);
        orient[i] = centroid_angle(&im, xy[2 * i], xy[2 * i + 1], umax);
    }
    return 0;
}

/* steered 256-pair comparisons on the sigma=2 blurred level
   (orb.cpp:212-248) */
int orc_describe(const float* p, int w, int h, const float* kin, int n, float** okps,
                 uint64_t** odesc, int* nout) {
    img_t im = img_wrap(p, w, h);
    pyr_t pyr;
    pyr_build(&im, &pyr);
    img_t blurred[LEVELS];
    int have[LEVELS] = {0};
    kp_t* ko = (kp_t*)malloc(sizeof(kp_t) * (n ? n : 1));
    uint64_t* d = (uint64_t*)malloc(sizeof(uint64_t) * 4 * (n ? n : 1));
    int m = 0;
    const kp_t* ks = (const kp_t*)kin;
    for (int i = 0; i < n; ++i) {
        const kp_t* k = &ks[i];
        const int L = (int)round(logf(k->octave_scale) / log(LEVEL_RATIO));
        if (L < 0 || L >= pyr.n) continue;
        const img_t* lv = &pyr.lv[L];
        const int lx = (int)roundf(k->x / k->octave_scale);
        const int ly = (int)roundf(k->y / k->octave_scale);
        if (lx < DESCRIBE_BORDER || ly < DESCRIBE_BORDER || lx >= lv->w - DESCRIBE_BORDER ||
            ly >= lv->h - DESCRIBE_BORDER)
            continue;
        if (!have[L]) {
            blurred[L] = img_new(lv->w, lv->h, 0.f);
            blur_into(lv, 2.0, &blurred[L]);
            have[L] = 1;
        }
        const img_t* b = &blurred[L];
        const float c = cosf(k->orientation), s = sinf(k->orientation);
        uint64_t bits[4] = {0, 0, 0, 0};
        for (int j = 0; j < 256; ++j) {
            const float px1 = k_pattern[4 * j], py1 = k_pattern[4 * j + 1];
            const float px2 = k_pattern[4 * j + 2], py2 = k_pattern[4 * j + 3];
            const int x1 = lx + (int)roundf(c * px1 - s * py1);
            const int y1 = ly + (int)roundf(s * px1 + c * py1);
            const int x2 = lx + (int)roundf(c * px2 - s * py2);
            const int y2 = ly + (int)roundf(s * px2 + c * py2);
            if (px(b, x1, y1) < px(b, x2, y2)) bits[j >> 6] |= 1ull << (j & 63);
        }
        ko[m] = *k;
        memcpy(d + 4 * m, bits, sizeof bits);
        ++m;
    }
    for (int L = 0; L < LEVELS; ++L)
        if (have[L]) free(blurred[L].d);
    pyr_free(&pyr);
    *okps = (float*)ko;
    *odesc = d;
    *nout = m;
    return 0;
}

/* L2 ratio matcher (sift.cpp:388-418): per pair a sequential float sum of
   (a_k - b_k)^2 (two roundings per step, -ffp-contract=off), top-2 scan in B
   order with strict '<' (lower B index wins ties), best/second held in
   double; missing second = distance 1024; keep iff sqrt(best) <
   ratio * min(sqrt(second), 1024) in double. */
int orc_match_ratio(const float* a, int na, const float* b, int nb, double ratio, int32_t** out,
                    int* n) {
    int32_t* o = (int32_t*)malloc(sizeof(int32_t) * 3 * (na ? na : 1));
    int m = 0;
    if (na > 0 && nb > 0)
        for (int i = 0; i < na; ++i) {
            const float* ai = a + 128 * (size_t)i;
            double best = 1e30, second = 1e30;
            int bi = -1;
            for (int j = 0; j < nb; ++j) {
                const float* bj = b + 128 * (size_t)j;
                float acc = 0.f;
                for (int k = 0; k < 128; ++k) {
                    const float d = ai[k] - bj[k];
                    acc += d * d;
                }
                if (acc < best) {
                    second = best;
                    best = acc;
                    bi = j;
                } else if (acc < second) {
                    second = acc;
                }
            }
            const double d1 = sqrt(best);
            const double d2 = second < 1e30 ? sqrt(second) : 1024.0;
            if (d1 < ratio * (d2 < 1024.0 ? d2 : 1024.0)) {
                const float df = (float)d1;
                o[3 * m] = i;
                o[3 * m + 1] = bi;
                memcpy(&o[3 * m + 2], &df, sizeof df);
                ++m;
            }
        }
    *out = o;
    *n = m;
    return 0;
}

/* top-2 scan in B order, lowest index wins ties, missing second = 256
   (orb.cpp:250-272) */
int orc_match(const uint64_t* a, int na, const uint64_t* b, int nb, double ratio, int32_t** out,
              int* n) {
    int32_t* o = (int32_t*)malloc(sizeof(int32_t) * 3 * (na ? na : 1));
    int m = 0;
    if (na > 0 && nb > 0)
        for (int i = 0; i < na; ++i) {
            int best = 257, second = 257, bi = -1;
            for (int j = 0; j < nb; ++j) {
                int d = 0;
                for (int w = 0; w < 4; ++w) d += __builtin_popcountll(a[4 * i + w] ^ b[4 * j + w]);
                if (d < best) {
                    second = best;
                    best = d;
                    bi = j;
                } else if (d < second) {
                    second = d;
                }
            }
            if (second > 256) second = 256;
            if (best < ratio * second) {
                o[3 * m] = i;
                o[3 * m + 1] = bi;
                o[3 * m + 2] = best;
                ++m;
            }
        }
    *out = o;
    *n = m;
    return 0;
}

/* pipeline.cpp:28-40 */
int orc_filter_to_content(const float* kin, int n, const double* back, int src_w, int src_h,
                          double margin, float** out, int* nout) {
    mat_t bk;
    memcpy(bk.m, back, sizeof bk.m);
    const kp_t* ks = (const kp_t*)kin;
    kp_t* o = (kp_t*)malloc(sizeof(kp_t) * (n ? n : 1));
    int m = 0;
    for (int i = 0; i < n; ++i) {
        double sx, sy;
        map_pt(&bk, ks[i].x, ks[i].y, &sx, &sy);
        if (sx >= margin && sx <= src_w - 1 - margin && sy >= margin && sy <= src_h - 1 - margin)
            o[m++] = ks[i];
    }
    *out = (float*)o;
    *nout = m;
    return 0;
}

/* ------------------------------------------------------ reference selection */

typedef struct {
    int32_t a, b;
    float d;
} rank_t;

static int rank_cmp(const void* x, const void* y) {
    const rank_t* p = (const rank_t*)x;
    const rank_t* q = (const rank_t*)y;
    if (p->d != q->d) return p->d < q->d ? -1 : 1;
    return (p->a > q->a) - (p->a < q->a);
}

/* scaling_coefficient (pipeline.cpp:70-101): rank by (distance, idx_a), take
   disjoint pairs (4i, 4i+1); segment lengths from float differences through
   hypotf (the reference's std::hypot(float, float)), weight from the float sum
   of the two distances. */
int orc_scaling_coefficient(const float* kps_a, int na, const float* kps_b, int nb,
                            const int32_t* m, int n, double* f, int* segments) {
    if (n < 2) return fail("insufficient matches for scaling estimation");
    rank_t* r = (rank_t*)malloc(sizeof(rank_t) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        r[i].a = m[3 * i];
        r[i].b = m[3 * i + 1];
        memcpy(&r[i].d, &m[3 * i + 2], sizeof(float));
        if (r[i].a < 0 || r[i].a >= na || r[i].b < 0 || r[i].b >= nb) {
            free(r);
            return fail("match indices out of range");
        }
    }
    qsort(r, (size_t)n, sizeof(rank_t), rank_cmp);
    const kp_t* ka = (const kp_t*)kps_a;
    const kp_t* kb = (const kp_t*)kps_b;
    double acc = 0;
    int seg = 0;
    for (int i = 0; 4 * i + 1 < n; ++i) {
        const rank_t m0 = r[4 * i], m1 = r[4 * i + 1];
        const double dis_a = hypotf(ka[m0.a].x - ka[m1.a].x, ka[m0.a].y - ka[m1.a].y);
        const double dis_b = hypotf(kb[m0.b].x - kb[m1.b].x, kb[m0.b].y - kb[m1.b].y);
        const float dsum = m0.d + m1.d;
        double w = 1.0 - dsum / 1000.0;
        if (w < 0.0) w = 0.0;
        acc += (dis_a - dis_b) * w;
        ++seg;
    }
    free(r);
    *f = acc;
    if (segments) *segments = seg;
    return 0;
}

static int fine_feats(const float* img, int w, int h, int cap, float** k, float** d, int* n) {
    float* raw;
    int nr;
    int rc = orc_detect_dog(img, w, h, cap, &raw, &nr);
    if (rc) return rc;
    rc = orc_describe_gradient(img, w, h, raw, nr, k, d, n);
    free(raw);
    return rc;
}

/* select_reference (pipeline.cpp:103-120) */
int orc_select_reference(const float* img1, int w1, int h1, const float* img2, int w2, int h2,
                         int cap, int* reference, double* f_forward, double* f_backward,
                         int* segments) {
    float *k1 = NULL, *d1 = NULL, *k2 = NULL, *d2 = NULL;
    int32_t *m12 = NULL, *m21 = NULL;
    int n1 = 0, n2 = 0, c12 = 0, c21 = 0, rc;
    *reference = 1;
    *f_forward = *f_backward = 0.0;
    *segments = 0;
    if ((rc = fine_feats(img1, w1, h1, cap, &k1, &d1, &n1))) goto done;
    if ((rc = fine_feats(img2, w2, h2, cap, &k2, &d2, &n2))) goto done;
    if ((rc = orc_match_ratio(d1, n1, d2, n2, 0.75, &m12, &c12))) goto done;
    if ((rc = orc_match_ratio(d2, n2, d1, n1, 0.75, &m21, &c21))) goto done;
    if (c12 < 2 || c21 < 2) {
        *reference = ((long)w2 * h2 > (long)w1 * h1) ? 2 : 1;
        goto done;
    }
    if ((rc = orc_scaling_coefficient(k1, n1, k2, n2, m12, c12, f_forward, segments))) goto done;
    if ((rc = orc_scaling_coefficient(k2, n2, k1, n1, m21, c21, f_backward, NULL))) goto done;
    *reference = (*f_forward >= *f_backward) ? 1 : 2;
done:
    free(k1); free(d1); free(k2); free(d2); free(m12); free(m21);
    return rc;
}

/* -------------------------------------------------------- ASIFT baseline */

typedef struct {
    float* kps;  /* described keypoints, 5 floats each */
    float* desc; /* 128 floats each */
    int n;
    mat_t back;
} simview_t;

/* simulate_views (pipeline.cpp:242-266): scale forced to 1, no content filter
   on the identity view */
static int sim_view(const float* img, int w, int h, const double* p_in, int cap, int a, simview_t* v) {
    double p[6], sim[9], fwd[9], tx, ty;
    memcpy(p, p_in, sizeof p);
    p[3] = 1.0;
    const int identity = p[1] == 1.0 && p[2] == 0.0 && p[3] == 1.0;
    v->kps = v->desc = NULL;
    v->n = 0;
    if (orc_simulation_from_params(p, sim)) return -1;
    float* filt = (float*)malloc(sizeof(float) * (size_t)w * h);
    float *view = NULL, *raw = NULL, *kept = NULL;
    int W, H, nr = 0, nk = 0, rc;
    if ((rc = orc_antialias_tilt(img, w, h, p[1], p[2], filt))) goto done;
    if ((rc = orc_warp(1, filt, w, h, sim, a, &view, &W, &H, &tx, &ty, fwd))) goto done;
    memcpy(v->back.m, fwd, sizeof fwd);
    {
        mat_t f;
        memcpy(f.m, fwd, sizeof fwd);
        if (mat_inv(&f, &v->back)) { rc = fail("invert: singular matrix"); goto done; }
    }
    if ((rc = orc_detect_dog(view, W, H, cap, &raw, &nr))) goto done;
    if (!identity) {
        if ((rc = orc_filter_to_content(raw, nr, v->back.m, w, h, (double)a, &kept, &nk))) goto done;
    } else {
        kept = raw;
        nk = nr;
        raw = NULL;
    }
    rc = orc_describe_gradient(view, W, H, kept, nk, &v->kps, &v->desc, &v->n);
done:
    free(filt); free(view); free(raw); free(kept);
    return rc;
}

/* asift_baseline (pipeline.cpp:298-343) up to RANSAC. The duplicate test scans
   every earlier correspondence: the reference's 2-px cell hash visits exactly
   the candidates that can pass the same predicate. */
int orc_asift_correspondences(const float* img1, int w1, int h1, const float* img2, int w2, int h2,
                              const double* grid, int n, int cap, double ratio, int a,
                              double** out, int* nout) {
    simview_t* v1 = (simview_t*)calloc((size_t)(n ? n : 1), sizeof(simview_t));
    simview_t* v2 = (simview_t*)calloc((size_t)(n ? n : 1), sizeof(simview_t));
    size_t m = 0, mcap = 1024;
    double* all = (double*)malloc(sizeof(double) * 5 * mcap);
    int rc = 0;
    *out = NULL;
    *nout = 0;
    if (n <= 0) { rc = fail("asift: empty parameter grid"); goto done; }
    for (int i = 0; i < n && !rc; ++i) rc = sim_view(img1, w1, h1, grid + 6 * i, cap, a, &v1[i]);
    for (int i = 0; i < n && !rc; ++i) rc = sim_view(img2, w2, h2, grid + 6 * i, cap, a, &v2[i]);
    for (int i = 0; i < n && !rc; ++i)
        for (int j = 0; j < n && !rc; ++j) {
            int32_t* mt = NULL;
            int nm = 0;
            if ((rc = orc_match_ratio(v1[i].desc, v1[i].n, v2[j].desc, v2[j].n, ratio, &mt, &nm))) break;
            const size_t first_fresh = m;
            for (int k = 0; k < nm; ++k) {
                const float* ka = v1[i].kps + 5 * mt[3 * k];
                const float* kb = v2[j].kps + 5 * mt[3 * k + 1];
                double c[5];
                float d;
                map_pt(&v1[i].back, ka[0], ka[1], &c[0], &c[1]);
                map_pt(&v2[j].back, kb[0], kb[1], &c[2], &c[3]);
                memcpy(&d, &mt[3 * k + 2], sizeof d);
                c[4] = d;
                int dup = 0;
                for (size_t q = 0; q < first_fresh && !dup; ++q) {
                    const double* o = all + 5 * q;
                    dup = hypot(o[0] - c[0], o[1] - c[1]) <= 2.0 && hypot(o[2] - c[2], o[3] - c[3]) <= 2.0;
                }
                if (dup) continue;
                if (m == mcap) {
                    mcap *= 2;
                    all = (double*)realloc(all, sizeof(double) * 5 * mcap);
                }
                memcpy(all + 5 * m++, c, sizeof c);
            }
            free(mt);
        }
done:
    for (int i = 0; i < n; ++i) {
        free(v1[i].kps); free(v1[i].desc); free(v2[i].kps); free(v2[i].desc);
    }
    free(v1);
    free(v2);
    if (rc) {
        free(all);
        return rc;
    }
    *out = all;
    *nout = (int)m;
    return 0;
}

/* ---------------------------------------------------------- coarse search */

typedef struct {
    const float *ref, *tdesc;
    int w, h, ntd, max_points, mode;
    double ratio;
    const double* grid;
    int n, stride, start;
    int *counts, *kpc;
    const uint64_t* td;
    int err;
} coarse_job_t;

/* one grid entry: blur -> warp -> detect -> content filter -> describe ->
   match count (pipeline.cpp:131-138) */
static int coarse_entry(const coarse_job_t* j, int i, int* count, int* kpc) {
    const double* p = j->grid + 6 * i;
    const int w = j->w, h = j->h;
    float* filt = (float*)malloc(sizeof(float) * (size_t)w * h);
    if (orc_antialias_tilt(j->ref, w, h, p[1], p[2], filt)) {
        free(filt);
        return -1;
    }
    double sim[9], fwd[9], back[9], tx, ty;
    if (orc_simulation_from_params(p, sim)) return -1;
    float* view;
    int W, H;
    if (orc_warp(j->mode & 1, filt, w, h, sim, 4, &view, &W, &H, &tx, &ty, fwd)) {
        free(filt);
        return -1;
    }
    free(filt);
    if (j->mode >= 2) /* uint8 views: lround + clamp (image_io.cpp:17-20) */
        for (size_t q = 0; q < (size_t)W * H; ++q) {
            long v = lroundf(view[q]);
            view[q] = (float)(v < 0 ? 0 : (v > 255 ? 255 : v));
        }
    float *kps, *kept, *dk;
    uint64_t* dd;
    int nk, nkept, nd;
    orc_detect(view, W, H, j->max_points, &kps, &nk);
    orc_invert(fwd, back);
    orc_filter_to_content(kps, nk, back, w, h, 5.0, &kept, &nkept);
    orc_describe(view, W, H, kept, nkept, &dk, &dd, &nd);
    int32_t* mm;
    int nm;
    orc_match(dd, nd, j->td, j->ntd, j->ratio, &mm, &nm);
    *count = nm;
    *kpc = nd;
    free(view);
    free(kps);
    free(kept);
    free(dk);
    free(dd);
    free(mm);
    return 0;
}

static void* coarse_worker(void* arg) {
    coarse_job_t* j = (coarse_job_t*)arg;
    for (int i = j->start; i < j->n; i += j->stride)
        if (coarse_entry(j, i, &j->counts[i], &j->kpc[i])) j->err = 1;
    return NULL;
}

static int worker_count(int n) {
    int t = g_threads;
    if (t <= 0) {
        const char* e = getenv("XAFFINE_THREADS");
        t = e ? atoi(e) : 0;
    }
    if (t <= 0) t = 1;
    return t < n ? t : n;
}

/* mode 0: nearest views (pipeline.cpp:122-152); mode 1: Lanczos views;
   modes 2/3: the same with every view quantised to uint8 before ORB (the
   device pipeline's view format, north_star "uint8 output"). */
int orc_coarse_search(const float* ref, int w, int h, const float* tgt, int tw, int th,
                      const double* grid, int n, int max_points, double ratio, int mode,
                      int* counts, int* kp_counts, int* best) {
    if (n <= 0) return fail("coarse: empty parameter grid");
    float *tk, *dk;
    uint64_t* td;
    int ntk, ntd;
    orc_detect(tgt, tw, th, max_points, &tk, &ntk);
    orc_describe(tgt, tw, th, tk, ntk, &dk, &td, &ntd);
    int* kpc = (int*)malloc(sizeof(int) * n);
    const int nw = worker_count(n);
    coarse_job_t* jobs = (coarse_job_t*)calloc(nw, sizeof(coarse_job_t));
    pthread_t* th_ = (pthread_t*)malloc(sizeof(pthread_t) * nw);
    for (int t = 0; t < nw; ++t) {
        coarse_job_t* j = &jobs[t];
        j->ref = ref;
        j->w = w;
        j->h = h;
        j->td = td;
        j->ntd = ntd;
        j->max_points = max_points;
        j->mode = mode;
        j->ratio = ratio;
        j->grid = grid;
        j->n = n;
        j->stride = nw;
        j->start = t;
        j->counts = counts;
        j->kpc = kpc;
        if (nw > 1)
            pthread_create(&th_[t], NULL, coarse_worker, j);
        else
            coarse_worker(j);
    }
    int err = 0;
    for (int t = 0; t < nw; ++t) {
        if (nw > 1) pthread_join(th_[t], NULL);
        err |= jobs[t].err;
    }
    free(jobs);
    free(th_);
    free(tk);
    free(dk);
    free(td);
    if (err) {
        free(kpc);
        return fail("coarse: entry failed");
    }
    int bc = -1;
    *best = 0;
    for (int i = 0; i < n; ++i) {
        if (kp_counts) kp_counts[i] = kpc[i];
        if (counts[i] > bc) {
            bc = counts[i];
            *best = i;
        }
    }
    free(kpc);
    return 0;
}

/* ------------------------------------------------------- test generators */

/* MT19937-64 (Matsumoto & Nishimura 2000), as std::mt19937_64 */
typedef struct {
    uint64_t s[312];
    int i;
} mt64_t;

static void mt64_seed(mt64_t* m, uint64_t seed) {
    m->s[0] = seed;
    for (int i = 1; i < 312; ++i)
        m->s[i] = 6364136223846793005ull * (m->s[i - 1] ^ (m->s[i - 1] >> 62)) + (uint64_t)i;
    m->i = 312;
}

static uint64_t mt64_next(mt64_t* m) {
    if (m->i >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x =
                (m->s[i] & 0xFFFFFFFF80000000ull) | (m->s[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            m->s[i] = m->s[(i + 156) % 312] ^ xa;
        }
        m->i = 0;
    }
    uint64_t y = m->s[m->i++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* libstdc++ uniform_real_distribution<double>: one 64-bit draw scaled by
   2^-64 (generate_canonical), clamped below 1, then a + u * (b - a). */
static double mt64_uniform(mt64_t* m, double a, double b) {
    double u = (double)mt64_next(m) / 18446744073709551616.0;
    if (u >= 1.0) u = nextafter(1.0, 0.0);
    return u * (b - a) + a;
}

/* dead-leaves texture of proj/tests/support/synthetic.cpp:29-60 */
int orc_make_texture(int w, int h, uint64_t seed, float* out) {
    mt64_t rng;
    mt64_seed(&rng, seed);
    const double min_side = w < h ? w : h;
    img_t im = img_new(w, h, 110.f);
    int rects = w * h / 900;
    if (rects < 60) rects = 60;
    for (int r = 0; r < rects; ++r) {
        const double cx = mt64_uniform(&rng, 0.0, w);
        const double cy = mt64_uniform(&rng, 0.0, h);
        const double hw = mt64_uniform(&rng, min_side / 64.0, min_side / 5.0) / 2;
        const double hh = mt64_uniform(&rng, min_side / 64.0, min_side / 5.0) / 2;
        const double ang = mt64_uniform(&rng, 0.0, M_PI);
        const float v = (float)mt64_uniform(&rng, 20.0, 235.0);
        const double ca = cos(ang), sa = sin(ang);
        const double reach = hypot(hw, hh);
        int x0 = (int)(cx - reach) - 1, x1 = (int)(cx + reach) + 1;
        int y0 = (int)(cy - reach) - 1, y1 = (int)(cy + reach) + 1;
        if (x0 < 0) x0 = 0;
        if (x1 > w - 1) x1 = w - 1;
        if (y0 < 0) y0 = 0;
        if (y1 > h - 1) y1 = h - 1;
        for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) {
                const double dx = x - cx, dy = y - cy;
                const double lx = dx * ca + dy * sa;
                const double ly = -dx * sa + dy * ca;
                if (fabs(lx) <= hw && fabs(ly) <= hh) im.d[(size_t)y * w + x] = v;
            }
    }
    img_t o = img_wrap(out, w, h);
    blur_into(&im, 0.6, &o);
    free(im.d);
    return 0;
}

int orc_make_checkerboard(int w, int h, int cell, float* out) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) out[(size_t)y * w + x] = (((x / cell) + (y / cell)) & 1) ? 220.f : 35.f;
    return 0;
}

/* ================================================================== SIFT
   Fine-stage DoG detector and gradient descriptor (sift.cpp:9-386), restated
   with the reference's float/double typing, operation order and glibc math
   (this file is compiled with -ffp-contract=off like the reference). */

#define SF_S 3                 /* scales per octave (sift.cpp:11) */
#define SF_NIMG (SF_S + 3)     /* gaussian images per octave */
#define SF_MAXO 16

typedef struct {
    int noct;
    img_t g[SF_MAXO][SF_NIMG];
    img_t d[SF_MAXO][SF_NIMG - 1];
} sf_pyr_t;

static void sf_pyr_free(sf_pyr_t* P) {
    for (int o = 0; o < P->noct; ++o) {
        for (int i = 0; i < SF_NIMG; ++i) free(P->g[o][i].d);
        for (int i = 0; i < SF_NIMG - 1; ++i) free(P->d[o][i].d);
    }
}

/* build_pyramid (sift.cpp:42-80): 2x bilinear upsample, blur to sigma 1.6,
   per octave 5 incremental blurs, DoG differences, next octave = every
   second pixel of gaussian image 3 */
static void sf_build(const img_t* img, sf_pyr_t* P) {
    img_t base = img_new(img->w * 2, img->h * 2, 0.f);
    resize_into(img, base.w, base.h, &base);
    const double sdiff = sqrt(fmax(1.6 * 1.6 - 4.0 * 0.5 * 0.5, 0.01));
    img_t b2 = img_new(base.w, base.h, 0.f);
    blur_into(&base, sdiff, &b2);
    free(base.d);
    double inc[SF_NIMG] = {0};
    const double k = pow(2.0, 1.0 / SF_S);
    double prev = 1.6;
    for (int i = 1; i < SF_NIMG; ++i) {
        const double total = 1.6 * pow(k, i);
        inc[i] = sqrt(total * total - prev * prev);
        prev = total;
    }
    int mn = b2.w < b2.h ? b2.w : b2.h;
    int no = (int)floor(log2((double)mn)) - 4;
    if (no < 1) no = 1;
    if (no > SF_MAXO) no = SF_MAXO;
    P->noct = no;
    for (int o = 0; o < no; ++o) {
        if (o == 0) {
            P->g[0][0] = b2;
        } else {
            const img_t* s = &P->g[o - 1][SF_S];
            img_t hv = img_new(s->w / 2, s->h / 2, 0.f);
            for (int y = 0; y < hv.h; ++y)
                for (int x = 0; x < hv.w; ++x) hv.d[(size_t)y * hv.w + x] = px(s, 2 * x, 2 * y);
            P->g[o][0] = hv;
        }
        for (int i = 1; i < SF_NIMG; ++i) {
            const img_t* s = &P->g[o][i - 1];
            P->g[o][i] = img_new(s->w, s->h, 0.f);
            blur_into(s, inc[i], &P->g[o][i]);
        }
        for (int i = 0; i + 1 < SF_NIMG; ++i) {
            const img_t* a = &P->g[o][i];
            const img_t* b = &P->g[o][i + 1];
            P->d[o][i] = img_new(a->w, a->h, 0.f);
            for (size_t p = 0; p < (size_t)a->w * a->h; ++p) P->d[o][i].d[p] = b->d[p] - a->d[p];
        }
    }
}

/* refine_extremum (sift.cpp:136-195) */
static double sf_det3(double M[3][3]) {
    return M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
           M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
           M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
}

static int sf_refine(const img_t* dog, int* layer, int* r, int* c, float* xr, float* xc, float* xs,
                     float* contrast) {
    const float sc = 1.f / 255.f;
    for (int step = 0;; ++step) {
        if (step >= 5) return 0;
        const img_t* cur = &dog[*layer];
        const img_t* prv = &dog[*layer - 1];
        const img_t* nxt = &dog[*layer + 1];
        const int C = *c, R = *r;
        const float dx = (px(cur, C + 1, R) - px(cur, C - 1, R)) * 0.5f * sc;
        const float dy = (px(cur, C, R + 1) - px(cur, C, R - 1)) * 0.5f * sc;
        const float ds = (px(nxt, C, R) - px(prv, C, R)) * 0.5f * sc;
        const float v2 = px(cur, C, R) * 2 * sc;
        const float dxx = (px(cur, C + 1, R) + px(cur, C - 1, R)) * sc - v2;
        const float dyy = (px(cur, C, R + 1) + px(cur, C, R - 1)) * sc - v2;
        const float dss = (px(nxt, C, R) + px(prv, C, R)) * sc - v2;
        const float dxy = (px(cur, C + 1, R + 1) - px(cur, C - 1, R + 1) - px(cur, C + 1, R - 1) +
                           px(cur, C - 1, R - 1)) * 0.25f * sc;
        const float dxs = (px(nxt, C + 1, R) - px(nxt, C - 1, R) - px(prv, C + 1, R) +
                           px(prv, C - 1, R)) * 0.25f * sc;
        const float dys = (px(nxt, C, R + 1) - px(nxt, C, R - 1) - px(prv, C, R + 1) +
                           px(prv, C, R - 1)) * 0.25f * sc;
        double H[3][3] = {{dxx, dxy, dxs}, {dxy, dyy, dys}, {dxs, dys, dss}};
        const double det = sf_det3(H);
        if (fabs(det) < 1e-20) return 0;
        double sol[3];
        for (int i = 0; i < 3; ++i) {
            double M[3][3];
            memcpy(M, H, sizeof M);
            M[0][i] = -dx;
            M[1][i] = -dy;
            M[2][i] = -ds;
            sol[i] = sf_det3(M) / det;
        }
        *xc = (float)sol[0];
        *xr = (float)sol[1];
        *xs = (float)sol[2];
        if (fabsf(*xc) < 0.5f && fabsf(*xr) < 0.5f && fabsf(*xs) < 0.5f) {
            *contrast = px(cur, C, R) * sc + 0.5f * (dx * *xc + dy * *xr + ds * *xs);
            const float tr = dxx + dyy;
            const float det2 = dxx * dyy - dxy * dxy;
            if (det2 <= 0) return 0;
            if (tr * tr * 10.0 >= (10.0 + 1) * (10.0 + 1) * det2) return 0;
            return fabsf(*contrast) * SF_S >= 0.03;
        }
        if (fabsf(*xc) > 1e6 || fabsf(*xr) > 1e6 || fabsf(*xs) > 1e6) return 0;
        *c += (int)lroundf(*xc);
        *r += (int)lroundf(*xr);
        *layer += (int)lroundf(*xs);
        if (*layer < 1 || *layer > SF_S || *c < 5 || *c >= cur->w - 5 || *r < 5 || *r >= cur->h - 5)
            return 0;
    }
}

/* orientation_histogram_peak (sift.cpp:93-125) */
static float sf_ori_hist(const img_t* im, int x, int y, double s, float hist[36]) {
    const int radius = (int)round(4.5 * s);
    const double wf = -1.0 / (2.0 * (1.5 * s) * (1.5 * s));
    float raw[36] = {0};
    for (int dy = -radius; dy <= radius; ++dy) {
        const int py = y + dy;
        if (py <= 0 || py >= im->h - 1) continue;
        for (int dx = -radius; dx <= radius; ++dx) {
            const int pxx = x + dx;
            if (pxx <= 0 || pxx >= im->w - 1) continue;
            const double gx = px(im, pxx + 1, py) - px(im, pxx - 1, py);
            const double gy = px(im, pxx, py - 1) - px(im, pxx, py + 1);
            const double mag = sqrt(gx * gx + gy * gy);
            const double ang = atan2(gy, gx);
            const double w = exp(wf * (dx * dx + dy * dy));
            int bin = (int)round(36 * (ang + M_PI) / (2 * M_PI));
            if (bin >= 36) bin -= 36;
            if (bin < 0) bin += 36;
            raw[bin] += (float)(w * mag);
        }
    }
    float peak = 0;
    for (int i = 0; i < 36; ++i) {
        hist[i] = (raw[(i - 2 + 36) % 36] + raw[(i + 2) % 36]) * (1.f / 16) +
                  (raw[(i - 1 + 36) % 36] + raw[(i + 1) % 36]) * (4.f / 16) + raw[i] * (6.f / 16);
        if (hist[i] > peak) peak = hist[i];
    }
    return peak;
}

static int sf_kp_less(const void* pa, const void* pb) {  /* sort_and_cap (sift.cpp:279-286) */
    const float* a = (const float*)pa;
    const float* b = (const float*)pb;
    if (a[2] != b[2]) return a[2] > b[2] ? -1 : 1;
    if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    return 0;
}

/* detect_dog_keypoints (sift.cpp:290-358); keypoints as 5 floats
   (x, y, response, orientation, octave_scale) */
int orc_detect_dog(const float* img, int w, int h, int max_points, float** out, int* n) {
    *out = NULL;
    *n = 0;
    if (w < 64 || h < 64 || max_points <= 0) return 0;
    img_t src = img_wrap(img, w, h);
    sf_pyr_t P;
    sf_build(&src, &P);
    const float prelim = (float)(0.5 * 0.03 / SF_S * 255.0);
    int cap = 1024, m = 0;
    float* kp = (float*)malloc(sizeof(float) * 5 * cap);
    for (int o = 0; o < P.noct; ++o) {
        const img_t* dogs = P.d[o];
        const int W = dogs[0].w, Hh = dogs[0].h;
        for (int layer = 1; layer <= SF_S; ++layer) {
            const img_t* cur = &dogs[layer];
            const img_t* ims[3] = {&dogs[layer - 1], cur, &dogs[layer + 1]};
            for (int r = 5; r < Hh - 5; ++r)
                for (int c = 5; c < W - 5; ++c) {
                    const float v = px(cur, c, r);
                    if (fabsf(v) <= prelim) continue;
                    int is_max = 1, is_min = 1;
                    for (int dy = -1; dy <= 1 && (is_max || is_min); ++dy)
                        for (int dx = -1; dx <= 1; ++dx)
                            for (int q = 0; q < 3; ++q) {
                                if (q == 1 && dx == 0 && dy == 0) continue;
                                const float nv = px(ims[q], c + dx, r + dy);
                                if (nv >= v) is_max = 0;
                                if (nv <= v) is_min = 0;
                            }
                    if (!is_max && !is_min) continue;
                    int ll = layer, rr = r, cc = c;
                    float xr, xc, xs, contrast;
                    if (!sf_refine(dogs, &ll, &rr, &cc, &xr, &xc, &xs, &contrast)) continue;
                    const double scl = 1.6 * pow(2.0, (ll + xs) / SF_S);
                    const double of = pow(2.0, o);
                    float k5[5];
                    k5[0] = (float)((cc + xc) * of * 0.5);
                    k5[1] = (float)((rr + xr) * of * 0.5);
                    k5[4] = (float)(scl * of * 0.5);
                    k5[2] = fabsf(contrast);
                    float hist[36];
                    const float peak = sf_ori_hist(&P.g[o][ll], cc, rr, scl, hist);
                    if (peak <= 0) continue;
                    const float thr = peak * 0.8f;
                    for (int bin = 0; bin < 36; ++bin) {
                        const int l = (bin - 1 + 36) % 36, rb = (bin + 1) % 36;
                        if (hist[bin] < thr || hist[bin] <= hist[l] || hist[bin] <= hist[rb]) continue;
                        float fbin = bin + 0.5f * (hist[l] - hist[rb]) / (hist[l] - 2 * hist[bin] + hist[rb]);
                        if (fbin < 0) fbin += 36;
                        if (fbin >= 36) fbin -= 36;
                        k5[3] = (float)(fbin * 2 * M_PI / 36 - M_PI);
                        if (m == cap) {
                            cap *= 2;
                            kp = (float*)realloc(kp, sizeof(float) * 5 * cap);
                        }
                        memcpy(kp + 5 * m, k5, sizeof k5);
                        ++m;
                    }
                }
        }
    }
    sf_pyr_free(&P);
    qsort(kp, m, 5 * sizeof(float), sf_kp_less);
    if (m > max_points) m = max_points;
    *out = kp;
    *n = m;
    return 0;
}

/* append_descriptor (sift.cpp:197-277) */
static void sf_descriptor(const img_t* im, float col, float row, float angle, double s, float* outv) {
    const float cos_t = cosf(angle), sin_t = sinf(angle);
    const float bpr = 8 / (2 * (float)M_PI);
    const float es = -1.f / (4 * 4 * 0.5f);
    const float hw = 3.f * (float)s;
    int radius = (int)roundf(hw * sqrtf(2.f) * (4 + 1) * 0.5f);
    const int rmax = (int)sqrt((double)im->w * im->w + (double)im->h * im->h);
    if (radius > rmax) radius = rmax;
    const float ct = cos_t / hw, st = sin_t / hw;
    float hist[6 * 6 * 10];
    memset(hist, 0, sizeof hist);
    const int icol = (int)roundf(col), irow = (int)roundf(row);
    for (int i = -radius; i <= radius; ++i)
        for (int j = -radius; j <= radius; ++j) {
            const float c_rot = j * ct - i * st;
            const float r_rot = j * st + i * ct;
            const float rbin = r_rot + 4 / 2 - 0.5f;
            const float cbin = c_rot + 4 / 2 - 0.5f;
            const int py = irow + i, pxx = icol + j;
            if (rbin <= -1 || rbin >= 4 || cbin <= -1 || cbin >= 4 || pxx <= 0 || pxx >= im->w - 1 ||
                py <= 0 || py >= im->h - 1)
                continue;
            const float gx = px(im, pxx + 1, py) - px(im, pxx - 1, py);
            const float gy = px(im, pxx, py - 1) - px(im, pxx, py + 1);
            const float mag = sqrtf(gx * gx + gy * gy);
            float theta = atan2f(gy, gx) - angle;
            while (theta < 0) theta += 2 * (float)M_PI;
            while (theta >= 2 * (float)M_PI) theta -= 2 * (float)M_PI;
            const float obin = theta * bpr;
            const float w = expf((c_rot * c_rot + r_rot * r_rot) * es) * mag;
            const int r0 = (int)floorf(rbin), c0 = (int)floorf(cbin);
            int o0 = (int)floorf(obin);
            const float rb = rbin - r0, cb = cbin - c0, ob = obin - o0;
            if (o0 >= 8) o0 -= 8;
            for (int dr = 0; dr <= 1; ++dr) {
                const int rr = r0 + dr + 1;
                if (rr < 0 || rr >= 6) continue;
                const float wr = w * (dr ? rb : 1 - rb);
                for (int dc = 0; dc <= 1; ++dc) {
                    const int cc = c0 + dc + 1;
                    if (cc < 0 || cc >= 6) continue;
                    const float wc = wr * (dc ? cb : 1 - cb);
                    for (int dor = 0; dor <= 1; ++dor) {
                        const float wo = wc * (dor ? ob : 1 - ob);
                        hist[(rr * 6 + cc) * 10 + o0 + dor] += wo;
                    }
                }
            }
        }
    float vec[128];
    int idx = 0;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            float* cell = &hist[((i + 1) * 6 + (j + 1)) * 10];
            cell[0] += cell[8];
            cell[1] += cell[9];
            for (int k = 0; k < 8; ++k) vec[idx++] = cell[k];
        }
    double norm = 0;
    for (int i = 0; i < 128; ++i) norm += (double)vec[i] * vec[i];
    const float thr = (float)sqrt(norm) * 0.2f;
    norm = 0;
    for (int i = 0; i < 128; ++i) {
        if (thr < vec[i]) vec[i] = thr;
        norm += (double)vec[i] * vec[i];
    }
    const double sn = sqrt(norm);
    const float scale = 512.f / (float)(sn > 1e-12 ? sn : 1e-12);
    for (int i = 0; i < 128; ++i) outv[i] = vec[i] * scale;
}

/* describe_gradient (sift.cpp:360-386) */
int orc_describe_gradient(const float* img, int w, int h, const float* kps, int n, float** okps,
                          float** odesc, int* nout) {
    *okps = NULL;
    *odesc = NULL;
    *nout = 0;
    if (w < 64 || h < 64) return 0;
    img_t src = img_wrap(img, w, h);
    sf_pyr_t P;
    sf_build(&src, &P);
    float* ok = (float*)malloc(sizeof(float) * 5 * (n ? n : 1));
    float* od = (float*)malloc(sizeof(float) * 128 * (n ? n : 1));
    int m = 0;
    for (int i = 0; i < n; ++i) {
        const float* kp = kps + 5 * i;
        if (kp[4] <= 0) continue;
        const double t = SF_S * log2(kp[4] * 2.0 / 1.6);
        int o = (int)floor((t - 0.5) / SF_S);
        if (o < 0) o = 0;
        if (o > P.noct - 1) o = P.noct - 1;
        int l = (int)lround(t - o * SF_S);
        if (l < 1) l = 1;
        if (l > SF_S) l = SF_S;
        const img_t* im = &P.g[o][l];
        const double of = pow(2.0, o) * 0.5;
        const float col = (float)(kp[0] / of), row = (float)(kp[1] / of);
        const double s = kp[4] / of;
        const float hw = 3.f * (float)s;
        const int radius = (int)roundf(hw * sqrtf(2.f) * (4 + 1) * 0.5f);
        if (col < radius || row < radius || col >= im->w - radius || row >= im->h - radius) continue;
        sf_descriptor(im, col, row, kp[3], s, od + 128 * m);
        memcpy(ok + 5 * m, kp, 5 * sizeof(float));
        ++m;
    }
    sf_pyr_free(&P);
    *okps = ok;
    *odesc = od;
    *nout = m;
    return 0;
}
