// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" face over the UNMODIFIED reference library compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libxaref.so.
// It exports the same `orc_*` interface as the C restatement in
// oracle/xa_oracle.c so tests can run both side by side and pin the
// restatement against the reference itself.
//
// Only the harness pieces are written here: argument marshalling, the
// Lanczos-view variant of the coarse loop (BASELINE.md §2 "harness variant")
// and two homography stubs (homography.cpp needs Eigen, absent in this image;
// RANSAC is outside the hot path and never reached from these entry points).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "synthetic.hpp"
#include "xaffine/eval.hpp"
#include "xaffine/features.hpp"
#include "xaffine/image_io.hpp"
#include "xaffine/geometry.hpp"
#include "xaffine/homography.hpp"
#include "xaffine/image.hpp"
#include "xaffine/orb.hpp"
#include "xaffine/orb_pattern.hpp"
#include "xaffine/parallel.hpp"
#include "xaffine/pipeline.hpp"
#include "xaffine/sift.hpp"
#include "xaffine/warp.hpp"

using namespace xaffine;

namespace xaffine {
// Stubs: pipeline.cpp's fine stage references these; the oracle never calls it.
AffineMatrix fit_homography_dlt(const std::vector<PointPair>&) {
    throw HomographyError("oracle/_ref: homography not built (Eigen absent)");
}
RansacResult estimate_homography_ransac(const std::vector<PointPair>&, const RansacConfig&) {
    throw HomographyError("oracle/_ref: homography not built (Eigen absent)");
}
// eval.cpp's load_sequence references it; image_io.cpp needs libpng (absent).
GrayImage load_image(const std::string&) { throw IoError("oracle/_ref: image I/O not built"); }
}  // namespace xaffine

namespace {
thread_local std::string g_err;

GrayImage to_img(const float* p, int w, int h) {
    GrayImage g(w, h);
    if (w > 0 && h > 0) std::memcpy(g.data.data(), p, sizeof(float) * size_t(w) * h);
    return g;
}

AffineMatrix to_mat(const double* m) {
    AffineMatrix r;
    for (int i = 0; i < 9; ++i) r.m[i] = m[i];
    return r;
}

AffineParams to_params(const double* p) {
    AffineParams a;
    a.psi = p[0];
    a.tilt = p[1];
    a.phi = p[2];
    a.scale = p[3];
    a.tx = p[4];
    a.ty = p[5];
    return a;
}

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

std::vector<float> kp_flat(const std::vector<Keypoint>& kps) {
    std::vector<float> f;
    f.reserve(kps.size() * 5);
    for (const auto& k : kps) {
        f.push_back(k.x);
        f.push_back(k.y);
        f.push_back(k.response);
        f.push_back(k.orientation);
        f.push_back(k.octave_scale);
    }
    return f;
}

std::vector<Keypoint> kp_unflat(const float* f, int n) {
    std::vector<Keypoint> v(n);
    for (int i = 0; i < n; ++i) {
        v[i].x = f[5 * i];
        v[i].y = f[5 * i + 1];
        v[i].response = f[5 * i + 2];
        v[i].orientation = f[5 * i + 3];
        v[i].octave_scale = f[5 * i + 4];
    }
    return v;
}

std::vector<BinaryDescriptor> desc_unflat(const uint64_t* p, int n) {
    std::vector<BinaryDescriptor> v(n);
    for (int i = 0; i < n; ++i)
        for (int w = 0; w < 4; ++w) v[i].bits[w] = p[4 * i + w];
    return v;
}

// Same back-map test as the reference's file-local filter (pipeline.cpp:28-40).
std::vector<Keypoint> keep_in_content(const std::vector<Keypoint>& kps, const AffineMatrix& back,
                                      int src_w, int src_h, double margin) {
    std::vector<Keypoint> out;
    for (const auto& kp : kps) {
        const auto [sx, sy] = map_point(back, kp.x, kp.y);
        if (sx >= margin && sx <= src_w - 1 - margin && sy >= margin && sy <= src_h - 1 - margin)
            out.push_back(kp);
    }
    return out;
}
}  // namespace

#define GUARD_BEGIN try {
#define GUARD_END                 \
    }                             \
    catch (const std::exception& e) { \
        g_err = e.what();         \
        return -1;                \
    }

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_free(void* p) { std::free(p); }
const char* orc_kind(void) { return "reference"; }

uint64_t orc_pattern_checksum(void) { return orb_pattern_checksum(); }

void orc_pattern(int8_t* out) {
    for (int i = 0; i < 256; ++i) {
        out[4 * i] = kOrbPattern[i].x1;
        out[4 * i + 1] = kOrbPattern[i].y1;
        out[4 * i + 2] = kOrbPattern[i].x2;
        out[4 * i + 3] = kOrbPattern[i].y2;
    }
}

int orc_make_texture(int w, int h, uint64_t seed, float* out) {
    GUARD_BEGIN
    const GrayImage g = testsupport::make_texture(w, h, seed);
    std::memcpy(out, g.data.data(), sizeof(float) * g.size());
    return 0;
    GUARD_END
}

int orc_make_checkerboard(int w, int h, int cell, float* out) {
    GUARD_BEGIN
    const GrayImage g = testsupport::make_checkerboard(w, h, cell);
    std::memcpy(out, g.data.data(), sizeof(float) * g.size());
    return 0;
    GUARD_END
}

int orc_gaussian_blur(const float* img, int w, int h, double sigma, float* out) {
    GUARD_BEGIN
    const GrayImage g = gaussian_blur(to_img(img, w, h), sigma);
    std::memcpy(out, g.data.data(), sizeof(float) * g.size());
    return 0;
    GUARD_END
}

int orc_resize_bilinear(const float* img, int w, int h, int nw, int nh, float* out) {
    GUARD_BEGIN
    const GrayImage g = resize_bilinear(to_img(img, w, h), nw, nh);
    std::memcpy(out, g.data.data(), sizeof(float) * g.size());
    return 0;
    GUARD_END
}

int orc_antialias_tilt(const float* img, int w, int h, double t, double phi, float* out) {
    GUARD_BEGIN
    const GrayImage g = antialias_tilt(to_img(img, w, h), t, phi);
    std::memcpy(out, g.data.data(), sizeof(float) * g.size());
    return 0;
    GUARD_END
}

double orc_lanczos_kernel(double x, int a) { return lanczos_kernel(x, a); }

double orc_sample_lanczos(const float* img, int w, int h, double x, double y, int a) {
    return sample_lanczos(to_img(img, w, h), x, y, a);
}

int orc_warp(int mode, const float* img, int w, int h, const double* m, int a, float** out,
             int* W, int* H, double* tx, double* ty, double* fwd) {
    GUARD_BEGIN
    const GrayImage src = to_img(img, w, h);
    const WarpResult r = mode == 0 ? warp_nearest(src, to_mat(m)) : warp_lanczos(src, to_mat(m), a);
    *out = dup(r.image.data);
    *W = r.image.width;
    *H = r.image.height;
    *tx = r.tx;
    *ty = r.ty;
    for (int i = 0; i < 9; ++i) fwd[i] = r.forward.m[i];
    return 0;
    GUARD_END
}

int orc_synth_warp_case(const float* img, int w, int h, const double* hm, float** out, int* W,
                        int* H, double* composed) {
    GUARD_BEGIN
    const auto [im, c] = synth_warp_case(to_img(img, w, h), to_mat(hm));
    *out = dup(im.data);
    *W = im.width;
    *H = im.height;
    for (int i = 0; i < 9; ++i) composed[i] = c.m[i];
    return 0;
    GUARD_END
}

int orc_detect(const float* img, int w, int h, int max_points, float** kps, int* n) {
    GUARD_BEGIN
    const auto v = detect_oriented_corners(to_img(img, w, h), max_points);
    *kps = dup(kp_flat(v));
    *n = static_cast<int>(v.size());
    return 0;
    GUARD_END
}

int orc_describe(const float* img, int w, int h, const float* kps, int n, float** okps,
                 uint64_t** odesc, int* nout) {
    GUARD_BEGIN
    const auto [k, d] = describe_binary(to_img(img, w, h), kp_unflat(kps, n));
    *okps = dup(kp_flat(k));
    std::vector<uint64_t> flat;
    for (const auto& x : d)
        for (int i = 0; i < 4; ++i) flat.push_back(x.bits[i]);
    *odesc = dup(flat);
    *nout = static_cast<int>(k.size());
    return 0;
    GUARD_END
}

int orc_match(const uint64_t* a, int na, const uint64_t* b, int nb, double ratio, int32_t** out,
              int* n) {
    GUARD_BEGIN
    const auto m = match_hamming(desc_unflat(a, na), desc_unflat(b, nb), ratio);
    std::vector<int32_t> flat;
    for (const auto& x : m) {
        flat.push_back(x.idx_a);
        flat.push_back(x.idx_b);
        flat.push_back(static_cast<int32_t>(x.distance));
    }
    *out = dup(flat);
    *n = static_cast<int>(m.size());
    return 0;
    GUARD_END
}

int orc_match_ratio(const float* a, int na, const float* b, int nb, double ratio, int32_t** out,
                    int* n) {
    GUARD_BEGIN
    auto unflat = [](const float* p, int cnt) {
        std::vector<GradientDescriptor> v(cnt);
        for (int i = 0; i < cnt; ++i) std::memcpy(v[i].values.data(), p + 128 * (size_t)i, 128 * sizeof(float));
        return v;
    };
    const auto m = match_ratio(unflat(a, na), unflat(b, nb), ratio);
    std::vector<int32_t> flat;
    for (const auto& x : m) {
        int32_t bits;
        std::memcpy(&bits, &x.distance, sizeof bits);
        flat.insert(flat.end(), {x.idx_a, x.idx_b, bits});
    }
    *out = dup(flat);
    *n = static_cast<int>(m.size());
    return 0;
    GUARD_END
}

int orc_detect_dog(const float* img, int w, int h, int max_points, float** kps, int* n) {
    GUARD_BEGIN
    const auto v = detect_dog_keypoints(to_img(img, w, h), max_points);
    *kps = dup(kp_flat(v));
    *n = static_cast<int>(v.size());
    return 0;
    GUARD_END
}

int orc_describe_gradient(const float* img, int w, int h, const float* kps, int n, float** okps,
                          float** odesc, int* nout) {
    GUARD_BEGIN
    const auto [k, d] = describe_gradient(to_img(img, w, h), kp_unflat(kps, n));
    *okps = dup(kp_flat(k));
    std::vector<float> flat;
    for (const auto& x : d) flat.insert(flat.end(), x.values.begin(), x.values.end());
    *odesc = dup(flat);
    *nout = static_cast<int>(k.size());
    return 0;
    GUARD_END
}

int orc_scaling_coefficient(const float* kps_a, int na, const float* kps_b, int nb,
                            const int32_t* m, int n, double* f, int* segments) {
    GUARD_BEGIN
    std::vector<MatchPair> v(n);
    for (int i = 0; i < n; ++i) {
        v[i].idx_a = m[3 * i];
        v[i].idx_b = m[3 * i + 1];
        std::memcpy(&v[i].distance, &m[3 * i + 2], sizeof(float));
    }
    *f = scaling_coefficient(kp_unflat(kps_a, na), kp_unflat(kps_b, nb), v, segments);
    return 0;
    GUARD_END
}

int orc_select_reference(const float* img1, int w1, int h1, const float* img2, int w2, int h2,
                         int cap, int* reference, double* f_forward, double* f_backward,
                         int* segments) {
    GUARD_BEGIN
    const ReferenceDecision d = select_reference(to_img(img1, w1, h1), to_img(img2, w2, h2), cap);
    *reference = d.reference;
    *f_forward = d.f_forward;
    *f_backward = d.f_backward;
    *segments = d.segment_count;
    return 0;
    GUARD_END
}

// asift_baseline (pipeline.cpp:298-343) up to RANSAC, restated over the
// reference's public functions (its simulate_views and duplicate filter are
// file-local): the same per-view steps and the same duplicate predicate.
int orc_asift_correspondences(const float* img1, int w1, int h1, const float* img2, int w2, int h2,
                              const double* grid, int n, int cap, double ratio, int a,
                              double** out, int* nout) {
    GUARD_BEGIN
    if (n <= 0) throw PipelineError("asift: empty parameter grid");
    struct View {
        std::vector<Keypoint> kps;
        std::vector<GradientDescriptor> descs;
        AffineMatrix back;
    };
    auto simulate = [&](const GrayImage& img) {
        std::vector<View> vs;
        for (int i = 0; i < n; ++i) {
            AffineParams p = to_params(grid + 6 * i);
            p.scale = 1.0;
            const bool identity = p.tilt == 1.0 && p.phi == 0.0 && p.scale == 1.0;
            const WarpResult w = warp_lanczos(antialias_tilt(img, p.tilt, p.phi), simulation_from_params(p), a);
            View v;
            v.back = invert(w.forward);
            auto kps = detect_dog_keypoints(w.image, cap);
            if (!identity) kps = keep_in_content(kps, v.back, img.width, img.height, (double)a);
            auto [k, d] = describe_gradient(w.image, kps);
            v.kps = std::move(k);
            v.descs = std::move(d);
            vs.push_back(std::move(v));
        }
        return vs;
    };
    const auto va = simulate(to_img(img1, w1, h1)), vb = simulate(to_img(img2, w2, h2));
    std::vector<double> all;
    for (const auto& x : va)
        for (const auto& y : vb) {
            const auto ms = match_ratio(x.descs, y.descs, ratio);
            const size_t earlier = all.size();
            for (const auto& m : ms) {
                const auto [x1, y1] = map_point(x.back, x.kps[m.idx_a].x, x.kps[m.idx_a].y);
                const auto [x2, y2] = map_point(y.back, y.kps[m.idx_b].x, y.kps[m.idx_b].y);
                bool dup = false;
                for (size_t q = 0; q < earlier && !dup; q += 5)
                    dup = std::hypot(all[q] - x1, all[q + 1] - y1) <= 2.0 &&
                          std::hypot(all[q + 2] - x2, all[q + 3] - y2) <= 2.0;
                if (!dup) all.insert(all.end(), {x1, y1, x2, y2, (double)m.distance});
            }
        }
    *out = dup(all);
    *nout = static_cast<int>(all.size() / 5);
    return 0;
    GUARD_END
}

int orc_build_grid(double a, int n, double b_deg, double delta_s, double** params, int* count) {
    GUARD_BEGIN
    GridConfig c;
    c.a = a;
    c.n = n;
    c.b_deg = b_deg;
    c.delta_s = delta_s;
    const ParamGrid g = build_param_grid(c);
    std::vector<double> flat;
    for (const auto& p : g.entries) {
        flat.insert(flat.end(), {p.psi, p.tilt, p.phi, p.scale, p.tx, p.ty});
    }
    *params = dup(flat);
    *count = static_cast<int>(g.entries.size());
    return 0;
    GUARD_END
}

int orc_simulation_from_params(const double* p, double* m) {
    GUARD_BEGIN
    const AffineMatrix r = simulation_from_params(to_params(p));
    for (int i = 0; i < 9; ++i) m[i] = r.m[i];
    return 0;
    GUARD_END
}

int orc_affine_from_params(const double* p, double* m) {
    GUARD_BEGIN
    const AffineMatrix r = affine_from_params(to_params(p));
    for (int i = 0; i < 9; ++i) m[i] = r.m[i];
    return 0;
    GUARD_END
}

int orc_invert(const double* m, double* out) {
    GUARD_BEGIN
    const AffineMatrix r = invert(to_mat(m));
    for (int i = 0; i < 9; ++i) out[i] = r.m[i];
    return 0;
    GUARD_END
}

int orc_filter_to_content(const float* kps, int n, const double* back, int src_w, int src_h,
                          double margin, float** out, int* nout) {
    GUARD_BEGIN
    const auto v = keep_in_content(kp_unflat(kps, n), to_mat(back), src_w, src_h, margin);
    *out = dup(kp_flat(v));
    *nout = static_cast<int>(v.size());
    return 0;
    GUARD_END
}

// mode 0: the reference's own coarse_search (nearest views, pipeline.cpp:122-152).
// mode 1: the same loop with warp_lanczos views (BASELINE.md §2 harness variant).
// Per-entry described keypoint counts (after the content filter and the describe
// border drop) are returned in kp_counts when non-null; mode 0 leaves them -1.
int orc_coarse_search(const float* ref, int w, int h, const float* tgt, int tw, int th,
                      const double* grid, int n, int max_points, double ratio, int mode,
                      int* counts, int* kp_counts, int* best) {
    GUARD_BEGIN
    ParamGrid g;
    for (int i = 0; i < n; ++i) g.entries.push_back(to_params(grid + 6 * i));
    const GrayImage R = to_img(ref, w, h), T = to_img(tgt, tw, th);
    if (mode == 0) {
        const CoarseResult r = coarse_search(R, T, g, max_points, ratio);
        for (int i = 0; i < n; ++i) {
            counts[i] = r.per_entry_counts[i].second;
            if (kp_counts) kp_counts[i] = -1;
        }
        *best = -1;
        for (int i = 0; i < n; ++i)
            if (counts[i] == r.best_count && *best < 0) *best = i;
        return 0;
    }
    if (g.entries.empty()) throw PipelineError("coarse: empty parameter grid");
    const auto target_kps = detect_oriented_corners(T, max_points);
    const auto [tkps, target_descs] = describe_binary(T, target_kps);
    std::vector<int> cnt(n, 0), kpc(n, 0);
    parallel_for(n, [&](int i) {
        const AffineParams& p = g.entries[i];
        const GrayImage filtered = antialias_tilt(R, p.tilt, p.phi);
        const WarpResult wr = warp_lanczos(filtered, simulation_from_params(p), 4);
        auto kps = detect_oriented_corners(wr.image, max_points);
        kps = keep_in_content(kps, invert(wr.forward), R.width, R.height, 5.0);
        const auto [wkps, wdescs] = describe_binary(wr.image, kps);
        kpc[i] = static_cast<int>(wdescs.size());
        cnt[i] = static_cast<int>(match_hamming(wdescs, target_descs, ratio).size());
    });
    int bc = -1;
    *best = 0;
    for (int i = 0; i < n; ++i) {
        counts[i] = cnt[i];
        if (kp_counts) kp_counts[i] = kpc[i];
        if (cnt[i] > bc) {
            bc = cnt[i];
            *best = i;
        }
    }
    return 0;
    GUARD_END
}

}  // extern "C"
