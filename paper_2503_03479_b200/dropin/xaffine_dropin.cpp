// xaffine_dropin.cpp — link-time drop-in for the reference's hot-path
// translation units, backed by libxa_b200.so (include/xaffine_b200.h).
//
// Compile against the reference's own headers (proj/include) and link this
// object INSTEAD OF proj/src/warp.cpp and proj/src/orb.cpp; every other
// reference object links unchanged. INTEGRATION.md gives the recipe and the
// optional one-line patch that routes pipeline.cpp's coarse_search through the
// batched xa_coarse_search.
//
// Replaced symbols (reference declaration -> this file):
//   warp.hpp:22  lanczos_kernel          scalar helper, host (not a batch path)
//   warp.hpp:23  sample_lanczos          scalar helper, host (not a batch path)
//   warp.hpp:25  warp_nearest            -> xa_warp(XA_NEAREST)
//   warp.hpp:27  warp_lanczos            -> xa_warp(XA_LANCZOS)
//   warp.hpp:31  antialias_tilt          -> xa_antialias_tilt
//   features.hpp:27 hamming_distance     scalar helper, host popcount
//   orb.hpp:14   detect_oriented_corners -> xa_detect_oriented_corners
//   orb.hpp:19   describe_binary         -> xa_describe_binary
//   orb.hpp:25   match_hamming           -> xa_match_hamming
// plus xaffine::b200::coarse_search (pipeline.hpp:86 signature) -> xa_coarse_search
// and  xaffine::b200::match_ratio   (sift.hpp:28 signature)     -> xa_match_ratio,
//      xaffine::b200::detect_dog_keypoints (sift.hpp:13)        -> xa_detect_dog_keypoints,
//      xaffine::b200::describe_gradient    (sift.hpp:22)        -> xa_describe_gradient,
//      xaffine::b200::select_reference     (pipeline.hpp:80)    -> the three above +
//                                           the reference's own scaling_coefficient,
//      xaffine::b200::synth_warp_case      (eval.hpp:58)        -> xa_synth_warp_case
// (the fine stage lives in sift.cpp next to code the drop-in does not replace,
// so these are routed with a one-line #ifdef).
//
// Errors: XA_EINVAL / XA_ESINGULAR from geometry come back as GeometryError
// (the reference throws it from invert and the tilt checks), XA_EPIPELINE as
// PipelineError, anything else as std::runtime_error with xa_last_error().
// Threading: the reference calls these from parallel_for workers; each host
// thread gets its own engine (thread_local), so calls are re-entrant.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "xaffine/eval.hpp"
#include "xaffine/features.hpp"
#include "xaffine/geometry.hpp"
#include "xaffine/image.hpp"
#include "xaffine/homography.hpp"
#include "xaffine/image_io.hpp"
#include "xaffine/orb.hpp"
#include "xaffine/pipeline.hpp"
#include "xaffine/warp.hpp"
#include "xaffine_b200.h"

namespace {

static_assert(sizeof(xaffine::Keypoint) == sizeof(xa_keypoint), "Keypoint layout");
static_assert(sizeof(xaffine::MatchPair) == sizeof(xa_match), "MatchPair layout");
static_assert(sizeof(xaffine::AffineParams) == sizeof(xa_params), "AffineParams layout");
static_assert(sizeof(xaffine::BinaryDescriptor) == 4 * sizeof(uint64_t), "descriptor layout");

[[noreturn]] void raise(int rc) {
    const std::string msg = xa_last_error();
    if (rc == XA_ESINGULAR || (rc == XA_EINVAL && (msg.find("tilt") != std::string::npos ||
                                                   msg.find("scale") != std::string::npos)))
        throw xaffine::GeometryError(msg);
    if (rc == XA_EPIPELINE) throw xaffine::PipelineError(msg);
    if (rc == XA_EEVAL) throw xaffine::EvalError(msg);
    if (rc == XA_EIO) throw xaffine::IoError(msg);
    if (rc == XA_EHOMOGRAPHY) throw xaffine::HomographyError(msg);
    throw std::runtime_error("xaffine_b200: " + msg);
}

void check(int rc) {
    if (rc != XA_OK) raise(rc);
}

struct EngineHolder {
    xa_engine* e = nullptr;
    EngineHolder() {
        const char* dev = std::getenv("XAFFINE_B200_DEVICE");
        check(xa_engine_create(dev ? std::atoi(dev) : 0, &e));
    }
    ~EngineHolder() { xa_engine_destroy(e); }
};

xa_engine* engine() {
    thread_local EngineHolder h;
    return h.e;
}

}  // namespace

namespace xaffine {

// warp.cpp:55-60 (scalar helper kept on the host: one kernel evaluation)
double lanczos_kernel(double x, int a) {
    if (x <= -a || x >= a) return 0.0;
    if (x == 0.0) return 1.0;
    const double px = M_PI * x;
    return (std::sin(px) / px) * (std::sin(px / a) * a / px);
}

// warp.cpp:62-84 (scalar helper: one sample, used by eval's projective warp)
double sample_lanczos(const GrayImage& img, double x, double y, int a) {
    const int fx = static_cast<int>(std::floor(x)), fy = static_cast<int>(std::floor(y));
    const double rx = x - fx, ry = y - fy;
    double wx[16], wy[16];
    for (int i = -a + 1; i <= a; ++i) {
        wx[i + a - 1] = lanczos_kernel(i - rx, a);
        wy[i + a - 1] = lanczos_kernel(i - ry, a);
    }
    double acc = 0, wsum = 0;
    for (int j = 0; j < 2 * a; ++j) {
        double row = 0, rw = 0;
        for (int i = 0; i < 2 * a; ++i) {
            row += wx[i] * img.at_clamped(fx + i - a + 1, fy + j - a + 1);
            rw += wx[i];
        }
        acc += wy[j] * row;
        wsum += wy[j] * rw;
    }
    return acc / wsum;
}

static WarpResult run_warp(int mode, const GrayImage& img, const AffineMatrix& m, int a) {
    WarpResult r;
    int W = 0, H = 0;
    check(xa_warp_frame(m.m.data(), img.width, img.height, &W, &H, &r.tx, &r.ty, r.forward.m.data()));
    r.image = GrayImage(W, H);
    check(xa_warp(engine(), mode, img.data.data(), img.width, img.height, m.m.data(), a,
                  r.image.data.data(), r.image.data.size(), &W, &H, &r.tx, &r.ty,
                  r.forward.m.data()));
    return r;
}

WarpResult warp_nearest(const GrayImage& img, const AffineMatrix& m) {
    return run_warp(XA_NEAREST, img, m, 4);
}

WarpResult warp_lanczos(const GrayImage& img, const AffineMatrix& m, int a) {
    return run_warp(XA_LANCZOS, img, m, a);
}

GrayImage antialias_tilt(const GrayImage& img, double t, double phi) {
    GrayImage out(img.width, img.height);
    check(xa_antialias_tilt(engine(), img.data.data(), img.width, img.height, t, phi,
                            out.data.data()));
    return out;
}

int hamming_distance(const BinaryDescriptor& a, const BinaryDescriptor& b) {
    int d = 0;
    for (int i = 0; i < 4; ++i) d += __builtin_popcountll(a.bits[i] ^ b.bits[i]);
    return d;
}

std::vector<Keypoint> detect_oriented_corners(const GrayImage& img, int max_points) {
    std::vector<Keypoint> out(max_points > 0 ? max_points : 0);
    int n = 0;
    check(xa_detect_oriented_corners(engine(), img.data.data(), img.width, img.height, max_points,
                                     reinterpret_cast<xa_keypoint*>(out.data()),
                                     static_cast<int>(out.size()), &n));
    out.resize(n);
    return out;
}

std::pair<std::vector<Keypoint>, std::vector<BinaryDescriptor>> describe_binary(
    const GrayImage& img, const std::vector<Keypoint>& kps) {
    std::pair<std::vector<Keypoint>, std::vector<BinaryDescriptor>> out;
    out.first.resize(kps.size());
    out.second.resize(kps.size());
    int n = 0;
    check(xa_describe_binary(engine(), img.data.data(), img.width, img.height,
                             reinterpret_cast<const xa_keypoint*>(kps.data()),
                             static_cast<int>(kps.size()),
                             reinterpret_cast<xa_keypoint*>(out.first.data()),
                             reinterpret_cast<uint64_t*>(out.second.data()), &n));
    out.first.resize(n);
    out.second.resize(n);
    return out;
}

std::vector<MatchPair> match_hamming(const std::vector<BinaryDescriptor>& desc_a,
                                     const std::vector<BinaryDescriptor>& desc_b, double ratio) {
    std::vector<MatchPair> out(desc_a.size());
    int n = 0;
    check(xa_match_hamming(engine(), reinterpret_cast<const uint64_t*>(desc_a.data()),
                           static_cast<int>(desc_a.size()),
                           reinterpret_cast<const uint64_t*>(desc_b.data()),
                           static_cast<int>(desc_b.size()), ratio,
                           reinterpret_cast<xa_match*>(out.data()), &n));
    out.resize(n);
    return out;
}

// homography.cpp replacement (homography.hpp:27-39): normalised DLT and
// seeded 4-point RANSAC on the host behind the C-ABI (xa_homography.cpp; Eigen
// is absent, the SVD is a one-sided Jacobi).
static_assert(sizeof(xaffine::PointPair) == 4 * sizeof(double), "PointPair layout");

AffineMatrix fit_homography_dlt(const std::vector<PointPair>& pts) {
    AffineMatrix h;
    check(xa_fit_homography_dlt(reinterpret_cast<const double*>(pts.data()), (int)pts.size(), h.m.data()));
    return h;
}

RansacResult estimate_homography_ransac(const std::vector<PointPair>& pts, const RansacConfig& cfg) {
    RansacResult r;
    std::vector<int32_t> inl(std::max<size_t>(pts.size(), 1));
    int n = 0;
    check(xa_estimate_homography_ransac(reinterpret_cast<const double*>(pts.data()), (int)pts.size(),
                                        cfg.threshold, cfg.max_iters, cfg.confidence, cfg.seed,
                                        r.homography.m.data(), inl.data(), (int)inl.size(), &n));
    r.inliers.assign(inl.begin(), inl.begin() + n);
    return r;
}

// image_io.cpp replacement (image_io.hpp:14-24): host file I/O behind the
// C-ABI (xa_image_io.cpp; libpng is absent, PNG goes through zlib).
GrayImage load_image(const std::string& path) {
    int w = 0, h = 0;
    check(xa_load_image(path.c_str(), nullptr, 0, &w, &h));
    GrayImage img(w, h);
    check(xa_load_image(path.c_str(), img.data.data(), img.data.size(), &w, &h));
    return img;
}

void save_image(const GrayImage& img, const std::string& path) {
    check(xa_save_image(img.data.data(), img.width, img.height, path.c_str()));
}

void save_png_rgb(const RgbImage& img, const std::string& path) {
    check(xa_save_png_rgb(img.data.data(), img.width, img.height, path.c_str()));
}

namespace b200 {

// Batched replacement for xaffine::coarse_search (pipeline.cpp:122-152): all
// grid entries in one device pipeline. Views are nearest-resampled (the
// reference coarse stage) and quantised to uint8 before ORB.
CoarseResult coarse_search(const GrayImage& ref, const GrayImage& target, const ParamGrid& grid,
                           int max_points, double ratio) {
    const int n = static_cast<int>(grid.entries.size());
    if (n == 0) throw PipelineError("coarse: empty parameter grid");
    std::vector<int32_t> counts(n), kpc(n);
    int32_t best = 0;
    check(xa_coarse_search(engine(), XA_F32, ref.data.data(), ref.width, ref.height,
                           target.data.data(), target.width, target.height,
                           reinterpret_cast<const xa_params*>(grid.entries.data()), n, max_points,
                           ratio, XA_NEAREST, counts.data(), kpc.data(), &best));
    CoarseResult r;
    r.best_count = -1;
    for (int i = 0; i < n; ++i) {
        r.per_entry_counts.emplace_back(grid.entries[i], counts[i]);
        if (counts[i] > r.best_count) {
            r.best_count = counts[i];
            r.best_params = grid.entries[i];
        }
    }
    return r;
}

// Replacement for xaffine::detect_dog_keypoints (sift.cpp:290-358): keypoints
// identical to the reference (tests/test_gpu_sift.py).
std::vector<Keypoint> detect_dog_keypoints(const GrayImage& img, int max_points) {
    if (img.width < 64 || img.height < 64 || max_points <= 0) return {};
    std::vector<Keypoint> out(max_points);
    int n = 0;
    check(xa_detect_dog_keypoints(engine(), img.data.data(), img.width, img.height, max_points,
                                  reinterpret_cast<xa_keypoint*>(out.data()), max_points, &n));
    out.resize(n);
    return out;
}

// Replacement for xaffine::describe_gradient (sift.cpp:360-386).
std::pair<std::vector<Keypoint>, std::vector<GradientDescriptor>> describe_gradient(
    const GrayImage& img, const std::vector<Keypoint>& kps) {
    std::pair<std::vector<Keypoint>, std::vector<GradientDescriptor>> out;
    out.first.resize(kps.size());
    out.second.resize(kps.size());
    int n = 0;
    check(xa_describe_gradient(engine(), img.data.data(), img.width, img.height,
                               reinterpret_cast<const xa_keypoint*>(kps.data()), static_cast<int>(kps.size()),
                               reinterpret_cast<xa_keypoint*>(out.first.data()),
                               reinterpret_cast<float*>(out.second.data()), &n));
    out.first.resize(n);
    out.second.resize(n);
    return out;
}

// Replacement for xaffine::match_ratio (sift.cpp:388-418), the fine stage's L2
// ratio matcher; bit-identical results (tests/test_gpu_l2match.py).
std::vector<MatchPair> match_ratio(const std::vector<GradientDescriptor>& desc_a,
                                   const std::vector<GradientDescriptor>& desc_b, double ratio) {
    static_assert(sizeof(GradientDescriptor) == 128 * sizeof(float), "packed descriptors");
    std::vector<MatchPair> out(desc_a.size());
    int n = 0;
    check(xa_match_ratio(engine(), reinterpret_cast<const float*>(desc_a.data()),
                         static_cast<int>(desc_a.size()), reinterpret_cast<const float*>(desc_b.data()),
                         static_cast<int>(desc_b.size()), ratio, reinterpret_cast<xa_match*>(out.data()),
                         &n));
    out.resize(n);
    return out;
}

// Replacement for xaffine::select_reference (pipeline.cpp:103-120): SIFT and
// both ratio matchings on the device; the scaling coefficient is the
// reference's own host function (pipeline.cpp:70-101, linked unchanged).
ReferenceDecision select_reference(const GrayImage& img1, const GrayImage& img2, int cap) {
    ReferenceDecision d;
    const auto k1 = detect_dog_keypoints(img1, cap), k2 = detect_dog_keypoints(img2, cap);
    const auto f1 = describe_gradient(img1, k1), f2 = describe_gradient(img2, k2);
    const auto m12 = match_ratio(f1.second, f2.second, 0.75);
    const auto m21 = match_ratio(f2.second, f1.second, 0.75);
    if (m12.size() < 2 || m21.size() < 2) {
        const long area1 = static_cast<long>(img1.width) * img1.height;
        const long area2 = static_cast<long>(img2.width) * img2.height;
        d.reference = (area2 > area1) ? 2 : 1;
        return d;
    }
    d.f_forward = scaling_coefficient(f1.first, f2.first, m12, &d.segment_count);
    d.f_backward = scaling_coefficient(f2.first, f1.first, m21);
    d.reference = (d.f_forward >= d.f_backward) ? 1 : 2;
    return d;
}


// Replacement for xaffine::synth_warp_case (eval.cpp:101-141): the harness's
// projective Lanczos render on the device; framing and composed homography
// bit-identical, pixels within the Lanczos tolerance (tests/test_gpu_views.py).
std::pair<GrayImage, AffineMatrix> synth_warp_case(const GrayImage& img, const AffineMatrix& h,
                                                   uint64_t /*seed*/) {
    int W = 0, H = 0;
    AffineMatrix composed;
    check(xa_synth_warp_case(engine(), img.data.data(), img.width, img.height, h.m.data(), XA_F32,
                             nullptr, 0, &W, &H, composed.m.data()));
    GrayImage out(W, H);
    check(xa_synth_warp_case(engine(), img.data.data(), img.width, img.height, h.m.data(), XA_F32,
                             out.data.data(), out.data.size(), &W, &H, composed.m.data()));
    return {std::move(out), composed};
}

}  // namespace b200
}  // namespace xaffine
