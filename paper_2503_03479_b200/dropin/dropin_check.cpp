// dropin_check.cpp — link-time substitution check (built by dropin/Makefile).
//
// Linked from the reference's own objects (image, geometry, orb_pattern,
// pipeline, sift, synthetic) plus xaffine_dropin.cpp in place of warp.cpp and
// orb.cpp, so the UNMODIFIED reference coarse_search (pipeline.cpp:122-152)
// runs its per-view loop on the B200 kernels. Prints one JSON line with the
// per-entry counts of (a) that substituted reference loop and (b) the batched
// xaffine::b200::coarse_search, plus a few drop-in ORB/match outputs for
// tests/test_gpu_dropin.py to compare against the oracle.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <string>
#include <filesystem>
#include <fstream>
#include <tuple>
#include <vector>

#include "synthetic.hpp"
#include "xaffine/eval.hpp"
#include "xaffine/homography.hpp"
#include "xaffine/image_io.hpp"
#include "xaffine/orb.hpp"
#include "xaffine/orb_pattern.hpp"
#include "xaffine/pipeline.hpp"
#include "xaffine/sift.hpp"
#include "xaffine/warp.hpp"

namespace xaffine {
namespace b200 {
CoarseResult coarse_search(const GrayImage&, const GrayImage&, const ParamGrid&, int, double);
std::vector<MatchPair> match_ratio(const std::vector<GradientDescriptor>&,
                                   const std::vector<GradientDescriptor>&, double);
std::vector<Keypoint> detect_dog_keypoints(const GrayImage&, int);
ReferenceDecision select_reference(const GrayImage&, const GrayImage&, int);
std::pair<GrayImage, AffineMatrix> synth_warp_case(const GrayImage&, const AffineMatrix&, uint64_t);
}
}  // namespace xaffine

using namespace xaffine;

static void print_counts(const char* name, const CoarseResult& r) {
    std::printf("\"%s\": [", name);
    for (size_t i = 0; i < r.per_entry_counts.size(); ++i)
        std::printf("%s%d", i ? "," : "", r.per_entry_counts[i].second);
    std::printf("], ");
}

int main() {
    const GrayImage img = testsupport::make_texture(128, 128, 19);
    AffineParams p;
    p.tilt = std::sqrt(2.0);
    p.phi = 0.4;
    const GrayImage target =
        warp_nearest(antialias_tilt(img, p.tilt, p.phi), simulation_from_params(p)).image;
    GridConfig gcfg;
    gcfg.n = 2;
    const ParamGrid grid = build_param_grid(gcfg);
    std::printf("{");
    print_counts("reference_loop_on_dropin", coarse_search(img, target, grid, 300, 0.75));
    print_counts("batched", b200::coarse_search(img, target, grid, 300, 0.75));
    const auto kps = detect_oriented_corners(img, 200);
    const auto [k2, d2] = describe_binary(img, kps);
    std::printf("\"n_kps\": %zu, \"n_desc\": %zu, \"desc0\": [", kps.size(), d2.size());
    for (int w = 0; w < 4 && !d2.empty(); ++w)
        std::printf("%s\"%016llx\"", w ? "," : "", (unsigned long long)d2[0].bits[w]);
    const auto m = match_hamming(d2, d2, 0.75);
    // L2 ratio matcher: the reference's own match_ratio (sift.cpp) vs the
    // routed B200 one on deterministic pseudo-descriptors with near-duplicates
    std::vector<GradientDescriptor> ga(200), gb(260);
    uint32_t st = 12345u;
    auto rnd = [&st]() { st = st * 1664525u + 1013904223u; return (st >> 8) * (1.0f / 16777216.0f); };
    for (auto& g : ga)
        for (auto& v : g.values) v = 40.f * rnd();
    for (size_t j = 0; j < gb.size(); ++j)
        for (int k = 0; k < 128; ++k)
            gb[j].values[k] = j % 3 == 0 && j / 3 < ga.size() ? ga[j / 3].values[k] + 0.5f * rnd()
                                                              : 40.f * rnd();
    int l2_equal = 1;
    size_t l2_n = 0;
    for (double r : {0.6, 0.8, 1.0}) {
        const auto x = match_ratio(ga, gb, r), y = b200::match_ratio(ga, gb, r);
        l2_n += x.size();
        l2_equal &= x.size() == y.size();
        for (size_t i = 0; l2_equal && i < x.size(); ++i)
            l2_equal &= x[i].idx_a == y[i].idx_a && x[i].idx_b == y[i].idx_b &&
                        std::memcmp(&x[i].distance, &y[i].distance, sizeof(float)) == 0;
    }
    // SIFT detector: the reference's sift.cpp vs the routed B200 one (as a
    // multiset: orientations of one extremum have no defined order)
    auto key = [](const Keypoint& k) {
        return std::make_tuple(-k.response, k.y, k.x, k.orientation, k.octave_scale);
    };
    auto dref = detect_dog_keypoints(img, 400), dgpu = b200::detect_dog_keypoints(img, 400);
    std::sort(dref.begin(), dref.end(), [&](const Keypoint& a, const Keypoint& b) { return key(a) < key(b); });
    std::sort(dgpu.begin(), dgpu.end(), [&](const Keypoint& a, const Keypoint& b) { return key(a) < key(b); });
    int sift_equal = dref.size() == dgpu.size();
    for (size_t i = 0; sift_equal && i < dref.size(); ++i) sift_equal &= key(dref[i]) == key(dgpu[i]);
    // reference selection: the reference's select_reference vs the routed one
    const GrayImage big = testsupport::make_texture(256, 256, 3);
    const GrayImage small = resize_bilinear(big, 128, 128);
    const ReferenceDecision sr = select_reference(big, small, 500);
    const ReferenceDecision sg = b200::select_reference(big, small, 500);
    const ReferenceDecision sw = b200::select_reference(small, big, 500);
    // the harness's projective render: the reference's eval.cpp vs the routed one
    AffineMatrix hs;
    hs.m = {0.9, -0.25, 12.0, 0.2, 0.95, -6.0, 8e-4, -5e-4, 1.0};
    const auto [sref, cref] = synth_warp_case(img, hs, 0);
    const auto [sgpu, cgpu] = b200::synth_warp_case(img, hs, 0);
    double synth_diff = sref.data.size() == sgpu.data.size() ? 0.0 : 1e30;
    for (size_t i = 0; synth_diff < 1e30 && i < sref.data.size(); ++i)
        synth_diff = std::max(synth_diff, (double)std::fabs(sref.data[i] - sgpu.data[i]));
    const int synth_frame = sref.width == sgpu.width && sref.height == sgpu.height && cref.m == cgpu.m;
    // image file I/O: the reference's own eval.cpp load_sequence over files
    // written by the drop-in save_image (PGM and PNG) -> routed load_image
    const std::filesystem::path dir = std::filesystem::temp_directory_path() / "xa_dropin_seq";
    std::filesystem::create_directories(dir);
    save_image(img, (dir / "img1.pgm").string());
    save_image(target, (dir / "img2.png").string());
    std::ofstream((dir / "H1to2p").string()) << "1 0 3\n0 1 -2\n0 0 1\n";
    const Sequence seq = load_sequence(dir.string());
    auto quantized_equal = [](const GrayImage& a, const GrayImage& b) {
        if (a.width != b.width || a.height != b.height) return 0;
        for (size_t i = 0; i < a.data.size(); ++i) {
            const long q = std::min(255L, std::max(0L, std::lround(a.data[i])));
            if ((float)q != b.data[i]) return 0;
        }
        return 1;
    };
    const int io_ok = seq.images.size() == 2 && quantized_equal(img, seq.images[0]) &&
                      quantized_equal(target, seq.images[1]) && seq.homographies.count(2) &&
                      seq.homographies.at(2).m[2] == 3.0;
    int io_error = 0;
    try {
        load_image((dir / "missing.png").string());
    } catch (const IoError&) {
        io_error = 1;
    }
    std::filesystem::remove_all(dir);
    // the reference's evaluation harness (eval.cpp run_benchmark + report
    // writers, pipeline.cpp match_images / asift_baseline / fine_only_match)
    // on the drop-in: the cases of proj/tests/test_eval.cpp:189-268
    PipelineConfig fc;
    fc.max_points_coarse = 500;
    fc.max_points_fine = 300;
    fc.grid.n = 1;
    Sequence self;
    self.name = "self";
    self.images.push_back(testsupport::make_texture(192, 192, 7));
    self.images.push_back(self.images[0]);
    self.homographies[2] = AffineMatrix::identity();
    const EvalReport rep =
        run_benchmark(self, {Method::Proposed, Method::BaselineAsift, Method::FineOnly}, fc);
    std::string rows = "[";
    for (size_t i = 0; i < rep.rows.size(); ++i) {
        const EvalRow& r = rep.rows[i];
        char buf[512];
        std::snprintf(buf, sizeof buf, "%s[\"%s\", %d, %d, %.17g, %.17g, %.3f]", i ? ", " : "",
                      r.method.c_str(), (int)r.error.empty(), r.points,
                      r.precision_pct ? *r.precision_pct : -1.0,
                      r.inlier_ratio_pct ? *r.inlier_ratio_pct : -1.0, r.time_ms);
        rows += buf;
    }
    rows += "]";
    Sequence mixed;
    mixed.name = "mixed";
    mixed.images.push_back(testsupport::make_texture(160, 160, 9));
    mixed.images.push_back(GrayImage(160, 160, 100.f));
    const EvalReport frep = run_benchmark(mixed, {Method::FineOnly}, fc);
    const int fail_row = frep.rows.size() == 1 && !frep.rows[0].error.empty() && !frep.rows[0].precision_pct;
    const std::string csv = report_to_csv(rep);
    const int csv_ok = csv.rfind("sequence,pair,method,points,precision_pct,inlier_ratio_pct,time_ms,error\n", 0) == 0 &&
                       report_to_json(rep).at("rows").size() == 3;
    // end-to-end synthetic case (test_eval.cpp:270-283)
    const GrayImage e2e_img = testsupport::make_texture(256, 256, 13);
    AffineParams ep;
    ep.tilt = 2.0;
    ep.phi = 0.4;
    const auto [e2e_warped, e2e_h] = synth_warp_case(e2e_img, invert(affine_from_params(ep)));
    PipelineConfig ec;
    ec.max_points_coarse = 600;
    ec.max_points_fine = 500;
    const MatchResult er = match_images(e2e_img, e2e_warped, ec);
    const auto efinal = er.final_matches(true);
    const double e2e_prec = efinal.empty() ? -1.0 : precision(efinal, e2e_h, std::sqrt(3.0));
    std::printf("], \"self_matches\": %zu, \"checksum\": \"%016llx\", \"l2_equal\": %d, "
                "\"l2_matches\": %zu, \"sift_equal\": %d, \"sift_n\": %zu, "
                "\"selref\": [%d, %.17g, %.17g, %d], \"selref_b200\": [%d, %.17g, %.17g, %d], "
                "\"selref_b200_swapped\": %d, \"synth_frame\": %d, \"synth_maxdiff\": %.9g, "
                "\"io_sequence\": %d, \"io_error\": %d, \"bench_rows\": %s, \"bench_fail_row\": %d, "
                "\"report_ok\": %d, \"e2e_final\": %zu, \"e2e_precision\": %.17g}\n", m.size(),
                (unsigned long long)orb_pattern_checksum(), l2_equal, l2_n, sift_equal, dref.size(),
                sr.reference, sr.f_forward, sr.f_backward, sr.segment_count, sg.reference,
                sg.f_forward, sg.f_backward, sg.segment_count, sw.reference, synth_frame, synth_diff, io_ok,
                io_error, rows.c_str(), fail_row, csv_ok, efinal.size(), e2e_prec);
    return 0;
}
