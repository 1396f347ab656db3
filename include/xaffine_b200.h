/* include/xaffine_b200.h — C-ABI of the B200 coarse-search hot path.
 *
 * This is the drop-in boundary. The reference exposes the hot
 * path as C++ free functions in namespace xaffine (proj/include/xaffine/*.hpp);
 * a C++ wrapper with the reference's exact signatures
 * (paper_2503_03479_b200/dropin/xaffine_dropin.cpp) and
 * the Python mirror (paper_2503_03479_b200/api.py) both bind to these entry
 * points. Every function that replaces a reference interface cites it.
 *
 * Conventions
 *   - Status codes: XA_OK (0) or a negative XA_E* code; xa_last_error() gives
 *     the thread's last message. The wrappers re-raise the reference's
 *     exception types (GeometryError, PipelineError) from these codes.
 *   - Images are row-major, width*height, no padding. XA_F32 images carry the
 *     reference GrayImage values; XA_U8 images are 8-bit grayscale.
 *   - xa_keypoint / xa_match / xa_params are layout-identical to the reference
 *     Keypoint, MatchPair and AffineParams structs (features.hpp:11-39,
 *     geometry.hpp:34-41), so C++ callers may pass their vectors' storage.
 *   - Descriptors are 4 x uint64 words per keypoint, bit i in word i>>6,
 *     LSB first (features.hpp:20-25).
 *   - "Host" entry points take host buffers and synchronise before returning.
 *     "_device" entry points take device pointers, enqueue on the given CUDA
 *     stream and return immediately.
 *   - An engine owns a CUDA stream and a grow-only device workspace; it is not
 *     thread-safe. Use one engine per host thread (the reference calls the hot
 *     path concurrently from parallel_for workers, parallel.hpp:22-36).
 */
#ifndef XAFFINE_B200_H
#define XAFFINE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    XA_OK = 0,
    XA_EINVAL = -1,    /* invalid argument (e.g. tilt < 1, empty grid) */
    XA_ESINGULAR = -2, /* singular matrix (reference GeometryError from invert) */
    XA_ECUDA = -3,     /* CUDA runtime error */
    XA_ENOMEM = -4,    /* device allocation failed */
    XA_ECAPACITY = -5, /* output or internal capacity exceeded */
    XA_EPIPELINE = -6, /* reference PipelineError */
    XA_EEVAL = -7,     /* reference EvalError (eval.hpp:14-16) */
    XA_EIO = -8,       /* reference IoError (image_io.hpp:10-12) */
    XA_EHOMOGRAPHY = -9 /* reference HomographyError (homography.hpp:11-13) */
};

enum { XA_U8 = 0, XA_F32 = 1 };             /* pixel types */
enum { XA_NEAREST = 0, XA_LANCZOS = 1 };    /* view resamplers */

typedef struct xa_engine xa_engine;

typedef struct {
    float x, y, response, orientation, octave_scale;
} xa_keypoint; /* == xaffine::Keypoint (features.hpp:11-17) */

typedef struct {
    int32_t idx_a, idx_b;
    float distance;
} xa_match; /* == xaffine::MatchPair (features.hpp:35-39) */

typedef struct {
    double psi, tilt, phi, scale, tx, ty;
} xa_params; /* == xaffine::AffineParams (geometry.hpp:34-41) */

typedef struct {
    double x1, y1; /* reference / Image 1 coordinates */
    double x2, y2; /* target coordinates */
    double distance;
} xa_correspondence; /* == xaffine::Correspondence (pipeline.hpp:46-50) */

/* ---- engine ------------------------------------------------------------ */
int xa_engine_create(int device, xa_engine** out);
int xa_engine_destroy(xa_engine* e);
const char* xa_last_error(void);
int xa_version(void);
/* The engine's CUDA stream (cudaStream_t) for callers that order work on it. */
void* xa_engine_stream(xa_engine* e);
/* Bytes of device workspace currently held by the engine. */
size_t xa_engine_workspace_bytes(xa_engine* e);

/* ---- host geometry (bit-identical to the reference's double arithmetic) - */
/* replaces xaffine::simulation_from_params (geometry.hpp:79, geometry.cpp:51-58) */
int xa_simulation_from_params(const xa_params* p, double m[9]);
/* replaces xaffine::affine_from_params (geometry.hpp:58, geometry.cpp:42-49) */
int xa_affine_from_params(const xa_params* p, double m[9]);
/* replaces xaffine::invert (geometry.hpp:63, geometry.cpp:65-78) */
int xa_invert(const double m[9], double out[9]);
/* replaces xaffine::build_param_grid (geometry.hpp:73, geometry.cpp:90-112) */
int xa_build_param_grid(double a, int n, double b_deg, double delta_s, xa_params* out, int cap,
                        int* count);
/* Output frame of a warp by m over a w x h source: size, framing translation
   and the forward map WarpResult::forward (warp.cpp:13-42, :92-95). */
int xa_warp_frame(const double m[9], int w, int h, int* W, int* H, double* tx, double* ty,
                  double forward[9]);

/* ---- host-buffer entry points (reference semantics) --------------------- */
/* replaces xaffine::gaussian_blur (image.hpp:59, image.cpp:25-49) */
int xa_gaussian_blur(xa_engine* e, const float* img, int w, int h, double sigma, float* out);
/* replaces xaffine::resize_bilinear (image.hpp:62, image.cpp:51-70) */
int xa_resize_bilinear(xa_engine* e, const float* img, int w, int h, int nw, int nh, float* out);
/* replaces xaffine::antialias_tilt (warp.hpp:31, warp.cpp:128-158) */
int xa_antialias_tilt(xa_engine* e, const float* img, int w, int h, double t, double phi,
                      float* out);
/* replaces xaffine::warp_nearest / warp_lanczos (warp.hpp:25-27, warp.cpp:86-126).
   `out` holds out_cap floats; the frame (W, H, tx, ty, forward) is returned
   as by xa_warp_frame. `a` is the Lanczos order (ignored for nearest). */
int xa_warp(xa_engine* e, int mode, const float* img, int w, int h, const double m[9], int a,
            float* out, size_t out_cap, int* W, int* H, double* tx, double* ty,
            double forward[9]);
/* replaces xaffine::synth_warp_case (eval.hpp:56-60, eval.cpp:101-141): renders
   img under the homography hm (row-major 3x3) with Lanczos-4 in the warp
   module's half-pixel framing. out_type XA_F32: `out` receives the reference's
   float image (W*H, out_cap elements); XA_U8: the lround + clamp bytes that
   save_image writes (image_io.cpp:17-20). out == NULL queries the frame only.
   composed (may be NULL) receives the framed homography. XA_EEVAL for the
   reference's EvalError cases (degenerate, unbounded, not invertible). */
int xa_synth_warp_case(xa_engine* e, const float* img, int w, int h, const double hm[9],
                       int out_type, void* out, size_t out_cap, int* W, int* H, double composed[9]);
/* replaces xaffine::detect_oriented_corners (orb.hpp:14, orb.cpp:182-210).
   `out` holds cap keypoints; *n receives min(found, max_points). */
int xa_detect_oriented_corners(xa_engine* e, const float* img, int w, int h, int max_points,
                               xa_keypoint* out, int cap, int* n);
/* replaces xaffine::describe_binary (orb.hpp:19-21, orb.cpp:212-248).
   out_kps / out_desc hold n entries; *n_out receives the survivors. */
int xa_describe_binary(xa_engine* e, const float* img, int w, int h, const xa_keypoint* kps,
                       int n, xa_keypoint* out_kps, uint64_t* out_desc, int* n_out);
/* replaces xaffine::match_hamming (orb.hpp:23-27, orb.cpp:250-272).
   `out` holds na entries; result sorted by idx_a. */
int xa_match_hamming(xa_engine* e, const uint64_t* a, int na, const uint64_t* b, int nb,
                     double ratio, xa_match* out, int* n_out);
/* replaces xaffine::detect_dog_keypoints (sift.hpp:12-13, sift.cpp:290-358),
   the fine stage's DoG detector. `out` holds cap keypoints; *n receives
   min(found, max_points), sorted by (response desc, y, x); keypoints of one
   extremum differing only in orientation are ordered by orientation. */
int xa_detect_dog_keypoints(xa_engine* e, const float* img, int w, int h, int max_points,
                            xa_keypoint* out, int cap, int* n);
/* replaces xaffine::describe_gradient (sift.hpp:18-23, sift.cpp:360-386):
   out_kps holds n keypoints and out_desc n x 128 floats; *n_out receives the
   survivors of the border filter. */
int xa_describe_gradient(xa_engine* e, const float* img, int w, int h, const xa_keypoint* kps, int n,
                         xa_keypoint* out_kps, float* out_desc, int* n_out);
/* replaces xaffine::match_ratio (sift.hpp:25-30, sift.cpp:388-418), the fine
   stage's L2 ratio matcher over 128-float gradient descriptors (a[na][128],
   b[nb][128], row-major). `out` holds na entries; result sorted by idx_a,
   distance = the Euclidean distance as float. */
int xa_match_ratio(xa_engine* e, const float* a, int na, const float* b, int nb, double ratio,
                   xa_match* out, int* n_out);
/* replaces xaffine::coarse_search (pipeline.hpp:86-88, pipeline.cpp:122-152),
   batched: every grid entry in a handful of launches. Views are simulated
   with `warp_mode` (the reference coarse stage uses XA_NEAREST) and quantised
   to uint8 before ORB. counts[n] receives the per-entry match counts,
   kp_counts[n] (optional) the described keypoints per entry, *best the
   winning entry (strict > in grid order, pipeline.cpp:142-150). */
int xa_coarse_search(xa_engine* e, int pixel_type, const void* ref, int w, int h,
                     const void* target, int tw, int th, const xa_params* grid, int n,
                     int max_points, double ratio, int warp_mode, int32_t* counts,
                     int32_t* kp_counts, int32_t* best);

/* Batched coarse_search over n_pairs image pairs (BASELINE config 5: 64
   pairs): pair p runs coarse_search(refs[p], targets[p], grid) exactly as the
   reference does (pipeline.cpp:122-152; the reference loops pairs one call at
   a time). Every reference image is w x h and every target tw x th, so all
   pairs share one view plan. counts / kp_counts are [n_pairs][n] (row p =
   pair p's per-entry counts), best[n_pairs] the winning entry per pair
   (strict > in grid order). Capacity overflows are retried internally with
   larger candidate buffers. */
int xa_coarse_search_batch(xa_engine* e, int pixel_type, const void* const* refs, int w, int h,
                           const void* const* targets, int tw, int th, int n_pairs,
                           const xa_params* grid, int n, int max_points, double ratio,
                           int warp_mode, int32_t* counts, int32_t* kp_counts, int32_t* best);

/* ---- multi-GPU (replaces the reference's host-thread
   parallel_for, parallel.hpp:22-36 / pipeline.cpp:130) --------------------
   Pairs are split into contiguous blocks, one per GPU; each block runs
   through that GPU's batched pipeline; counts are gathered. Results are
   identical to xa_coarse_search_batch for any number of GPUs. */
/* One process, one engine per device (each driven by its own host thread). */
int xa_coarse_search_multi(xa_engine* const* engines, int n_engines, int pixel_type,
                           const void* const* refs, int w, int h, const void* const* targets, int tw,
                           int th, int n_pairs, const xa_params* grid, int n, int max_points,
                           double ratio, int warp_mode, int32_t* counts, int32_t* kp_counts,
                           int32_t* best);
/* One process per GPU: every rank passes the whole job (all n_pairs host
   pointers; only its block is read) and its NCCL communicator (ncclComm_t);
   the per-pair results of all ranks are all-gathered over NCCL so every rank
   returns the whole job's counts / kp_counts / best. */
int xa_coarse_search_nccl(xa_engine* e, void* nccl_comm, int rank, int world, int pixel_type,
                          const void* const* refs, int w, int h, const void* const* targets, int tw,
                          int th, int n_pairs, const xa_params* grid, int n, int max_points,
                          double ratio, int warp_mode, int32_t* counts, int32_t* kp_counts,
                          int32_t* best);
/* NCCL bootstrap for callers without one: id is an ncclUniqueId (128 bytes)
   created on one rank and shared with the others out of band. */
int xa_nccl_unique_id(void* id, size_t bytes);
int xa_nccl_comm_init(void** comm, int world, const void* id, int rank, int device);
int xa_nccl_comm_destroy(void* comm);
const char* xa_multi_last_error(void);

/* ---- device entry points (inputs resident in HBM, stream-ordered) ------- */
/* Same as xa_coarse_search with device-resident images; d_counts and
   d_kp_counts (optional) are device int32[n]. Does not synchronise. */
int xa_coarse_search_device(xa_engine* e, int pixel_type, const void* d_ref, int w, int h,
                            const void* d_target, int tw, int th, const xa_params* grid, int n,
                            int max_points, double ratio, int warp_mode, int32_t* d_counts,
                            int32_t* d_kp_counts, void* stream);
/* Device-resident batch (see xa_coarse_search_batch): d_refs / d_targets are
   host arrays of n_pairs device pointers; d_counts / d_kp_counts (optional)
   device int32[n_pairs * n]. The pairs run in chunks of K pairs (as many as
   fit in half of the free device memory, at most 8, or XA_BATCH_PAIRS) through
   one CUDA graph that is replayed while the arguments stay the same. Does not
   synchronise; capacity overflows are reported by xa_engine_check. */
int xa_coarse_search_batch_device(xa_engine* e, int pixel_type, const void* const* d_refs, int w,
                                  int h, const void* const* d_targets, int tw, int th, int n_pairs,
                                  const xa_params* grid, int n, int max_points, double ratio,
                                  int warp_mode, int32_t* d_counts, int32_t* d_kp_counts,
                                  void* stream);
/* Batched view simulation (BASELINE config 3): anti-alias blur + resampling of
   one uint8 source into n uint8 views. Returns the total output bytes needed
   in *out_bytes when d_out is NULL; otherwise writes view i at
   d_out + offsets[i] (offsets[n] filled by this call on the host). */
int xa_simulate_views_device(xa_engine* e, const uint8_t* d_src, int w, int h,
                             const xa_params* views, int n, int warp_mode, uint8_t* d_out,
                             int64_t* offsets, int* widths, int* heights, size_t* out_bytes,
                             void* stream);
/* Brute-force Hamming top-2 with ratio test (BASELINE config 4). For every
   query: d_best_idx (uint32), d_best (uint16), d_second (uint16, clamped to
   256); *d_count (int32) receives the number passing best < ratio*second. */
int xa_match_hamming_device(xa_engine* e, const uint64_t* d_a, int na, const uint64_t* d_b,
                            int nb, double ratio, uint32_t* d_best_idx, uint16_t* d_best,
                            uint16_t* d_second, int32_t* d_count, void* stream);

/* L2 ratio matcher on device-resident descriptors. For every query:
   d_best_idx (int32, -1 when nb == 0), d_dist (float, sqrt of the best
   squared distance), d_keep (uint8, 1 iff it passes the ratio test);
   *d_count (int32) receives the number kept. */
int xa_match_ratio_device(xa_engine* e, const float* d_a, int na, const float* d_b, int nb,
                          double ratio, int32_t* d_best_idx, float* d_dist, uint8_t* d_keep,
                          int32_t* d_count, void* stream);

/* Dual-simulation ASIFT baseline (replaces asift_baseline, pipeline.cpp:298-343,
   up to its RANSAC screen, which stays on the host): both images simulated at
   every grid entry (scale forced to 1), SIFT per view, L2 ratio matching of
   every view pair, merge with 2-px duplicate suppression in (view of image 1,
   view of image 2) order. Writes up to cap correspondences; *n_out is the
   total (XA_ECAPACITY when it exceeds cap). */
int xa_asift_correspondences(xa_engine* e, const float* img1, int w1, int h1, const float* img2,
                             int w2, int h2, const xa_params* grid, int n, int max_points,
                             double ratio, int lanczos_a, xa_correspondence* out, int cap,
                             int* n_out);

/* ---- introspection ------------------------------------------------------ */
/* Synchronise the engine and report (then clear) capacity overflows raised by
   earlier _device calls: XA_OK or XA_ECAPACITY. */
int xa_engine_check(xa_engine* e);
/* Stage profiling: when on, CUDA events are recorded on the call's stream
   between the kernels of coarse_search / match_hamming_device; stage_times
   returns the per-stage milliseconds of the last such call (names are static
   strings: antialias, warp, pyramid, fast_nms, measures, select, describe,
   match, collect, hamming). */
int xa_engine_set_profiling(xa_engine* e, int on);
/* ORB counters of the last detect / coarse call, 5 int32 per image (image 0 =
   coarse target, 1..n = views): candidates, thr-20 survivors, thr-7 survivors
   (counted only for auto-relaxed images), detected, described. Reads up to
   cap_images images. */
int xa_engine_orb_counters(xa_engine* e, int cap_images, int32_t* out, int* n_images);
int xa_engine_stage_times(xa_engine* e, int cap, float* ms, const char** names, int* n);
/* Kernel launches issued by the last host/device entry point on this engine. */
int xa_engine_last_launches(xa_engine* e);
/* Diagnostics: the first `floats` floats of the engine's ORB pyramid buffer
   (levels of the last detect / describe / coarse call; per level a pitched
   float raster, pitch = width rounded up to 4, levels 32-float aligned). */
int xa_engine_read_pyramid(xa_engine* e, float* out, size_t floats);
/* FNV-1a checksum of the device-resident rBRIEF pattern (orb_pattern.cpp:270-285). */
uint64_t xa_pattern_checksum(void);
/* Number of glibc cosf/sinf fixups compiled in (see tools/gen_trig_table.c). */
int xa_trig_fixups(void);

/* ---- image file I/O of the evaluation harness (host only) -----------------
   Replaces xaffine::load_image / save_image / save_png_rgb
   (proj/include/xaffine/image_io.hpp:14-24, proj/src/image_io.cpp).
   xa_load_image: PGM/PPM/PNM (P2, P3, P5, P6) or PNG by extension, as a float
   grayscale raster (RGB -> (float)(0.299 R + 0.587 G + 0.114 B) in double).
   Call with out = NULL to get *w, *h; XA_ECAPACITY if cap < w*h; XA_EIO for
   unreadable / unsupported files (the reference's IoError).
   xa_save_image: 8-bit grayscale .pgm (P5) or .png, each pixel quantised as
   lround + clamp to [0, 255] (image_io.cpp:18-21). xa_quantize: that rule on
   a host buffer. */
int xa_load_image(const char* path, float* out, size_t cap, int* w, int* h);
int xa_save_image(const float* img, int w, int h, const char* path);
int xa_save_png_rgb(const uint8_t* rgb, int w, int h, const char* path);
int xa_quantize(const float* img, size_t n, uint8_t* out);

/* ---- geometric verification (host only) ------------------------------------
   Replaces xaffine::fit_homography_dlt / estimate_homography_ransac
   (proj/include/xaffine/homography.hpp:27-39, proj/src/homography.cpp).
   pts: n correspondences as (x1, y1, x2, y2) doubles. h: row-major 3x3 with
   h22 = 1 when nonzero. RANSAC: symmetric-transfer threshold, max_iters,
   confidence and seed as RansacConfig (homography.hpp:20-25); inliers gets the
   ascending inlier indices (XA_ECAPACITY if more than cap; *n_inliers is set
   either way). XA_EHOMOGRAPHY: fewer than 4 points / no consensus;
   XA_ESINGULAR: singular final model (the reference's GeometryError). */
int xa_fit_homography_dlt(const double* pts, int n, double h[9]);
int xa_estimate_homography_ransac(const double* pts, int n, double threshold, int max_iters,
                                  double confidence, uint64_t seed, double h[9], int32_t* inliers,
                                  int cap, int* n_inliers);

#ifdef __cplusplus
}
#endif
#endif
