/* oracle/xa_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference hot path (affine view simulation, ORB,
 * Hamming ratio matching, coarse pose search) in plain C. It is the parity
 * checker for the CUDA path and the "port" CPU baseline; it is never linked
 * into, or called by, the product library. The same `orc_*` interface is
 * exported by oracle/_ref/libxaref.so (the reference itself, see
 * oracle/ref_shim.cpp), which pins this restatement in tests/test_oracle.py.
 *
 * Conventions shared by both implementations:
 *   images      float32, row-major, width*height, no padding
 *   matrices    9 doubles, row-major 3x3 (reference AffineMatrix)
 *   params      6 doubles (psi, tilt, phi, scale, tx, ty) (AffineParams)
 *   keypoints   5 floats (x, y, response, orientation, octave_scale)
 *   descriptors 4 uint64 words, bit i in word i>>6, LSB first
 *   matches     3 int32 (idx_a, idx_b, distance)
 * Variable-length outputs are malloc'd and released with orc_free().
 * Status: 0 ok, -1 error (message in orc_last_error()).
 */
#ifndef XA_ORACLE_H
#define XA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
void orc_free(void* p);
const char* orc_kind(void);

uint64_t orc_pattern_checksum(void);
void orc_pattern(int8_t* out1024);

int orc_make_texture(int w, int h, uint64_t seed, float* out);
int orc_make_checkerboard(int w, int h, int cell, float* out);

int orc_gaussian_blur(const float* img, int w, int h, double sigma, float* out);
int orc_resize_bilinear(const float* img, int w, int h, int nw, int nh, float* out);
int orc_antialias_tilt(const float* img, int w, int h, double t, double phi, float* out);
double orc_lanczos_kernel(double x, int a);
double orc_sample_lanczos(const float* img, int w, int h, double x, double y, int a);
int orc_warp(int mode, const float* img, int w, int h, const double* m, int a, float** out,
             int* W, int* H, double* tx, double* ty, double* fwd);

/* synth_warp_case (eval.cpp:101-141): projective Lanczos render + framing;
   fails with the reference's EvalError messages */
int orc_synth_warp_case(const float* img, int w, int h, const double* hm, float** out, int* W,
                        int* H, double* composed);
int orc_detect(const float* img, int w, int h, int max_points, float** kps, int* n);
int orc_describe(const float* img, int w, int h, const float* kps, int n, float** okps,
                 uint64_t** odesc, int* nout);
int orc_match(const uint64_t* a, int na, const uint64_t* b, int nb, double ratio, int32_t** out,
              int* n);
/* match_ratio (sift.cpp:388-418): out[3*i] = idx_a, out[3*i+1] = idx_b,
   out[3*i+2] = the float distance's bit pattern */
int orc_match_ratio(const float* a, int na, const float* b, int nb, double ratio, int32_t** out,
                    int* n);

/* fine stage: detect_dog_keypoints (sift.cpp:290-358), describe_gradient
   (sift.cpp:360-386); keypoints as 5 floats, descriptors as 128 floats */
int orc_detect_dog(const float* img, int w, int h, int max_points, float** kps, int* n);
int orc_describe_gradient(const float* img, int w, int h, const float* kps, int n, float** okps,
                          float** odesc, int* nout);

/* reference selection (pipeline.cpp:70-120): matches as orc_match_ratio's
   triples; segments may be NULL */
int orc_scaling_coefficient(const float* kps_a, int na, const float* kps_b, int nb,
                            const int32_t* matches, int n, double* f, int* segments);
int orc_select_reference(const float* img1, int w1, int h1, const float* img2, int w2, int h2,
                         int cap, int* reference, double* f_forward, double* f_backward,
                         int* segments);

/* asift_baseline (pipeline.cpp:298-343) up to RANSAC: out = 5 doubles per
   correspondence (x1, y1, x2, y2, distance) */
int orc_asift_correspondences(const float* img1, int w1, int h1, const float* img2, int w2, int h2,
                              const double* grid, int n, int cap, double ratio, int a,
                              double** out, int* nout);

int orc_build_grid(double a, int n, double b_deg, double delta_s, double** params, int* count);
int orc_simulation_from_params(const double* p, double* m);
int orc_affine_from_params(const double* p, double* m);
int orc_invert(const double* m, double* out);
int orc_filter_to_content(const float* kps, int n, const double* back, int src_w, int src_h,
                          double margin, float** out, int* nout);
int orc_coarse_search(const float* ref, int w, int h, const float* tgt, int tw, int th,
                      const double* grid, int n, int max_points, double ratio, int mode,
                      int* counts, int* kp_counts, int* best);

/* Restatement-only stage probes (used to localise GPU mismatches). */
int orc_detect_candidates(const float* img, int w, int h, float threshold, int32_t** xyl,
                          float** score, int* n);
int orc_corner_measures(const float* level, int w, int h, const int32_t* xy, int n, float* resp,
                        float* orient);
int orc_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
