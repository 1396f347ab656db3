// xa_kernels.h — host-visible launch tables and launcher declarations shared
// between the kernel translation units and the engine (xa_engine.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "xa_common.cuh"

namespace xa {

// XA_PIX_PYR0: level 0 is already in the pyramid buffer (written by the view
// resampler); k_pyramid builds levels 1.. from it.
enum { XA_PIX_U8 = 0, XA_PIX_F32 = 1, XA_PIX_PYR0 = 2 };
constexpr int kMaxBlurTaps = 257;

// One tap of the directional blur: offset of the bilinear cell and its
// fractional weights (exact per view, see k_antialias).
struct BlurTap {
    double k;       // normalised Gaussian weight (double, warp.cpp:137-141)
    double px, py;  // i*dx, i*dy (the per-pixel tap coordinate is x + i*dx, warp.cpp:152)
    int ox, oy;     // floor(i*dx), floor(i*dy) (host stencil folding)
    float wx, wy;   // (float) fractional parts (host stencil folding)
};

// Pipeline blur stencil cell: integer offset and combined weight.
struct BlurCell {
    int ox, oy;
    float w;
    int pad;
};
constexpr int kMaxBlurCells = 1024;
constexpr int kMaxBlurReach = 32;  // |offset| bound of the stencil kernel
constexpr int kBlurTW = 64, kBlurTH = 64;  // k_blur_stencil output tile
// largest staged tile, two copies (as loaded + shifted by one float):
// 2 x (64 + 64 + 6 -> 132 columns, 16-byte rows) x (64 + 64) rows
constexpr int kBlurSmemFloats = 2 * ((kBlurTW + 2 * kMaxBlurReach + 6) & ~3) * (kBlurTH + 2 * kMaxBlurReach);

struct BlurView {
    int ntaps, aligned, tap_off, pad;
    long long out_off;  // float offset of this view's blurred image
    int cell_off, ncells;
    int bx0, bx1, by0, by1;  // stencil offset bounds (inclusive)
    // k_blur_runs: the stencil as runs along its long axis (rowmode: runs of
    // cells sharing oy, contiguous in ox; else sharing ox, contiguous in oy)
    int rowmode, run_off, nruns, rw_off, nrw;
    int pad2;
};

// One run of k_blur_runs: cells (m, a + j) for j < 4 nblk (rowmode: m = oy,
// minor = ox), weights rw[woff + j], zero-padded to blocks of 4; `major` holds
// the run start's offset in the staged tile (host-resolved).
struct BlurRun {
    int major, a, nblk, woff;
};
// k_blur_runs staged tile: row stride SW (odd: conflict-free lanes across rows)
__host__ __device__ inline void blur_runs_geometry(const BlurView& v, int& SW, int& SH) {
    SW = (64 + v.bx1 - v.bx0 + (v.rowmode ? 3 : 0)) | 1;
    SH = 64 + v.by1 - v.by0 + (v.rowmode ? 0 : 3);
}
constexpr int kMaxBlurRuns = 80, kMaxBlurRunW = 1024;

struct WarpView {
    double back[6];     // invert(forward), top rows (warp.cpp:95)
    int W, H;           // output frame
    int sw, sh;         // source dims
    long long out_off;  // element offset of the output view
    const void* src;    // source (blurred f32 or original u8)
    int src_type;
    int tile_start;     // first tile of this view in the flattened launch
    int tiles_x;
    int tile;           // output tile width (Lanczos: 64/32/16/8; nearest: 32)
    int pyr_pitch;      // pyramid level-0 row pitch (floats) when the view is also
    int tile_h;         // output tile height (tile or tile / 2)
    long long pyr_off;  // written as ORB level 0 (launch_warp pyr != nullptr)
    int lz_res;         // Lanczos footprint row stride mod 32 (floats, multiple of 4)
    int lz_pw;          // Lanczos warp patch width (log2; height = 32 >> width)
    int lz_stride;      // the view's footprint row stride (floats) = its tensor-map box width
    int lz_box_h;       // footprint rows of its largest tile = box height
    int tmap_idx;       // tensor map of the float source for this view (-1: none)
    int pad_;
};
constexpr int kLanczosSmemFloats = 16384;  // per-CTA source footprint cap (64 KB)
// Lanczos footprint layout: one copy, staged from the 16-byte aligned column
// at or left of the box, with 3 (alignment) + 2 (10-float tap window) extra
// columns; rows are 16-byte aligned and 4 (mod 8) floats apart (bank spread).
// The host picks the residue of the stride mod 32 per view (lz_res) so that a
// warp's 32 tap windows fall in distinct 8-byte banks (lanczos_bank_plan).
__host__ __device__ inline int lanczos_stride(int bw, int res) {
    const int s = (bw + 3 + 2 + 3) & ~3;
    return s + ((res - s) & 31);
}
// half-pixel bilinear resize sample (image.cpp:55-66), exact rounding
template <class T>
__device__ __forceinline__ float resize_px(const T* in, int w, int h, double sx, double sy, int x,
                                           int y) {
    const double fy = dsub(dmul(dadd((double)y, 0.5), sy), 0.5);
    const int y0 = (int)floor(fy);
    const float wy = (float)dsub(fy, (double)y0);
    const double fx = dsub(dmul(dadd((double)x, 0.5), sx), 0.5);
    const int x0 = (int)floor(fx);
    const float wx = (float)dsub(fx, (double)x0);
    const int xa = clampi(x0, 0, w - 1), xb = clampi(x0 + 1, 0, w - 1);
    const int ya = clampi(y0, 0, h - 1), yb = clampi(y0 + 1, 0, h - 1);
    const float v00 = ld_px(in, (size_t)ya * w + xa), v10 = ld_px(in, (size_t)ya * w + xb);
    const float v01 = ld_px(in, (size_t)yb * w + xa), v11 = ld_px(in, (size_t)yb * w + xb);
    const float iwx = fsub(1.f, wx), iwy = fsub(1.f, wy);
    return fadd(fmul(iwy, fadd(fmul(iwx, v00), fmul(wx, v10))),
                fmul(wy, fadd(fmul(iwx, v01), fmul(wx, v11))));
}

// ---- launchers (each returns the number of kernels it enqueued) ----------
int launch_antialias(const BlurView* d_views, const BlurTap* d_taps, int nviews, const void* src,
                     int src_type, int w, int h, float* out, cudaStream_t st);
int launch_blur_stencil(const BlurView* d_views, const BlurCell* d_cells, int nviews, int max_smem,
                        const void* src, int src_type, int w, int h, float* out, cudaStream_t st,
                        const BlurRun* d_runs = nullptr, const float* d_rw = nullptr, int runs_smem = 0);
// tile floats k_blur_runs stages for a view (footprint + block padding)
int blur_runs_tile_floats(const BlurView& v);
int warp_init_attributes();
// maps: CUtensorMaps indexed by WarpView::tmap_idx (interior Lanczos
// footprints staged by one 2-D TMA per tile), or nullptr
// sep_tile0 >= 0 (Lanczos): tiles from sep_tile0 on belong to views with a
// diagonal back-map, resampled by the separable kernel (k_lanczos_sep)
int launch_warp(const WarpView* d_views, int nviews, int total_tiles, int mode, int out_type,
                void* out, float* pyr, int smem_floats, cudaStream_t st, const void* maps = nullptr,
                int sep_tile0 = -1, int zpass = 0);
// synth_warp_case renderer (eval.cpp:101-141): full 3x3 inverse of the framed
// homography, output frame size
struct ProjView {
    double back[9];
    int W, H;
};
int launch_warp_projective(const float* src, int w, int h, const ProjView& pv, int out_type, void* out,
                           cudaStream_t st);
int launch_gauss(const float* in, float* tmp, float* out, int w, int h, const float* d_k, int r,
                 cudaStream_t st);
int launch_resize(const float* in, int w, int h, float* out, int nw, int nh, cudaStream_t st);

// ORB (xa_orb.cu). Segment tables are host-built prefix sums in CTA units.
struct LevelSeg {
    int img, level;
    int blk_start;  // first CTA of this (image, level) segment
    int tiles_x;    // FAST tiles across (detect) / blocks across (pyramid)
    int r0 = 0;     // pyramid: first row of the segment
    int c0 = 0;     // pyramid: first 128-column block of the segment
};

int launch_pyramid(const OrbImage* d_imgs, const LevelSeg* d_segs, int nsegs, int total_blocks,
                   float* pyr, cudaStream_t st, bool zero = false);
// FAST tile range of one k_fast_nms CTA (a row of tiles): tiles [lo, hi) of
// the row can hold corners; the rest lie beyond the view content (all zero).
struct TileRange {
    int lo, hi;
    int img;  // image of this tile row (lets the auto-relax pass exit before the segment lookup)
};
// maps: a CUtensorMap (128 bytes) per image and level (index img * kLevels + L)
// describing the pyramid level as a 2-D float tensor of width `pitch`, box
// 72 x 38 (the FAST tile window), staged by one TMA per tile
int launch_fast_nms(const OrbImage* d_imgs, const LevelSeg* d_segs, int nsegs, int total_blocks,
                    const TileRange* d_rng, const float* pyr, const void* maps, Cand* cand,
                    ImgCounters* cnt, cudaStream_t st, int nimg);
int encode_level_maps(const struct OrbImage* imgs, int nimg, const float* pyr, void* out /* nimg*kLevels*128 B */);
int launch_measures(const OrbImage* d_imgs, int nimg, const float* pyr, const Cand* cand,
                    const ImgCounters* cnt, CandKey* keys, xa_kp* kps, cudaStream_t st);
// ---- SIFT (fine stage, xa_sift.cu)
struct SiftImg {  // one pyramid image in the SIFT buffer
    long long off;
    int w, h;
};
struct SiftCand {  // DoG extremum before refinement
    int o, layer, r, c;
};
struct SiftJob {  // one keypoint to describe (pyramid image resolved on the host)
    int img;      // gauss table index 6 * octave + layer
    float col, row, angle;
    double scl;   // octave-local scale
};
int launch_halve(const float* in, int w, float* out, int ow, int oh, cudaStream_t st);
int launch_dog(const float* a, const float* b, float* d, size_t n, cudaStream_t st);
int launch_dog_extrema(const float* base, SiftImg prv, SiftImg cur, SiftImg nxt, float prelim, int o,
                       int layer, SiftCand* cand, int* count, int cap, cudaStream_t st);
int launch_sift_keypoints(const float* base, const SiftImg* gauss, const SiftImg* dog,
                          const SiftCand* cand, const int* ncand, int cand_cap, xa_kp* out, int* nout,
                          int out_cap, cudaStream_t st);
int launch_sift_describe(const float* base, const SiftImg* gauss, const SiftJob* jobs, int n,
                         float* desc, cudaStream_t st);

// Per-image top-N selection state (zeroed before launch_select).
struct SelState {
    int hist[2048];  // keys per top-11-bit bin
    int valid;       // valid keys
    int lo, need;    // bin holding the N-th key (2048 = take all) and its rank there
    int nsel, nbnd;  // keys kept outright / listed from bin lo
    int big;         // the selection exceeds the shared-memory sort: k_select_big sorts it
    int pad[2];
};
int launch_select(const OrbImage* d_imgs, int nimg, int max_points, const CandKey* keys,
                  const xa_kp* kps, const Cand* cand, const float* pyr, Cand* det_cand,
                  int* det_map, ImgCounters* cnt, xa_kp* det_out, DescKp* desc_in,
                  xa_kp* desc_kp_out, int max_cand, SelState* sel, CandKey* sel_list,
                  uint2* bnd_list, CandKey* big_scratch, int big_cap, cudaStream_t st);
int launch_describe_prep(const OrbImage* d_imgs, const xa_kp* in, int n, ImgCounters* cnt,
                         DescKp* desc_in, xa_kp* desc_kp_out, cudaStream_t st);
int launch_describe(const OrbImage* d_imgs, int nimg, const float* pyr, const ImgCounters* cnt,
                    const DescKp* desc_in, uint64_t* desc, cudaStream_t st);

// Hamming (xa_match.cu)
struct MatchJob {
    long long a_off;    // query descriptor offset (descriptors)
    long long b_off;    // train descriptor offset
    const int* na_dev;  // device count of queries (or null -> na)
    const int* nb_dev;  // device count of train (or null -> nb)
    int na, nb;         // static counts / capacities
    long long out_off;  // per-query output offset
    int* count_out;     // device match counter for this job
};
int launch_match(const MatchJob* d_jobs, int njobs, int max_na, const uint64_t* a,
                 const uint64_t* b, const uint16_t* d_keep_thr, uint32_t* best_idx,
                 uint16_t* best, uint16_t* second, cudaStream_t st, int max_nb);
size_t match_l2_scratch(int na, int nsplit);
// tcgen05 Hamming matcher (xa_match.cu): descriptors expanded to +-1 s8 rows
// (256 B) by launch_desc_pm1; tmap = two 2-D uint8 tensor maps over those rows
// (SWIZZLE_128B, box 128 B x 128 rows for queries, x match_umma_tile_n() rows
// for train tiles); part (nsplit > 1, single job): uint2 key pairs
// [split][query] finished by launch_match_tc_merge
int match_umma_init();
int match_umma_tile_n();  // train rows per tile (the B tensor map's box height)
int launch_desc_pm1(const uint64_t* bits, long long n, void* out, cudaStream_t st);
int launch_match_umma(const MatchJob* d_jobs, const MatchJob& one, int njobs, int max_na, int nsplit,
                      const void* tmap, const uint16_t* keep_thr, uint32_t* best_idx, uint16_t* best,
                      uint16_t* second, void* part, int sms, cudaStream_t st);
int launch_match_tc_merge(const void* part, int na, int nsplit, const uint16_t* keep_thr, uint32_t* best_idx,
                          uint16_t* best, uint16_t* second, int* count, cudaStream_t st);
int match_l2_split(int na, int nb, int sms);
int launch_match_l2(const float* a, int na, const float* b, int nb, double ratio, int32_t* best_idx,
                    float* dist, uint8_t* keep, int32_t* count, void* scratch, int nsplit,
                    cudaStream_t st);
int launch_match_large(const uint64_t* a, int na, const uint64_t* b, int nb,
                       const uint16_t* d_keep_thr, uint32_t* best_idx, uint16_t* best,
                       uint16_t* second, int* count, void* scratch, int nsplit, cudaStream_t st);
size_t match_large_scratch(int na, int nsplit);

// trig fixups / pattern / constants (xa_orb.cu)
int orb_init_constants();
uint64_t pattern_checksum_host();
int trig_fixup_count();

}  // namespace xa
