// xa_engine.cu — host orchestration and the extern "C" boundary
// (include/xaffine_b200.h). Builds per-call launch tables on the host
// (view geometry, level segments, buffer offsets), uploads them in one copy
// and enqueues the kernel chain on the engine's stream. No CPU fallback:
// every entry point that computes runs on the device or fails loudly.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/xaffine_b200.h"
#include "xa_geometry.h"
#include "xa_kernels.h"

using namespace xa;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                           \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess)                                                             \
            return set_err(_e == cudaErrorMemoryAllocation ? XA_ENOMEM : XA_ECUDA,         \
                           std::string(#call) + ": " + cudaGetErrorString(_e));            \
    } while (0)

#define RET(call)               \
    do {                        \
        int _r = (call);        \
        if (_r != XA_OK) return _r; \
    } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Buffers the engine keeps between calls (grow-only).
enum Buf {
    B_IN0, B_IN1, B_BLUR, B_VIEW, B_PYR, B_CAND, B_KEYS, B_CKP, B_DET, B_DESCIN, B_DESCKP,
    B_DESC, B_CNT, B_TABLES, B_MBEST, B_MIDX, B_MSEC, B_OUT, B_KEEP, B_TMP0, B_TMP1, B_SCRATCH,
    B_DETCAND, B_DETMAP, B_SEL, B_SELL, B_BND, B_SIFT, B_SCAND, B_SKP, B_SJOB, B_SDESC,
    B_ADESC1, B_ADESC2, B_AMATCH, B_CNTALL, B_SELBIG, B_PM1, B_COUNT
};

}  // namespace

struct xa_engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    void* buf[B_COUNT] = {};
    size_t cap[B_COUNT] = {};
    char* staging = nullptr;  // pinned host staging for launch tables
    size_t staging_cap = 0;
    cudaEvent_t staging_done = nullptr;
    int last_launches = 0;
    double keep_ratio = -1.0;
    // stage profiling: events recorded between launches (xa_engine_set_profiling);
    // a batched coarse call records one set of stage marks per chunk
    int profiling = 0;
    std::vector<cudaEvent_t> marks;
    std::vector<const char*> mark_names;
    int nmarks = 0;
    bool mark_slot(int i) {
        while ((int)marks.size() <= i) {
            cudaEvent_t ev = nullptr;
            if (cudaEventCreate(&ev) != cudaSuccess) return false;
            marks.push_back(ev);
            mark_names.push_back(nullptr);
        }
        return true;
    }
    void mark_begin(cudaStream_t st) {
        nmarks = 0;
        if (!profiling || !mark_slot(0)) return;
        cudaEventRecordWithFlags(marks[0], st, cudaEventRecordExternal);  // a graph node when captured
        mark_names[0] = "begin";
        nmarks = 1;
    }
    void mark(cudaStream_t st, const char* name) {
        if (!profiling || nmarks == 0 || !mark_slot(nmarks)) return;
        cudaEventRecordWithFlags(marks[nmarks], st, cudaEventRecordExternal);
        mark_names[nmarks++] = name;
    }
    // ORB candidate capacity per image as a fraction of its pyramid pixels
    // (plus 4096). Host entry points grow it and retry when an image overflows;
    // device entry points report the overflow through xa_engine_check and the
    // next plan uses the grown factor.
    double cand_factor = 1.0 / 64;
    int orb_images = 0;  // images whose counters the last detect / coarse call left
    bool cnt_all = false;  // ... in B_CNTALL (every chunk of a coarse call), else B_CNT
    int* d_flags = nullptr;  // [0] overflow seen by the last device call
    cudaStream_t copy_stream = nullptr;     // host API: H2D of the pairs, overlapped with compute
    std::vector<cudaEvent_t> pair_ready;    // host API: pair p's inputs are on the device
    uint64_t gen = 0;        // bumped whenever a device buffer moves
    int tables_tag = 0;      // which cached plan owns B_TABLES (0 = none)
    struct CoarseCache* cc = nullptr;

    int ensure(Buf b, size_t bytes) {
        bytes = std::max<size_t>(bytes, 256);
        if (cap[b] >= bytes) return XA_OK;
        if (buf[b]) {
            CK(cudaStreamSynchronize(stream));
            CK(cudaFree(buf[b]));
            buf[b] = nullptr;
            cap[b] = 0;
        }
        const size_t nb = align_up(bytes + bytes / 4, 1 << 20);
        CK(cudaMalloc(&buf[b], nb));
        cap[b] = nb;
        ++gen;  // pointers baked into cached launch tables / graphs are stale now
        return XA_OK;
    }
    template <class T>
    T* p(Buf b) { return static_cast<T*>(buf[b]); }

    int ensure_staging(size_t bytes) {
        if (staging_done) CK(cudaEventSynchronize(staging_done));
        if (staging_cap >= bytes) return XA_OK;
        if (staging) CK(cudaFreeHost(staging));
        staging_cap = align_up(bytes + bytes / 2, 1 << 16);
        CK(cudaMallocHost(&staging, staging_cap));
        return XA_OK;
    }

    // Upload the ratio-test table: keep iff best < thr[second] (orb.cpp:267-268).
    int set_ratio(double ratio, cudaStream_t st) {
        if (ratio == keep_ratio) return XA_OK;
        RET(ensure(B_KEEP, 257 * sizeof(uint16_t)));
        uint16_t thr[257];
        for (int s = 0; s <= 256; ++s) {
            int b = 0;
            while (b <= 257 && b < ratio * s) ++b;
            thr[s] = (uint16_t)b;
        }
        CK(cudaMemcpyAsync(buf[B_KEEP], thr, sizeof thr, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        keep_ratio = ratio;
        return XA_OK;
    }
};

namespace {

// Table builder: packs heterogeneous launch tables into one staging blob.
struct Tables {
    std::vector<char> blob;
    template <class T>
    size_t add(const std::vector<T>& v) {
        const size_t off = align_up(blob.size(), 64);
        blob.resize(off + sizeof(T) * v.size());
        if (!v.empty()) std::memcpy(blob.data() + off, v.data(), sizeof(T) * v.size());
        return off;
    }
};

int upload_tables(xa_engine* e, const Tables& t, cudaStream_t st, int tag = 0) {
    e->tables_tag = tag;
    RET(e->ensure(B_TABLES, t.blob.size()));
    RET(e->ensure_staging(t.blob.size()));
    std::memcpy(e->staging, t.blob.data(), t.blob.size());
    CK(cudaMemcpyAsync(e->buf[B_TABLES], e->staging, t.blob.size(), cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(e->staging_done, st));
    return XA_OK;
}

template <class T>
const T* tab(xa_engine* e, size_t off) {
    return reinterpret_cast<const T*>(static_cast<char*>(e->buf[B_TABLES]) + off);
}

// ---------------------------------------------------------------- ORB batch

struct OrbSrc {
    const void* src;
    int type, w, h;
    bool filter;
    int src_w, src_h;
    Mat3 back;
    // coarse views: level 0 is zero outside the content quad (the source
    // rectangle mapped into the view frame); FAST skips tiles that cannot see it
    bool clip = false;
};

struct OrbPlan {
    std::vector<OrbImage> imgs;
    std::vector<LevelSeg> pyr_segs, fast_segs;
    // coarse views: blocks of the read band whose bilinear sources all lie in
    // the zero background (exactly 0.f); written once per call, not per chunk
    std::vector<LevelSeg> zero_segs;
    std::vector<TileRange> fast_rng;  // per k_fast_nms CTA
    int pyr_blocks = 0, fast_blocks = 0, zero_blocks = 0;
    long long pyr_floats = 0, cand_total = 0, kp_total = 0;
};

// Content quad of a view in level-0 frame coordinates: the source rectangle
// [-0.5, w-0.5] x [-0.5, h-0.5] (a superset of both resamplers' domains:
// Lanczos needs sx in [0, w-1], nearest lround(sx) in [0, w-1]) mapped by the
// forward transform (the inverse of the view's back-map).
struct Quad {
    double x[4], y[4];
};

bool content_quad(const Mat3& back, int sw, int sh, Quad& q) {
    Mat3 fwd;
    if (!mat_inv(back, fwd)) return false;
    const double cx[4] = {-0.5, sw - 0.5, sw - 0.5, -0.5}, cy[4] = {-0.5, -0.5, sh - 0.5, sh - 0.5};
    for (int k = 0; k < 4; ++k) map_pt_h(fwd, cx[k], cy[k], q.x[k], q.y[k]);
    return true;
}

// Separating-axis test: does the axis-aligned box [x0,x1] x [y0,y1] meet the
// convex quad? (axes: x, y and the four edge normals)
bool box_meets_quad(const Quad& q, double x0, double y0, double x1, double y1) {
    double mnx = q.x[0], mxx = q.x[0], mny = q.y[0], mxy = q.y[0];
    for (int k = 1; k < 4; ++k) {
        mnx = std::min(mnx, q.x[k]);
        mxx = std::max(mxx, q.x[k]);
        mny = std::min(mny, q.y[k]);
        mxy = std::max(mxy, q.y[k]);
    }
    if (mxx < x0 || mnx > x1 || mxy < y0 || mny > y1) return false;
    const double bx[4] = {x0, x1, x1, x0}, by[4] = {y0, y0, y1, y1};
    for (int e = 0; e < 4; ++e) {
        const double nx = -(q.y[(e + 1) & 3] - q.y[e]), ny = q.x[(e + 1) & 3] - q.x[e];
        double qa = 1e300, qb = -1e300, ba = 1e300, bb = -1e300;
        for (int k = 0; k < 4; ++k) {
            const double pq = nx * q.x[k] + ny * q.y[k], pb = nx * bx[k] + ny * by[k];
            qa = std::min(qa, pq);
            qb = std::max(qb, pq);
            ba = std::min(ba, pb);
            bb = std::max(bb, pb);
        }
        if (bb < qa || ba > qb) return false;
    }
    return true;
}

// Tiles [lo, hi) of FAST tile row ty at level L that can hold a corner. A
// position is a corner only if its pixel or a ring pixel (radius 3) is
// nonzero; a level-L pixel is a bilinear mix of level-0 pixels within 1 px
// (level-0 units) of its resize coordinate (image.cpp:55-66), and level 0 is
// zero outside the quad. Boxes are grown by 1 more level-0 px of margin.
TileRange fast_tile_range(const Quad& q, int W0, int H0, int wL, int hL, int tiles_x, int ty) {
    const double sx = (double)W0 / wL, sy = (double)H0 / hL;
    const int oy = kDetectBorder + ty * kFastTileH;
    const double y0 = (oy - 4 + 0.5) * sy - 0.5 - 2.0, y1 = (oy + kFastTileH + 3 + 0.5) * sy - 0.5 + 2.0;
    TileRange r{0, 0, 0};
    bool any = false;
    for (int tx = 0; tx < tiles_x; ++tx) {
        const int ox = kDetectBorder + tx * kFastTileW;
        const double x0 = (ox - 4 + 0.5) * sx - 0.5 - 2.0, x1 = (ox + kFastTileW + 3 + 0.5) * sx - 0.5 + 2.0;
        if (box_meets_quad(q, x0, y0, x1, y1)) {
            if (!any) r.lo = tx;
            r.hi = tx + 1;
            any = true;
        }
    }
    return r;
}

// Pyramid blocks [lo, hi) of block row rb at level L that anything downstream
// can read. Readers stay near the view content: FAST stages tile windows of the
// tiles fast_tile_range keeps (<= 69 level px beyond a box meeting the quad),
// Harris / orientation / describe read <= 34 level px around corners, which
// lie within 4 px of the content. A block is kept iff, grown by 80 level px
// (+2 level-0 px for the bilinear reach), it meets the content quad; the rest
// of the level is never written nor read.
TileRange pyr_block_range(const Quad& q, int W0, int H0, int wL, int hL, int chunks, int rb,
                          double m = 80.0) {
    const double sx = (double)W0 / wL, sy = (double)H0 / hL;
    const int ya = rb * kPyrRows, yb = std::min(hL, ya + kPyrRows) - 1;
    const double y0 = (ya - m + 0.5) * sy - 0.5 - 2.0, y1 = (yb + m + 0.5) * sy - 0.5 + 2.0;
    TileRange r{0, 0, 0};
    bool any = false;
    for (int c = 0; c < chunks; ++c) {
        const int xa = c * 128, xb = std::min(wL, xa + 128) - 1;
        const double x0 = (xa - m + 0.5) * sx - 0.5 - 2.0, x1 = (xb + m + 0.5) * sx - 0.5 + 2.0;
        if (box_meets_quad(q, x0, y0, x1, y1)) {
            if (!any) r.lo = c;
            r.hi = c + 1;
            any = true;
        }
    }
    return r;
}

// Level sizes (orb.cpp:133-139) and buffer offsets for a batch of images.
OrbPlan plan_orb(const std::vector<OrbSrc>& srcs, int max_points, double cand_factor) {
    OrbPlan P;
    for (size_t i = 0; i < srcs.size(); ++i) {
        const OrbSrc& s = srcs[i];
        OrbImage im;
        std::memset(&im, 0, sizeof im);
        im.nlev = 1;
        im.w[0] = s.w;
        im.h[0] = s.h;
        for (int L = 1; L < kLevels; ++L) {
            const double sc = std::pow(kLevelRatio, L);
            const int w = static_cast<int>(std::round(s.w / sc));
            const int h = static_cast<int>(std::round(s.h / sc));
            if (w < kMinSide || h < kMinSide) break;
            im.w[L] = w;
            im.h[L] = h;
            im.nlev = L + 1;
        }
        Quad quad;
        // XA_FAST_CLIP=0 turns the tile skipping off (tests/test_gpu_coarse.py
        // checks that it changes nothing)
        static const char* clip_env = std::getenv("XA_FAST_CLIP");
        const bool clip = s.clip && !(clip_env && clip_env[0] == '0') &&
                          content_quad(s.back, s.src_w, s.src_h, quad);
        long long levpx = 0;
        for (int L = 0; L < im.nlev; ++L) {
            im.poff[L] = P.pyr_floats;
            im.pitch[L] = (int)align_up(im.w[L], 4);  // 16-byte rows for the FAST staging
            const long long n = (long long)im.w[L] * im.h[L];
            P.pyr_floats += align_up((long long)im.pitch[L] * im.h[L], 32);
            levpx += n;
            const int chunks = (im.w[L] + 127) / 128;  // k_pyramid: 128-column x kPyrRows blocks
            if (L > 0 || s.type != XA_PIX_PYR0) {     // PYR0: level 0 written by the resampler
                const int rows = (im.h[L] + kPyrRows - 1) / kPyrRows;
                if (clip && L > 0) {  // coarse views: only blocks near the content (one segment per block row)
                    // XA_PYR_TIGHT=0: compute the whole read band every chunk
                    static const char* tight_env = std::getenv("XA_PYR_TIGHT");
                    const bool tight = !(tight_env && tight_env[0] == '0');
                    for (int rb = 0; rb < rows; ++rb) {
                        const TileRange br = pyr_block_range(quad, s.w, s.h, im.w[L], im.h[L], chunks, rb);
                        if (br.hi <= br.lo) continue;
                        // computed: blocks whose pixels' 2x2 sources can meet the
                        // content (margin 0 level px + the 2 level-0 px reach);
                        // the rest of the band is the zero background
                        TileRange tr = tight ? pyr_block_range(quad, s.w, s.h, im.w[L], im.h[L], chunks, rb, 0.0) : br;
                        tr.lo = std::max(tr.lo, br.lo);
                        tr.hi = std::min(tr.hi, br.hi);
                        if (tr.hi > tr.lo) {
                            LevelSeg ps{(int)i, L, P.pyr_blocks, tr.hi - tr.lo, rb * kPyrRows, tr.lo};
                            P.pyr_segs.push_back(ps);
                            P.pyr_blocks += tr.hi - tr.lo;
                        } else {
                            tr.lo = tr.hi = br.hi;
                        }
                        const int zl[2] = {br.lo, tr.hi}, zh[2] = {tr.lo, br.hi};
                        for (int z = 0; z < 2; ++z) {
                            if (zh[z] <= zl[z]) continue;
                            LevelSeg zs{(int)i, L, P.zero_blocks, zh[z] - zl[z], rb * kPyrRows, zl[z]};
                            P.zero_segs.push_back(zs);
                            P.zero_blocks += zh[z] - zl[z];
                        }
                    }
                } else {
                    LevelSeg ps{(int)i, L, P.pyr_blocks, chunks};
                    P.pyr_segs.push_back(ps);
                    P.pyr_blocks += chunks * rows;
                }
            }
            const int sw = im.w[L] - 2 * kDetectBorder, sh = im.h[L] - 2 * kDetectBorder;
            if (sw > 0 && sh > 0) {
                const int tx = (sw + kFastTileW - 1) / kFastTileW;  // k_fast_nms tiles
                const int ty = (sh + kFastTileH - 1) / kFastTileH;
                LevelSeg fs{(int)i, L, P.fast_blocks, tx};
                P.fast_segs.push_back(fs);
                P.fast_blocks += ty;  // one CTA per row of tiles
                for (int r = 0; r < ty; ++r) {
                    TileRange tr = clip ? fast_tile_range(quad, s.w, s.h, im.w[L], im.h[L], tx, r)
                                        : TileRange{0, tx, 0};
                    tr.img = (int)i;
                    P.fast_rng.push_back(tr);
                }
            }
        }
        im.src = s.src;
        im.src_type = s.type;
        im.max_points = max_points;
        im.cand_off = P.cand_total;
        im.cand_cap = (int)std::min<long long>(levpx * cand_factor + 4096, 1LL << 30);
        P.cand_total += im.cand_cap;
        im.filter = s.filter ? 1 : 0;
        im.src_w = s.src_w;
        im.src_h = s.src_h;
        im.margin = 5.0;  // pipeline.cpp:135
        for (int k = 0; k < 6; ++k) im.back[k] = s.back.m[k];
        im.kp_off = P.kp_total;
        P.kp_total += std::max(max_points, 1);
        P.imgs.push_back(im);
    }
    return P;
}

struct OrbDev {
    size_t imgs_off, pyr_off, fast_off, rng_off;
    size_t zero_off = 0;  // coarse: zero-background pyramid blocks (written once per call)
    size_t maps_off = 0;  // FAST tile tensor maps (encode_level_maps)
};

// One TMA tensor map per image level (index img * kLevels + L): the level as a
// 2-D float tensor (width = its pitch, height h, row stride pitch * 4 bytes)
// with the FAST tile window (72 x 38 floats) as the box. Encoded on the host
// through the driver entry point (no libcuda link dependency).
struct TMap {
    alignas(64) unsigned char b[128];
};
static_assert(sizeof(TMap) == sizeof(CUtensorMap), "tensor map size");

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// A 2-D float tensor map (row pitch in floats, 16-byte multiple) with box bw x bh.
int encode_map(TMap& m, const float* base, int width, int height, int pitch, int bw, int bh) {
    const PFN_cuTensorMapEncodeTiled_v12000 fn = tmap_encoder();
    if (!fn) return set_err(XA_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)height};
    const cuuint64_t strides[1] = {(cuuint64_t)pitch * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(reinterpret_cast<CUtensorMap*>(&m), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(XA_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return XA_OK;
}

// The +-1 s8 descriptor rows (256 B each) of the tcgen05 matcher as a 2-D
// uint8 tensor (256 B x rows) with a 128 B x 128-row box and 128-byte swizzle:
// one TMA lands one K half of 128 rows in the K-major SWIZZLE_128B canonical
// layout that k_match_umma's smem descriptors describe.
int encode_pm1_map(TMap& m, const void* base, long long rows, int box_rows) {
    const PFN_cuTensorMapEncodeTiled_v12000 fn = tmap_encoder();
    if (!fn) return set_err(XA_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {256, (cuuint64_t)std::max<long long>(rows, 1)};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(reinterpret_cast<CUtensorMap*>(&m), CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base),
                          dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(XA_ECUDA, "cuTensorMapEncodeTiled (pm1) failed (" + std::to_string((int)r) + ")");
    return XA_OK;
}

// query-block map (128-row boxes) and train-tile map (match_umma_tile_n() rows)
int encode_pm1_maps(TMap (&m)[2], const void* base, long long rows) {
    RET(encode_pm1_map(m[0], base, rows, 128));
    return encode_pm1_map(m[1], base, rows, match_umma_tile_n());
}

// XA_MATCH_UMMA=0: the warp-level IMMA matcher instead of tcgen05
bool use_umma() {
    static const bool on = [] {
        const char* e = std::getenv("XA_MATCH_UMMA");
        return !(e && e[0] == '0');
    }();
    return on;
}

int sm_count(int dev) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

int encode_level_maps(const std::vector<OrbImage>& imgs, const float* pyr, std::vector<TMap>& out) {
    out.assign(imgs.size() * kLevels, TMap{});
    for (size_t i = 0; i < imgs.size(); ++i) {
        const OrbImage& im = imgs[i];
        for (int L = 0; L < im.nlev; ++L)
            RET(encode_map(out[i * kLevels + L], pyr + im.poff[L], im.pitch[L], im.h[L], im.pitch[L], 72,
                           kFastTileH + 8));
    }
    return XA_OK;
}

// Entries of k_select_big's global sort buffer: every valid key of the largest
// image (NMS survivors are at most its candidate capacity), as a power of two.
int big_sort_cap(const OrbPlan& P) {
    int m = kSortCap;
    for (const OrbImage& im : P.imgs) m = std::max(m, im.cand_cap);
    int p = 1;
    while (p < m && p < (1 << 24)) p <<= 1;
    return p;
}

int ensure_orb(xa_engine* e, const OrbPlan& P) {
    // + tail slack: the FAST staging reads aligned 76-float rows past a level's edge
    RET(e->ensure(B_PYR, sizeof(float) * (P.pyr_floats + 1024)));
    RET(e->ensure(B_CAND, sizeof(Cand) * P.cand_total));
    RET(e->ensure(B_KEYS, sizeof(CandKey) * P.cand_total));
    RET(e->ensure(B_CKP, sizeof(xa_kp) * P.cand_total));
    RET(e->ensure(B_DET, sizeof(xa_kp) * P.kp_total));
    RET(e->ensure(B_DESCIN, sizeof(DescKp) * P.kp_total));
    RET(e->ensure(B_DESCKP, sizeof(xa_kp) * P.kp_total));
    RET(e->ensure(B_DESC, 32 * P.kp_total));
    RET(e->ensure(B_DETCAND, sizeof(Cand) * P.kp_total));
    RET(e->ensure(B_DETMAP, sizeof(int) * P.kp_total));
    RET(e->ensure(B_SEL, sizeof(SelState) * P.imgs.size()));
    RET(e->ensure(B_SELL, sizeof(CandKey) * kSortCap * P.imgs.size()));
    RET(e->ensure(B_BND, sizeof(uint2) * kListCap * P.imgs.size()));
    RET(e->ensure(B_CNT, sizeof(ImgCounters) * P.imgs.size()));
    RET(e->ensure(B_SELBIG, sizeof(CandKey) * (size_t)big_sort_cap(P)));
    return XA_OK;
}

// detect: pyramid -> FAST/NMS -> measures -> select(+describe list) over
// nimg images whose tables are already on the device
int run_detect(xa_engine* e, const OrbImage* imgs, int n, const LevelSeg* pyr_segs, int npyr,
               int pyr_blocks, const LevelSeg* fast_segs, int nfast, int fast_blocks,
               const TileRange* rng, const void* maps, int max_cand, int max_points, cudaStream_t st) {
    CK(cudaMemsetAsync(e->buf[B_CNT], 0, sizeof(ImgCounters) * n, st));
    e->orb_images = n;
    e->cnt_all = false;
    int L = 0;
    L += launch_pyramid(imgs, pyr_segs, npyr, pyr_blocks, e->p<float>(B_PYR), st);
    e->mark(st, "pyramid");
    L += launch_fast_nms(imgs, fast_segs, nfast, fast_blocks, rng, e->p<float>(B_PYR), maps, e->p<Cand>(B_CAND),
                         e->p<ImgCounters>(B_CNT), st, n);
    e->mark(st, "fast_nms");
    L += launch_measures(imgs, n, e->p<float>(B_PYR), e->p<Cand>(B_CAND), e->p<ImgCounters>(B_CNT),
                         e->p<CandKey>(B_KEYS), e->p<xa_kp>(B_CKP), st);
    e->mark(st, "measures");
    CK(cudaMemsetAsync(e->buf[B_SEL], 0, sizeof(SelState) * n, st));
    L += launch_select(imgs, n, max_points, e->p<CandKey>(B_KEYS), e->p<xa_kp>(B_CKP), e->p<Cand>(B_CAND),
                       e->p<float>(B_PYR), e->p<Cand>(B_DETCAND), e->p<int>(B_DETMAP),
                       e->p<ImgCounters>(B_CNT), e->p<xa_kp>(B_DET), e->p<DescKp>(B_DESCIN),
                       e->p<xa_kp>(B_DESCKP), max_cand, e->p<SelState>(B_SEL), e->p<CandKey>(B_SELL),
                       e->p<uint2>(B_BND), e->p<CandKey>(B_SELBIG),
                       (int)(e->cap[B_SELBIG] / sizeof(CandKey)), st);
    e->mark(st, "select");
    CK(cudaGetLastError());
    e->last_launches += L;
    return XA_OK;
}

int run_detect(xa_engine* e, const OrbPlan& P, const OrbDev& D, cudaStream_t st) {
    int max_cand = 0;
    for (const OrbImage& im : P.imgs) max_cand = std::max(max_cand, im.cand_cap);
    return run_detect(e, tab<OrbImage>(e, D.imgs_off), (int)P.imgs.size(), tab<LevelSeg>(e, D.pyr_off),
                      (int)P.pyr_segs.size(), P.pyr_blocks, tab<LevelSeg>(e, D.fast_off),
                      (int)P.fast_segs.size(), P.fast_blocks, tab<TileRange>(e, D.rng_off),
                      tab<TMap>(e, D.maps_off), max_cand, std::max(1, P.imgs[0].max_points), st);
}

// Finite, high-contrast pyramid poison (XA_POISON_PYR=1): hashed bytes in
// [0, 255], so a read of an unwritten pyramid region creates FAST corners or
// changes Harris / rBRIEF values instead of comparing false like NaN would.
__global__ void k_poison(float* __restrict__ p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u;
        h ^= h >> 15;
        p[i] = (h & 0x100u) ? 255.f : (float)(h & 0x3Fu);
    }
}

int launch_poison(float* p, size_t n, cudaStream_t st) {
    k_poison<<<148 * 8, 256, 0, st>>>(p, n);
    CK(cudaGetLastError());
    return XA_OK;
}

int check_counters(xa_engine* e, int n, std::vector<ImgCounters>& h) {
    h.resize(n);
    CK(cudaMemcpyAsync(h.data(), e->buf[B_CNT], sizeof(ImgCounters) * n, cudaMemcpyDeviceToHost,
                       e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (int i = 0; i < n; ++i)
        if (h[i].overflow)
            return set_err(XA_ECAPACITY, "ORB candidate/sort capacity exceeded (image " +
                                             std::to_string(i) + ", code " +
                                             std::to_string(h[i].overflow) + ")");
    return XA_OK;
}

// ---------------------------------------------------------------- views

struct ViewPlan {
    std::vector<BlurView> blur;
    std::vector<BlurTap> taps;
    std::vector<BlurCell> cells;
    int stencil_smem = 0;  // floats of the largest stencil tile
    std::vector<BlurRun> runs;  // k_blur_runs tables (runs_smem = 0: not representable, use the stencil kernel)
    std::vector<float> rw;
    int runs_smem = 0;
    bool runs_ok = true;
    std::vector<WarpView> warp;
    std::vector<Frame> frames;
    std::vector<int> blur_of;  // per view: blur index or -1
    int warp_tiles = 0;
    int warp_smem = 0;  // floats of the largest Lanczos source footprint
    long long out_elems = 0;
};

// antialias_tilt taps (warp.cpp:128-142), fixed per view.
int blur_taps(double t, double phi, BlurView& bv, std::vector<BlurTap>& taps) {
    const double sigma = 0.8 * std::sqrt(t * t - 1.0);
    const double dx = std::cos(phi), dy = -std::sin(phi);
    const int r = std::max(1, static_cast<int>(std::ceil(3.0 * sigma)));
    if (2 * r + 1 > kMaxBlurTaps) return set_err(XA_EINVAL, "antialias_tilt: tilt too large for device tap table");
    std::vector<double> k(2 * r + 1);
    double sum = 0;
    for (int i = -r; i <= r; ++i) {
        k[i + r] = std::exp(-0.5 * i * i / (sigma * sigma));
        sum += k[i + r];
    }
    for (auto& v : k) v /= sum;
    bv.ntaps = 2 * r + 1;
    bv.aligned = (dy == 0.0);
    bv.tap_off = (int)taps.size();
    for (int i = -r; i <= r; ++i) {
        BlurTap tp;
        tp.k = k[i + r];
        const double px = i * dx, py = i * dy;
        tp.px = px;
        tp.py = py;
        const double fx = std::floor(px), fy = std::floor(py);
        tp.ox = bv.aligned ? i : (int)fx;
        tp.oy = bv.aligned ? 0 : (int)fy;
        tp.wx = bv.aligned ? 0.f : (float)(px - fx);
        tp.wy = bv.aligned ? 0.f : (float)(py - fy);
        taps.push_back(tp);
    }
    return XA_OK;
}

// Fold the taps of one view into a 2-D stencil over integer offsets: tap i's
// bilinear cell weights k_i*(1-wx)(1-wy), k_i*wx(1-wy), ... summed per offset
// (in double, rounded once to float). Used by the pipeline's k_blur_stencil.
// The folded stencil as runs along its long axis for k_blur_runs (rowmode:
// one run per stencil row oy covering its ox range; otherwise per column),
// weights zero-padded to blocks of 4. Returns false if the view exceeds the
// kernel's run tables.
bool blur_runs(BlurView& bv, const std::vector<BlurCell>& cells, std::vector<BlurRun>& runs, std::vector<float>& rw) {
    bv.rowmode = (bv.bx1 - bv.bx0) >= (bv.by1 - bv.by0);
    bv.run_off = (int)runs.size();
    bv.rw_off = (int)rw.size();
    const int lo = bv.rowmode ? bv.by0 : bv.bx0, hi = bv.rowmode ? bv.by1 : bv.bx1;
    int nr = 0, nw = 0;
    for (int m = lo; m <= hi; ++m) {
        int a = 1 << 30, b = -(1 << 30);
        for (int i = 0; i < bv.ncells; ++i) {
            const BlurCell& c = cells[bv.cell_off + i];
            if ((bv.rowmode ? c.oy : c.ox) != m) continue;
            const int mi = bv.rowmode ? c.ox : c.oy;
            a = std::min(a, mi);
            b = std::max(b, mi);
        }
        if (a > b) continue;
        const int nblk = (b - a + 4) / 4;
        // k_blur_runs reads run m from the staged tile at this offset (its
        // row stride SW depends only on the view's stencil bounds)
        int SW, SH;
        blur_runs_geometry(bv, SW, SH);
        const int off = bv.rowmode ? (m - bv.by0) * SW + (a - bv.bx0) : (a - bv.by0) * SW + (m - bv.bx0);
        runs.push_back({off, a, nblk, nw});
        std::vector<float> wv(4 * nblk, 0.f);
        for (int i = 0; i < bv.ncells; ++i) {
            const BlurCell& c = cells[bv.cell_off + i];
            if ((bv.rowmode ? c.oy : c.ox) != m) continue;
            wv[(bv.rowmode ? c.ox : c.oy) - a] = c.w;
        }
        rw.insert(rw.end(), wv.begin(), wv.end());
        nw += 4 * nblk;
        ++nr;
    }
    bv.nruns = nr;
    bv.nrw = nw;
    return nr <= kMaxBlurRuns && nw <= kMaxBlurRunW;
}

int blur_stencil(BlurView& bv, const std::vector<BlurTap>& taps, std::vector<BlurCell>& cells,
                 int& smem_floats) {
    std::vector<std::pair<std::pair<int, int>, double>> acc;
    auto add = [&](int ox, int oy, double wgt) {
        if (wgt == 0.0) return;
        for (auto& a : acc)
            if (a.first.first == ox && a.first.second == oy) {
                a.second += wgt;
                return;
            }
        acc.push_back({{ox, oy}, wgt});
    };
    for (int i = 0; i < bv.ntaps; ++i) {
        const BlurTap& t = taps[bv.tap_off + i];
        const double wx = t.wx, wy = t.wy;
        add(t.ox, t.oy, t.k * (1 - wx) * (1 - wy));
        add(t.ox + 1, t.oy, t.k * wx * (1 - wy));
        add(t.ox, t.oy + 1, t.k * (1 - wx) * wy);
        add(t.ox + 1, t.oy + 1, t.k * wx * wy);
    }
    bv.cell_off = (int)cells.size();
    bv.ncells = (int)acc.size();
    bv.bx0 = bv.by0 = 0;
    bv.bx1 = bv.by1 = 0;
    for (auto& a : acc) {
        bv.bx0 = std::min(bv.bx0, a.first.first);
        bv.bx1 = std::max(bv.bx1, a.first.first);
        bv.by0 = std::min(bv.by0, a.first.second);
        bv.by1 = std::max(bv.by1, a.first.second);
        cells.push_back({a.first.first, a.first.second, (float)a.second, 0});
    }
    if (bv.ncells > kMaxBlurCells || bv.bx1 - bv.bx0 > 2 * kMaxBlurReach ||
        bv.by1 - bv.by0 > 2 * kMaxBlurReach)
        return set_err(XA_EINVAL, "antialias_tilt: tilt too large for the device stencil");
    // k_blur_stencil tile: two copies of 16-byte rows of 64 + width + alignment columns
    const int row = (kBlurTW + (bv.bx1 - bv.bx0) + 6) & ~3;
    smem_floats = std::max(smem_floats, 2 * row * (kBlurTH + bv.by1 - bv.by0));
    return XA_OK;
}

// Shared-memory bank plan for k_lanczos_smem. A warp covers a pw x (32/pw)
// patch of output pixels; each lane reads its 8 tap rows as 8-byte words at
// (floor(sy) - by0) * stride + ((floor(sx) - 3 - ax) & ~1), so the bank pattern
// of a load depends only on the back-map's linear part, the patch shape, the
// lanes' sub-pixel phase and stride mod 32. Model (64-bit loads): each
// half-warp costs one wavefront per distinct word in its busiest bank pair.
// The plan takes the (shape, stride residue) with the fewest modelled
// wavefronts over a fixed set of phases (preferring row-major 8x4 patches for
// coalesced stores); memoised per linear part and tile shape.
struct BankPlan {
    int res, pw;
};

int model_wavefronts(const double* b, int pw, int stride) {
    int total = 0;
    uint32_t st = 0x9e3779b9u;
    for (int smp = 0; smp < 48; ++smp) {
        st = st * 1664525u + 1013904223u;
        const double u = (st >> 8) * (1.0 / 16777216.0);
        st = st * 1664525u + 1013904223u;
        const double v = (st >> 8) * (1.0 / 16777216.0);
        const int off = smp & 3;
        for (int half = 0; half < 2; ++half) {
            int addr[16];
            for (int l = 0; l < 16; ++l) {
                const int lane = half * 16 + l;
                const int i = lane & ((1 << pw) - 1), k = lane >> pw;
                const double sx = 50.0 + u + b[0] * i + b[1] * k;
                const double sy = 50.0 + v + b[3] * i + b[4] * k;
                addr[l] = (int)std::floor(sy) * stride + (((int)std::floor(sx) + off) & ~1);
            }
            int worst = 0;
            for (int bank = 0; bank < 16; ++bank) {
                int seen[16], ns = 0;
                for (int l = 0; l < 16; ++l) {
                    if (((addr[l] >> 1) & 15) != bank) continue;
                    bool dup = false;
                    for (int q = 0; q < ns; ++q) dup |= seen[q] == addr[l];
                    if (!dup) seen[ns++] = addr[l];
                }
                worst = std::max(worst, ns);
            }
            total += worst;
        }
    }
    return total;
}

BankPlan lanczos_bank_plan(const double* back, int TW, int TH) {
    static std::mutex mu;
    static std::map<std::tuple<double, double, double, double, int, int>, BankPlan> memo;
    const auto key = std::make_tuple(back[0], back[1], back[3], back[4], TW, TH);
    {
        std::lock_guard<std::mutex> g(mu);
        const auto it = memo.find(key);
        if (it != memo.end()) return it->second;
    }
    BankPlan best{4, 3};
    int best_cost = 1 << 30;
    static const int kPw[] = {3, 2, 4, 1};                       // 8x4, 4x8, 16x2, 2x16
    static const int kRes[] = {4, 12, 20, 28, 0, 8, 16, 24};
    for (const int pw : kPw) {
        if ((1 << pw) > TW || (32 >> pw) > TH) continue;
        for (const int res : kRes) {
            const int c = model_wavefronts(back, pw, 64 + res);
            if (c < best_cost) {
                best_cost = c;
                best = {res, pw};
            }
        }
    }
    std::lock_guard<std::mutex> g(mu);
    memo[key] = best;
    return best;
}

// Output tiling of one view. Nearest: 32x32 tiles, one load per pixel.
// Lanczos (k_lanczos_smem): the largest tile in 64x64, 64x32, 32x32, 32x16,
// 16x16, 8x8 whose worst-case source footprint (back-mapped extent + 8-tap
// support + slack, at the planned stride) fits the per-CTA cap.
// Lanczos views with a diagonal back-map (phi = 0, including the identity
// view) whose 64 x 64 tile source region fits k_lanczos_sep (XA_LZ_SEP=0: off)
bool lanczos_separable(const WarpView& wv) {
    static const bool on = [] {
        const char* e = std::getenv("XA_LZ_SEP");
        return !(e && e[0] == '0');
    }();
    return on && wv.back[1] == 0.0 && wv.back[3] == 0.0 && std::fabs(wv.back[0]) * 63 + 10 <= 136 &&
           std::fabs(wv.back[4]) * 63 + 10 <= 76;
}

int warp_tiling(WarpView& wv, int w, int h, int mode, int& smem_floats) {
    wv.lz_res = 4;
    wv.lz_pw = 3;
    wv.lz_stride = wv.lz_box_h = 0;
    wv.tmap_idx = -1;
    wv.pad_ = 0;
    if (mode == XA_NEAREST) {
        wv.tile = wv.tile_h = 32;
        wv.tiles_x = (wv.W + 31) / 32;
        return XA_OK;
    }
    // 128-pixel tiles first (fewer per-tile prologues) where the footprint
    // still fits 48 KB and one tensor-TMA box (<= 256 per side); XA_LZ_BIG=0: off
    static const bool big_env = [] {
        const char* b = std::getenv("XA_LZ_BIG");
        return !(b && b[0] == '0');
    }();
    static const int kShapes[][2] = {{128, 128}, {128, 64}, {64, 128}, {64, 64}, {64, 32}, {32, 32}, {32, 16}, {16, 16}, {8, 8}};
    for (const auto& sh : kShapes) {
        const int TW = sh[0], TH = sh[1];
        if ((TW > 64 || TH > 64) && !big_env) continue;
        // device footprint: the back-mapped tile spans |b0|(TW-1) + |b1|(TH-1)
        // source columns and |b3|(TW-1) + |b4|(TH-1) rows; + 10 for the 8-tap
        // support and one slack column/row each side, +1 against rounding
        const int fw = std::min((int)std::ceil(std::fabs(wv.back[0]) * (TW - 1) +
                                               std::fabs(wv.back[1]) * (TH - 1)) + 11, w + 10);
        const int fh = std::min((int)std::ceil(std::fabs(wv.back[3]) * (TW - 1) +
                                               std::fabs(wv.back[4]) * (TH - 1)) + 11, h + 10);
        const BankPlan bp = lanczos_bank_plan(wv.back, TW, TH);
        const int need = lanczos_stride(fw, bp.res) * fh;  // one footprint copy
        // tiles above 32x32 only when they keep 4 CTAs per SM (48 KB)
        const bool box_ok = (TW <= 64 && TH <= 64) || (lanczos_stride(fw, bp.res) <= 256 && fh <= 256);
        if (box_ok && need <= (TW * TH > 1024 ? kLanczosSmemFloats * 3 / 4 : kLanczosSmemFloats)) {
            wv.tile = TW;
            wv.tile_h = TH;
            wv.tiles_x = (wv.W + TW - 1) / TW;
            wv.lz_res = bp.res;
            wv.lz_pw = bp.pw;
            wv.lz_stride = lanczos_stride(fw, bp.res);
            wv.lz_box_h = fh;
            smem_floats = std::max(smem_floats, need);
            return XA_OK;
        }
    }
    return set_err(XA_EINVAL, "warp_lanczos: view footprint too large for the device tile");
}

int check_params(const xa_params& p, const char* who) {
    if (p.tilt < 1.0) return set_err(XA_EINVAL, std::string(who) + ": tilt must be >= 1");
    if (p.scale <= 0.0) return set_err(XA_EINVAL, std::string(who) + ": scale must be > 0");
    return XA_OK;
}

// Geometry + tables for n views of one w x h source.
int plan_views(const xa_params* grid, int n, int w, int h, int mode, const void* src, int src_type,
               ViewPlan& V) {
    V.frames.resize(n);
    V.blur_of.assign(n, -1);
    for (int i = 0; i < n; ++i) {
        RET(check_params(grid[i], "simulation_from_params"));
        const Mat3 sim = compose_params(&grid[i].psi, true);
        if (warp_frame(sim, w, h, mode == XA_NEAREST, V.frames[i]))
            return set_err(XA_ESINGULAR, "invert: singular matrix");
        if (grid[i].tilt != 1.0) {
            BlurView bv;
            RET(blur_taps(grid[i].tilt, grid[i].phi, bv, V.taps));
            RET(blur_stencil(bv, V.taps, V.cells, V.stencil_smem));
            // XA_BLUR_RUNS=0: the per-cell stencil kernel instead of runs
            static const bool runs_env = [] {
                const char* r = std::getenv("XA_BLUR_RUNS");
                return !(r && r[0] == '0');
            }();
            V.runs_ok = runs_env && V.runs_ok && blur_runs(bv, V.cells, V.runs, V.rw);
            V.runs_smem = std::max(V.runs_smem, blur_runs_tile_floats(bv));
            bv.out_off = (long long)V.blur.size() * align_up((size_t)w * h, 64);
            bv.pad = 0;
            V.blur_of[i] = (int)V.blur.size();
            V.blur.push_back(bv);
        }
    }
    for (int i = 0; i < n; ++i) {
        const Frame& f = V.frames[i];
        WarpView wv;
        std::memset(&wv, 0, sizeof wv);
        for (int k = 0; k < 6; ++k) wv.back[k] = f.back.m[k];
        wv.W = f.W;
        wv.H = f.H;
        wv.sw = w;
        wv.sh = h;
        wv.out_off = V.out_elems;
        V.out_elems += align_up((size_t)f.W * f.H, 128);
        wv.src = src;  // patched to the blurred image by the caller when blurred
        wv.src_type = src_type;
        RET(warp_tiling(wv, w, h, mode, V.warp_smem));
        wv.tile_start = V.warp_tiles;
        V.warp_tiles += wv.tiles_x * ((f.H + wv.tile_h - 1) / wv.tile_h);
        V.warp.push_back(wv);
    }
    return XA_OK;
}

struct ViewLaunch {
    size_t ob = 0, ot = 0, ow = 0, oc = 0, orun = 0, orw = 0;
    float* blur = nullptr;
};

// Buffers and table entries for a view batch (no launches; not capturable).
int views_prepare(xa_engine* e, ViewPlan& V, int w, int h, Tables& T, ViewLaunch& VL) {
    RET(e->ensure(B_BLUR, sizeof(float) * std::max<size_t>(1, V.blur.size()) * align_up((size_t)w * h, 64)));
    VL.blur = e->p<float>(B_BLUR);
    for (size_t i = 0; i < V.warp.size(); ++i)
        if (V.blur_of[i] >= 0) {
            V.warp[i].src = VL.blur + V.blur[V.blur_of[i]].out_off;
            V.warp[i].src_type = XA_PIX_F32;
        }
    VL.ob = T.add(V.blur);
    VL.ot = T.add(V.taps);
    VL.ow = T.add(V.warp);
    VL.oc = T.add(V.cells);
    VL.orun = T.add(V.runs);
    VL.orw = T.add(V.rw);
    return XA_OK;
}

// Blur + resample launches for a prepared batch (capturable).
int views_enqueue(xa_engine* e, const ViewPlan& V, const ViewLaunch& VL, const void* d_src,
                  int src_type, int w, int h, int mode, int out_type, void* d_out, float* d_pyr,
                  cudaStream_t st) {
    int L = 0;
    if (V.cells.empty())  // reference-facing antialias_tilt path: per-tap bilinear, double sum
        L += launch_antialias(tab<BlurView>(e, VL.ob), tab<BlurTap>(e, VL.ot), (int)V.blur.size(),
                              d_src, src_type, w, h, VL.blur, st);
    else
        L += launch_blur_stencil(tab<BlurView>(e, VL.ob), tab<BlurCell>(e, VL.oc), (int)V.blur.size(),
                                 V.stencil_smem, d_src, src_type, w, h, VL.blur, st,
                                 V.runs_ok && !V.runs.empty() ? tab<BlurRun>(e, VL.orun) : nullptr,
                                 tab<float>(e, VL.orw), V.runs_ok ? V.runs_smem : 0);
    e->mark(st, "antialias");
    L += launch_warp(tab<WarpView>(e, VL.ow), (int)V.warp.size(), V.warp_tiles, mode, out_type, d_out,
                     d_pyr, V.warp_smem, st);
    e->mark(st, "warp");
    CK(cudaGetLastError());
    e->last_launches += L;
    return XA_OK;
}

int run_views(xa_engine* e, ViewPlan& V, const void* d_src, int src_type, int w, int h, int mode,
              int out_type, void* d_out, cudaStream_t st) {
    Tables T;
    ViewLaunch VL;
    RET(views_prepare(e, V, w, h, T, VL));
    RET(upload_tables(e, T, st));
    return views_enqueue(e, V, VL, d_src, src_type, w, h, mode, out_type, d_out, nullptr, st);
}

// Per-pair results of one chunk: kpc[(p0 + k) * n + j] = described keypoints of
// view j of the chunk's pair k; any ORB overflow of the chunk raises *flag.
__global__ void k_collect(const ImgCounters* __restrict__ cnt, int kc, int n, int32_t* __restrict__ kpc,
                          int* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < kc * n) {
        const int k = i / n, j = i - k * n;
        const ImgCounters& c = cnt[k * (n + 1) + 1 + j];
        if (kpc) kpc[i] = c.n_desc;
        if (c.overflow || cnt[k * (n + 1)].overflow) atomicOr(flag, 1);
    }
}

// ---------------------------------------------------------------- coarse

}  // namespace

// Everything a (batched) coarse call needs after planning, kept across calls
// so a repeated call (same geometry, pointers and parameters) skips the host
// planning and replays one CUDA graph of the whole launch chain.
//
// All pairs of a batch share the reference size, the target size and the grid,
// so every pair has the same views, pyramid layout and FAST/pyramid segment
// tables. The plan is built once for ONE pair and replicated for the K pairs of
// a chunk (image index, pyramid/candidate/keypoint offsets shifted per pair);
// chunks of K pairs run one after another through the same buffers. Only the
// small per-chunk tables that carry pointers (warp views, ORB images, match
// jobs) are stored per chunk. A last chunk of kc < K pairs uses the first kc
// pairs of the template: every table is ordered pair-major, so its segments,
// tiles and images are a prefix.
struct CoarseCache {
    std::string key;
    uint64_t gen = 0;
    int P = 0, K = 0, n = 0, mode = 0, mp = 0, src_type = 0, w = 0, h = 0;
    TMap pm1_map[2];     // tcgen05 matcher: query / train tensor maps of the chunk's expanded descriptors
    bool umma = false;
    ViewPlan V1;  // one pair's views (blur tables shared by every pair)
    ViewLaunch VL;
    OrbPlan P1;   // one pair's ORB plan (target + n views)
    OrbPlan PK;   // the template: K pairs
    OrbDev D;     // shared segment tables of the template
    size_t blur_plane = 0;  // floats per blurred plane
    size_t warp_maps = 0;   // table offset of the Lanczos source tensor maps (pair k, view j: k * n + j)
    struct Chunk {
        int p0, kc;
        size_t ow, oi, oj;  // per-chunk warp view / ORB image / match job tables
        int tiles = 0, sep_t0 = 0, nviews = 0;  // resampler tiles; separable views' first tile
    };
    std::vector<Chunk> chunks;
    std::vector<const void*> refs;
    Tables T;
    int32_t* d_counts = nullptr;
    int32_t* d_kpc = nullptr;
    int launches = 0;
    cudaGraphExec_t exec = nullptr;       // the launch chain
    cudaGraphExec_t exec_prof = nullptr;  // same chain with stage event nodes
    int prof_marks = 0;
    std::vector<const char*> prof_names;
    ~CoarseCache() {
        if (exec) cudaGraphExecDestroy(exec);
        if (exec_prof) cudaGraphExecDestroy(exec_prof);
    }
};

namespace {

std::string coarse_key(int ptype, const void* const* d_refs, int w, int h, const void* const* d_tgts,
                       int tw, int th, int P, const xa_params* grid, int n, int max_points, double ratio,
                       int mode, const int32_t* d_counts, const int32_t* d_kpc, int K) {
    std::string k;
    auto put = [&k](const void* p, size_t b) { k.append(static_cast<const char*>(p), b); };
    const int iv[10] = {ptype, w, h, tw, th, n, max_points, mode, P, K};
    const void* pv[2] = {d_counts, d_kpc};
    put(iv, sizeof iv);
    put(pv, sizeof pv);
    put(d_refs, sizeof(void*) * (size_t)P);
    put(d_tgts, sizeof(void*) * (size_t)P);
    put(&ratio, sizeof ratio);
    put(grid, sizeof(xa_params) * (size_t)n);
    return k;
}

// Replicate a one-pair ORB plan (image 0 = target, 1..n = views) for K pairs.
OrbPlan replicate_orb(const OrbPlan& P1, int K) {
    OrbPlan R;
    const int ni = (int)P1.imgs.size();
    for (int k = 0; k < K; ++k) {
        for (OrbImage im : P1.imgs) {
            for (int L = 0; L < im.nlev; ++L) im.poff[L] += k * P1.pyr_floats;
            im.cand_off += k * P1.cand_total;
            im.kp_off += k * P1.kp_total;
            R.imgs.push_back(im);
        }
        for (LevelSeg s : P1.pyr_segs) {
            s.img += k * ni;
            s.blk_start += k * P1.pyr_blocks;
            R.pyr_segs.push_back(s);
        }
        for (LevelSeg s : P1.fast_segs) {
            s.img += k * ni;
            s.blk_start += k * P1.fast_blocks;
            R.fast_segs.push_back(s);
        }
        for (LevelSeg s : P1.zero_segs) {
            s.img += k * ni;
            s.blk_start += k * P1.zero_blocks;
            R.zero_segs.push_back(s);
        }
        for (TileRange r : P1.fast_rng) {
            r.img += k * ni;
            R.fast_rng.push_back(r);
        }
    }
    R.pyr_blocks = K * P1.pyr_blocks;
    R.fast_blocks = K * P1.fast_blocks;
    R.zero_blocks = K * P1.zero_blocks;
    R.pyr_floats = K * P1.pyr_floats;
    R.cand_total = K * P1.cand_total;
    R.kp_total = K * P1.kp_total;
    return R;
}

// Device bytes one pair of the template needs (pyramid + candidates + keypoints + blur planes).
size_t pair_bytes(const OrbPlan& P1, size_t blur_floats) {
    return sizeof(float) * (size_t)P1.pyr_floats +
           (sizeof(Cand) + sizeof(CandKey) + sizeof(xa_kp)) * (size_t)P1.cand_total +
           (3 * sizeof(xa_kp) + sizeof(DescKp) + 32 + sizeof(Cand) + sizeof(int)) * (size_t)P1.kp_total +
           sizeof(float) * blur_floats;
}

// Pairs per chunk: XA_BATCH_PAIRS, else as many as fit in half of the free
// device memory (at most 8: beyond that the chunk tails are already amortised).
int pick_chunk(size_t per_pair, int P) {
    const char* env = std::getenv("XA_BATCH_PAIRS");
    if (env && std::atoi(env) > 0) return std::max(1, std::min(P, std::atoi(env)));
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 8ull << 30;
    const int fit = (int)std::max<size_t>(1, (free_b / 2) / std::max<size_t>(per_pair, 1));
    const int K = std::max(1, std::min({P, fit, 8}));
    const int chunks = (P + K - 1) / K;
    return (P + chunks - 1) / chunks;  // balanced chunks
}

// XA_LZ_SKIP=0: every chunk writes the zeros of the Lanczos tiles outside the content.
bool use_lz_skip() {
    static const bool on = [] {
        const char* v = std::getenv("XA_LZ_SKIP");
        return !(v && v[0] == '0');
    }();
    return on;
}

// Host planning, buffer sizing and table upload (not capturable).
int coarse_prepare(xa_engine* e, CoarseCache& c, int ptype, const void* const* d_refs, int w, int h,
                   const void* const* d_tgts, int tw, int th, int P, const xa_params* grid, int n,
                   int max_points, int mode, int32_t* d_counts, int32_t* d_kpc, cudaStream_t st) {
    c.src_type = ptype == XA_U8 ? XA_PIX_U8 : XA_PIX_F32;
    c.w = w;
    c.h = h;
    c.n = n;
    c.P = P;
    c.mode = mode;
    c.d_counts = d_counts;
    c.d_kpc = d_kpc;
    c.mp = std::max(max_points, 0);
    c.refs.assign(d_refs, d_refs + P);
    RET(plan_views(grid, n, w, h, mode, nullptr, c.src_type, c.V1));
    // The views are never materialised as uint8 images: the resampler writes
    // each quantised view straight into its ORB pyramid level 0.
    std::vector<OrbSrc> srcs;
    srcs.push_back({nullptr, c.src_type, tw, th, false, 0, 0, Mat3()});
    for (int i = 0; i < n; ++i)
        srcs.push_back({nullptr, XA_PIX_PYR0, c.V1.frames[i].W, c.V1.frames[i].H, true, w, h,
                        c.V1.frames[i].back, true});
    c.P1 = plan_orb(srcs, c.mp, e->cand_factor);
    c.blur_plane = align_up((size_t)w * h, 64);
    const int nb = (int)c.V1.blur.size();
    const int K = pick_chunk(pair_bytes(c.P1, nb * c.blur_plane), P);
    c.K = K;
    c.PK = replicate_orb(c.P1, K);
    // buffers first (ensure may move them), then the tables that point into them
    RET(e->ensure(B_BLUR, sizeof(float) * std::max<size_t>(1, (size_t)K * nb * c.blur_plane)));
    RET(ensure_orb(e, c.PK));
    RET(e->ensure(B_OUT, sizeof(int) * 4));
    RET(e->ensure(B_CNTALL, sizeof(ImgCounters) * (size_t)P * (n + 1)));
    c.umma = use_umma() && c.PK.kp_total < (1LL << 22);
    if (c.umma) RET(e->ensure(B_PM1, 256 * (size_t)std::max<long long>(c.PK.kp_total, 1)));
    c.VL.blur = e->p<float>(B_BLUR);
    c.VL.ob = c.T.add(c.V1.blur);
    c.VL.ot = c.T.add(c.V1.taps);
    c.VL.oc = c.T.add(c.V1.cells);
    c.VL.orun = c.T.add(c.V1.runs);
    c.VL.orw = c.T.add(c.V1.rw);
    c.D.imgs_off = 0;
    c.D.pyr_off = c.T.add(c.PK.pyr_segs);
    c.D.fast_off = c.T.add(c.PK.fast_segs);
    c.D.rng_off = c.T.add(c.PK.fast_rng);
    c.D.zero_off = c.T.add(c.PK.zero_segs);
    c.D.imgs_off = c.T.add(c.PK.imgs);  // the template's image table (zero fill)
    if (std::getenv("XA_PLAN_STATS"))
        std::fprintf(stderr, "[xa] coarse plan: %d pyramid blocks + %d zero blocks per pair, %d FAST rows\n",
                     c.P1.pyr_blocks, c.P1.zero_blocks, c.P1.fast_blocks);
    {
        std::vector<TMap> maps;
        RET(encode_level_maps(c.PK.imgs, e->p<float>(B_PYR), maps));
        c.D.maps_off = c.T.add(maps);
    }
    if (c.umma) RET(encode_pm1_maps(c.pm1_map, e->buf[B_PM1], c.PK.kp_total));
    const ImgCounters* dcnt = e->p<ImgCounters>(B_CNT);
    const int ni = n + 1;
    // tensor maps of the blurred source planes, one per (pair, view) with the
    // view's footprint box (Lanczos interior tiles: one 2-D TMA per tile)
    std::vector<TMap> wmaps((size_t)K * n);
    std::vector<int> widx((size_t)K * n, -1);
    if (mode == XA_LANCZOS && (w & 3) == 0) {
        for (int k = 0; k < K; ++k)
            for (int j = 0; j < n; ++j) {
                const WarpView& t = c.V1.warp[j];
                const int b = c.V1.blur_of[j];
                if (b < 0 || t.lz_stride <= 0 || t.lz_stride > 256 || t.lz_box_h > 256) continue;
                RET(encode_map(wmaps[(size_t)k * n + j], c.VL.blur + ((size_t)k * nb + b) * c.blur_plane, w, h,
                               w, t.lz_stride, t.lz_box_h));
                widx[(size_t)k * n + j] = k * n + j;
            }
    }
    c.warp_maps = c.T.add(wmaps);
    // separable Lanczos views (diagonal back-maps, 64 x 64 tiles) go last in
    // each chunk's view table: their tiles form the k_lanczos_sep launch
    std::vector<char> sep(n, 0);
    if (mode == XA_LANCZOS)
        for (int j = 0; j < n; ++j) sep[j] = lanczos_separable(c.V1.warp[j]);
    c.chunks.clear();
    for (int p0 = 0; p0 < P; p0 += K) {
        CoarseCache::Chunk ch;
        ch.p0 = p0;
        ch.kc = std::min(K, P - p0);
        std::vector<WarpView> warp, warp_sep;
        std::vector<OrbImage> imgs(c.PK.imgs.begin(), c.PK.imgs.begin() + (size_t)ch.kc * ni);
        std::vector<MatchJob> jobs;
        for (int k = 0; k < ch.kc; ++k) {
            const int p = p0 + k;
            imgs[(size_t)k * ni].src = d_tgts[p];
            for (int j = 0; j < n; ++j) {
                WarpView wv = c.V1.warp[j];
                wv.tile_start += k * c.V1.warp_tiles;
                wv.tmap_idx = widx[(size_t)k * n + j];
                const int b = c.V1.blur_of[j];
                if (b >= 0) {
                    wv.src = c.VL.blur + ((size_t)k * nb + b) * c.blur_plane;
                    wv.src_type = XA_PIX_F32;
                } else {
                    wv.src = d_refs[p];
                    wv.src_type = c.src_type;
                }
                const OrbImage& vi = c.PK.imgs[(size_t)k * ni + 1 + j];
                wv.pyr_off = vi.poff[0];
                wv.pyr_pitch = vi.pitch[0];
                if (sep[j]) {
                    wv.tile = wv.tile_h = 64;
                    wv.tiles_x = (wv.W + 63) / 64;
                    warp_sep.push_back(wv);
                } else {
                    warp.push_back(wv);
                }
                MatchJob J;
                J.a_off = vi.kp_off;
                J.b_off = c.PK.imgs[(size_t)k * ni].kp_off;
                J.na_dev = &dcnt[k * ni + 1 + j].n_desc;
                J.nb_dev = &dcnt[k * ni].n_desc;
                J.na = c.mp;
                J.nb = c.mp;
                J.out_off = vi.kp_off;
                J.count_out = d_counts + (size_t)p * n + j;
                jobs.push_back(J);
            }
        }
        // flattened tile numbering: general views, then the separable ones
        int tiles = 0;
        for (WarpView& wv : warp) {
            wv.tile_start = tiles;
            tiles += wv.tiles_x * ((wv.H + wv.tile_h - 1) / wv.tile_h);
        }
        ch.sep_t0 = tiles;
        for (WarpView& wv : warp_sep) {
            wv.tile_start = tiles;
            tiles += wv.tiles_x * ((wv.H + 63) / 64);
        }
        ch.tiles = tiles;
        ch.nviews = (int)(warp.size() + warp_sep.size());
        warp.insert(warp.end(), warp_sep.begin(), warp_sep.end());
        ch.ow = c.T.add(warp);
        ch.oi = c.T.add(imgs);
        ch.oj = c.T.add(jobs);
        c.chunks.push_back(ch);
    }
    RET(e->ensure(B_TABLES, c.T.blob.size()));
    c.gen = e->gen;  // every buffer this plan points into is final now
    return upload_tables(e, c.T, st, 1);
}

// The launch chain of one coarse call (capturable: memsets + kernels only).
int coarse_enqueue(xa_engine* e, const CoarseCache& c, cudaStream_t st, const cudaEvent_t* in_ready) {
    e->last_launches = 0;
    const int n = c.n, ni = n + 1, nb = (int)c.V1.blur.size();
    const int segs_pp = (int)c.P1.pyr_segs.size(), fsegs_pp = (int)c.P1.fast_segs.size();
    CK(cudaMemsetAsync(c.d_counts, 0, sizeof(int32_t) * (size_t)c.P * n, st));
    // The zero background of the read band, once for every chunk of this call
    // (each chunk's pyramid slots have the same geometry and no kernel of the
    // chain writes there), and likewise the level-0 tiles of the general
    // Lanczos views that lie outside the content (zeroed by the kernel's own
    // tile test, skipped per chunk). A forked graph branch beside the first
    // chunk's blur measured no gain (the blur fills the SMs).
    const bool lz_skip = c.mode == XA_LANCZOS && use_lz_skip() && !c.chunks.empty();
    cudaStream_t zs = st;
    e->last_launches += launch_pyramid(tab<OrbImage>(e, c.D.imgs_off), tab<LevelSeg>(e, c.D.zero_off),
                                       (int)c.PK.zero_segs.size(), c.PK.zero_blocks, e->p<float>(B_PYR), zs, true);
    if (lz_skip) {
        const CoarseCache::Chunk& c0 = c.chunks.front();  // the widest chunk: every slot
        e->last_launches += launch_warp(tab<WarpView>(e, c0.ow), c0.nviews, c0.tiles, c.mode,
                                        c.src_type == XA_PIX_F32 ? XA_PIX_F32 : XA_PIX_U8, nullptr,
                                        e->p<float>(B_PYR), c.V1.warp_smem, zs, tab<TMap>(e, c.warp_maps),
                                        c0.sep_t0, 1);
    }

    for (const CoarseCache::Chunk& ch : c.chunks) {
        const int kc = ch.kc;
        int L = 0;
        // host API: this chunk starts when its pairs' H2D copies (issued in
        // order on the copy stream) have landed -- an external-event wait node,
        // so later chunks' copies overlap the earlier chunks' kernels
        if (in_ready) CK(cudaStreamWaitEvent(st, in_ready[ch.p0 + kc - 1], cudaEventWaitExternal));
        // anti-alias blur of every tilted view, one launch per pair (per source)
        // float inputs keep the reference's float views: the exact double blur
        // (k_antialias) and unquantised resampling; uint8 inputs quantise the
        // views to uint8 (north_star) and blur with the folded float stencil
        const bool fview = c.src_type == XA_PIX_F32;
        for (int k = 0; k < kc; ++k) {
            float* out = c.VL.blur + (size_t)k * nb * c.blur_plane;
            if (fview)
                L += launch_antialias(tab<BlurView>(e, c.VL.ob), tab<BlurTap>(e, c.VL.ot), nb,
                                      c.refs[ch.p0 + k], c.src_type, c.w, c.h, out, st);
            else
                L += launch_blur_stencil(tab<BlurView>(e, c.VL.ob), tab<BlurCell>(e, c.VL.oc), nb,
                                         c.V1.stencil_smem, c.refs[ch.p0 + k], c.src_type, c.w, c.h, out, st,
                                         c.V1.runs_ok && !c.V1.runs.empty() ? tab<BlurRun>(e, c.VL.orun) : nullptr,
                                         tab<float>(e, c.VL.orw), c.V1.runs_ok ? c.V1.runs_smem : 0);
        }
        e->mark(st, "antialias");
        L += launch_warp(tab<WarpView>(e, ch.ow), ch.nviews, ch.tiles, c.mode,
                         fview ? XA_PIX_F32 : XA_PIX_U8, nullptr, e->p<float>(B_PYR), c.V1.warp_smem, st,
                         tab<TMap>(e, c.warp_maps), ch.sep_t0, lz_skip ? 2 : 0);
        e->mark(st, "warp");
        const OrbImage* imgs = tab<OrbImage>(e, ch.oi);
        int max_cand = 0;
        for (int i = 0; i < ni; ++i) max_cand = std::max(max_cand, c.P1.imgs[i].cand_cap);
        RET(run_detect(e, imgs, kc * ni, tab<LevelSeg>(e, c.D.pyr_off), kc * segs_pp, kc * c.P1.pyr_blocks,
                       tab<LevelSeg>(e, c.D.fast_off), kc * fsegs_pp, kc * c.P1.fast_blocks,
                       tab<TileRange>(e, c.D.rng_off), tab<TMap>(e, c.D.maps_off), max_cand, std::max(1, c.mp),
                       st));
        L += launch_describe(imgs, kc * ni, e->p<float>(B_PYR), e->p<ImgCounters>(B_CNT),
                             e->p<DescKp>(B_DESCIN), e->p<uint64_t>(B_DESC), st);
        e->mark(st, "describe");
        if (c.umma) {
            // tcgen05 matcher: this chunk's descriptors as +-1 rows, then all jobs
            L += launch_desc_pm1(e->p<uint64_t>(B_DESC), (long long)kc * c.P1.kp_total, e->buf[B_PM1], st);
            L += launch_match_umma(tab<MatchJob>(e, ch.oj), MatchJob{}, kc * n, std::max(c.mp, 1), 1, c.pm1_map,
                                   e->p<uint16_t>(B_KEEP), nullptr, nullptr, nullptr, nullptr, sm_count(e->device), st);
        } else {
            L += launch_match(tab<MatchJob>(e, ch.oj), kc * n, std::max(c.mp, 1), e->p<uint64_t>(B_DESC),
                              e->p<uint64_t>(B_DESC), e->p<uint16_t>(B_KEEP), nullptr, nullptr, nullptr, st,
                              std::max(c.mp, 1));
        }
        e->mark(st, "match");
        k_collect<<<(kc * n + 127) / 128, 128, 0, st>>>(e->p<ImgCounters>(B_CNT), kc, n,
                                                         c.d_kpc ? c.d_kpc + (size_t)ch.p0 * n : nullptr,
                                                         e->d_flags);
        // every chunk's per-image counters, for exact work accounting (orb_counters)
        CK(cudaMemcpyAsync(e->p<ImgCounters>(B_CNTALL) + (size_t)ch.p0 * ni, e->buf[B_CNT],
                           sizeof(ImgCounters) * (size_t)kc * ni, cudaMemcpyDeviceToDevice, st));
        e->mark(st, "collect");
        L += 1;
        e->last_launches += L;
    }
    CK(cudaGetLastError());
    return XA_OK;
}

int coarse_device(xa_engine* e, int ptype, const void* const* d_refs, int w, int h,
                  const void* const* d_tgts, int tw, int th, int P, const xa_params* grid, int n,
                  int max_points, double ratio, int mode, int32_t* d_counts, int32_t* d_kpc,
                  cudaStream_t st, const cudaEvent_t* in_ready = nullptr) {
    if (n <= 0 || !grid) return set_err(XA_EPIPELINE, "coarse: empty parameter grid");
    if (P <= 0 || !d_refs || !d_tgts) return set_err(XA_EINVAL, "coarse: no image pairs");
    if (ptype != XA_U8 && ptype != XA_F32) return set_err(XA_EINVAL, "pixel_type");
    if (mode != XA_NEAREST && mode != XA_LANCZOS) return set_err(XA_EINVAL, "warp_mode");
    RET(e->set_ratio(ratio, st));
    const std::string key = coarse_key(ptype, d_refs, w, h, d_tgts, tw, th, P, grid, n, max_points,
                                       ratio, mode, d_counts, d_kpc,
                                       std::getenv("XA_BATCH_PAIRS") ? std::atoi(std::getenv("XA_BATCH_PAIRS")) : 0) +
                            std::string(reinterpret_cast<const char*>(&e->cand_factor), sizeof(double)) +
                            (in_ready ? "E" : "D");
    CoarseCache* c = e->cc;
    const bool hit = c && c->key == key && c->gen == e->gen;
    if (!hit) {
        delete e->cc;
        c = e->cc = new CoarseCache();
        RET(coarse_prepare(e, *c, ptype, d_refs, w, h, d_tgts, tw, th, P, grid, n, max_points, mode,
                           d_counts, d_kpc, st));
        c->key = key;
    } else if (e->tables_tag != 1) {
        RET(upload_tables(e, c->T, st, 1));  // another entry point reused B_TABLES
    }
    // XA_POISON_PYR=1 (tests): fill the pyramid with a finite high-contrast
    // pattern first, so a read of any region the plan leaves unwritten
    // (skipped pyramid blocks) would create corners or change descriptors
    static const char* poison = std::getenv("XA_POISON_PYR");
    const bool poisoned = poison && poison[0] == '1';
    // Replay a captured graph of the launch chain; with profiling on, the
    // captured chain also records the stage events (event-record nodes).
    cudaGraphExec_t& exec = e->profiling ? c->exec_prof : c->exec;
    if (!exec) {
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        e->mark_begin(st);
        int rc = XA_OK;
        if (poisoned) rc = launch_poison(e->p<float>(B_PYR), (size_t)c->PK.pyr_floats + 1024, st);
        if (rc == XA_OK) rc = coarse_enqueue(e, *c, st, in_ready);
        const cudaError_t ce = cudaStreamEndCapture(st, &g);
        RET(rc);
        CK(ce);
        CK(cudaGraphInstantiate(&exec, g, 0));
        cudaGraphDestroy(g);
        c->launches = e->last_launches + (poisoned ? 1 : 0);
        if (e->profiling) {
            c->prof_marks = e->nmarks;
            c->prof_names.assign(e->mark_names.begin(), e->mark_names.begin() + e->nmarks);
        }
    }
    if (e->profiling) {
        e->nmarks = c->prof_marks;
        for (int i = 0; i < c->prof_marks; ++i) e->mark_names[i] = c->prof_names[i];
    }
    CK(cudaGraphLaunch(exec, st));
    e->last_launches = c->launches;
    e->orb_images = P * (n + 1);
    e->cnt_all = true;
    return XA_OK;
}

int upload(xa_engine* e, Buf b, const void* host, size_t bytes) {
    RET(e->ensure(b, bytes));
    CK(cudaMemcpyAsync(e->buf[b], host, bytes, cudaMemcpyHostToDevice, e->stream));
    return XA_OK;
}

// ---------------------------------------------------------------- SIFT

// gaussian_kernel (image.cpp:10-21): float taps of a double exp, normalised.
std::vector<float> gauss_kernel(double sigma) {
    const int r = std::max(1, static_cast<int>(std::ceil(3.0 * sigma)));
    std::vector<float> k(2 * r + 1);
    double sum = 0;
    for (int i = -r; i <= r; ++i) {
        const double v = std::exp(-0.5 * i * i / (sigma * sigma));
        k[i + r] = static_cast<float>(v);
        sum += v;
    }
    for (auto& v : k) v = static_cast<float>(v / sum);
    return k;
}

struct SiftPyr {
    int noct = 0;
    std::vector<SiftImg> gauss, dog;  // 6 and 5 per octave
    size_t og = 0, od = 0;            // their table offsets
    size_t ok = 0;                    // blur kernels' table offset
    std::vector<size_t> koff;         // per kernel: first tap in the kernel table
    std::vector<int> kr;              // per kernel: radius
    long long floats = 0;             // pyramid size
};

// build_pyramid (sift.cpp:42-80) layout on the host: image offsets (floats
// from the pyramid base) and the blur kernels, appended to T.
void sift_layout(int w, int h, SiftPyr& P, Tables& T) {
    const int bw = 2 * w, bh = 2 * h;
    P.noct = std::max(1, static_cast<int>(std::floor(std::log2((double)std::min(bw, bh)))) - 4);
    long long off = 0;
    int ow = bw, oh = bh;
    for (int o = 0; o < P.noct; ++o) {
        if (o) {
            ow /= 2;
            oh /= 2;
        }
        for (int i = 0; i < 6; ++i) {
            P.gauss.push_back({off, ow, oh});
            off += align_up((long long)ow * oh, 32);
        }
        for (int i = 0; i < 5; ++i) {
            P.dog.push_back({off, ow, oh});
            off += align_up((long long)ow * oh, 32);
        }
    }
    P.floats = off;
    // blur kernels: sigma_diff for the base, then inc[1..5]
    std::vector<std::vector<float>> ks;
    ks.push_back(gauss_kernel(std::sqrt(std::max(1.6 * 1.6 - 4.0 * 0.5 * 0.5, 0.01))));
    const double kk = std::pow(2.0, 1.0 / 3);
    double prev = 1.6;
    for (int i = 1; i < 6; ++i) {
        const double total = 1.6 * std::pow(kk, i);
        ks.push_back(gauss_kernel(std::sqrt(total * total - prev * prev)));
        prev = total;
    }
    std::vector<float> kflat;
    for (auto& k : ks) {
        P.koff.push_back(kflat.size());
        P.kr.push_back((int)k.size() / 2);
        kflat.insert(kflat.end(), k.begin(), k.end());
    }
    P.ok = T.add(kflat);
    P.og = T.add(P.gauss);
    P.od = T.add(P.dog);
}

// The pyramid's launches into S (P.floats floats) with the tables already on
// the device; tmp0/tmp1 hold 4 w h floats each.
int sift_enqueue(xa_engine* e, const float* d_img, int w, int h, const SiftPyr& P, float* S,
                 float* tmp0, float* tmp1, cudaStream_t st) {
    const int bw = 2 * w, bh = 2 * h;
    const float* K = tab<float>(e, P.ok);
    int L = 0;
    L += launch_resize(d_img, w, h, tmp0, bw, bh, st);
    L += launch_gauss(tmp0, tmp1, S + P.gauss[0].off, bw, bh, K + P.koff[0], P.kr[0], st);
    for (int o = 0; o < P.noct; ++o) {
        const SiftImg* g = &P.gauss[6 * o];
        const SiftImg* d = &P.dog[5 * o];
        if (o) {
            const SiftImg& s3 = P.gauss[6 * (o - 1) + 3];
            L += launch_halve(S + s3.off, s3.w, S + g[0].off, g[0].w, g[0].h, st);
        }
        for (int i = 1; i < 6; ++i)
            L += launch_gauss(S + g[i - 1].off, tmp1, S + g[i].off, g[i].w, g[i].h, K + P.koff[i], P.kr[i], st);
        for (int i = 0; i < 5; ++i)
            L += launch_dog(S + g[i].off, S + g[i + 1].off, S + d[i].off, (size_t)d[i].w * d[i].h, st);
    }
    CK(cudaGetLastError());
    e->last_launches += L;
    return XA_OK;
}

// Single-image pyramid in B_SIFT (detect_dog_keypoints / describe_gradient).
int sift_pyramid(xa_engine* e, const float* d_img, int w, int h, SiftPyr& P, Tables& T, cudaStream_t st) {
    sift_layout(w, h, P, T);
    RET(e->ensure(B_SIFT, sizeof(float) * P.floats));
    RET(e->ensure(B_TMP0, sizeof(float) * 4 * (size_t)w * h));
    RET(e->ensure(B_TMP1, sizeof(float) * 4 * (size_t)w * h));
    RET(upload_tables(e, T, st));
    return sift_enqueue(e, d_img, w, h, P, e->p<float>(B_SIFT), e->p<float>(B_TMP0), e->p<float>(B_TMP1), st);
}

}  // namespace

namespace {

// pyramid_position + border filter of describe_gradient (sift.cpp:84-91,
// 366-379) on the host: one descriptor job per surviving keypoint.
void describe_jobs(const SiftPyr& P, const xa_keypoint* kps, int n, std::vector<SiftJob>& jobs,
                   std::vector<int>& src) {
    for (int i = 0; i < n; ++i) {
        const xa_keypoint& kp = kps[i];
        if (kp.octave_scale <= 0) continue;
        const double t = 3 * std::log2(kp.octave_scale * 2.0 / 1.6);
        int o = static_cast<int>(std::floor((t - 0.5) / 3));
        o = std::clamp(o, 0, P.noct - 1);
        int l = static_cast<int>(std::lround(t - o * 3));
        l = std::clamp(l, 1, 3);
        const SiftImg& im = P.gauss[6 * o + l];
        const double of = std::pow(2.0, o) * 0.5;
        const float col = static_cast<float>(kp.x / of), row = static_cast<float>(kp.y / of);
        const double scl = kp.octave_scale / of;
        const float hw = 3.f * static_cast<float>(scl);
        const int radius = static_cast<int>(std::round(hw * std::sqrt(2.f) * (4 + 1) * 0.5f));
        if (col < radius || row < radius || col >= im.w - radius || row >= im.h - radius) continue;
        jobs.push_back({6 * o + l, col, row, kp.orientation, scl});
        src.push_back(i);
    }
}

// One simulated view of the ASIFT baseline (pipeline.cpp:242-266).
struct SimView {
    std::vector<xa_keypoint> kps;  // described keypoints
    Mat3 back;
    long long desc_off = 0;  // first descriptor row in the side's buffer
};

// XA_ASIFT_TIMING=1: phase wall times of xa_asift_correspondences on stderr
struct PhaseClock {
    bool on = std::getenv("XA_ASIFT_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(cudaStream_t st, const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "asift %-14s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// simulate_views (pipeline.cpp:242-266) for one image on the device: every
// grid entry at scale 1, anti-alias blur + Lanczos float views in one batch,
// then SIFT on every view with ONE pyramid per view for detection and
// description. Views go through in chunks whose pyramids, candidates and
// keypoints have their own device slots, so a chunk's launches run back to
// back with two host round trips (candidate and keypoint counts) per chunk
// instead of per view. Descriptors of all views are concatenated in desc_buf.
int asift_side(xa_engine* e, const float* img, int w, int h, const xa_params* grid, int n,
               int max_points, int a, Buf desc_buf, std::vector<SimView>& views, long long& ndesc,
               cudaStream_t st) {
    std::vector<xa_params> g(grid, grid + n);
    for (auto& p : g) p.scale = 1.0;  // no scale series in the baseline
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    ViewPlan V;
    RET(plan_views(g.data(), n, w, h, XA_LANCZOS, e->buf[B_IN0], XA_PIX_F32, V));
    RET(e->ensure(B_VIEW, sizeof(float) * (size_t)V.out_elems));
    RET(e->ensure(desc_buf, sizeof(float) * 128 * (size_t)n * (size_t)max_points));
    PhaseClock clk;
    RET(run_views(e, V, e->buf[B_IN0], XA_PIX_F32, w, h, XA_LANCZOS, XA_PIX_F32, e->buf[B_VIEW], st));
    clk.lap(st, "views");
    views.assign(n, SimView());
    ndesc = 0;
    const float prelim = static_cast<float>(0.5 * 0.03 / 3 * 255.0);
    const int ccap = 1 << 18, kcap = 1 << 17;
    size_t tmp_floats = 0;
    for (const Frame& f : V.frames) tmp_floats = std::max(tmp_floats, 4 * (size_t)f.W * f.H);
    RET(e->ensure(B_TMP0, sizeof(float) * tmp_floats));
    RET(e->ensure(B_TMP1, sizeof(float) * tmp_floats));
    constexpr int kChunk = 8;
    for (int v0 = 0; v0 < n; v0 += kChunk) {
        const int nb = std::min(kChunk, n - v0);
        Tables T;
        std::vector<SiftPyr> P(nb);
        std::vector<long long> soff(nb + 1, 0);
        for (int b = 0; b < nb; ++b) {
            const Frame& f = V.frames[v0 + b];
            if (f.W >= 64 && f.H >= 64) sift_layout(f.W, f.H, P[b], T);  // sift.cpp:291
            soff[b + 1] = soff[b] + align_up(P[b].floats, 64);
        }
        RET(e->ensure(B_SIFT, sizeof(float) * std::max<long long>(soff[nb], 1)));
        RET(e->ensure(B_SCAND, sizeof(SiftCand) * (size_t)ccap * nb));
        RET(e->ensure(B_SKP, sizeof(xa_kp) * (size_t)kcap * nb));
        RET(e->ensure(B_OUT, sizeof(int) * 2 * kChunk));
        RET(upload_tables(e, T, st));
        int* cnt = e->p<int>(B_OUT);
        CK(cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * nb, st));
        float* S0 = e->p<float>(B_SIFT);
        for (int b = 0; b < nb; ++b) {
            if (!P[b].noct) continue;
            const Frame& f = V.frames[v0 + b];
            float* S = S0 + soff[b];
            RET(sift_enqueue(e, e->p<float>(B_VIEW) + V.warp[v0 + b].out_off, f.W, f.H, P[b], S,
                             e->p<float>(B_TMP0), e->p<float>(B_TMP1), st));
            for (int o = 0; o < P[b].noct; ++o)
                for (int layer = 1; layer <= 3; ++layer)
                    e->last_launches += launch_dog_extrema(
                        S, P[b].dog[5 * o + layer - 1], P[b].dog[5 * o + layer], P[b].dog[5 * o + layer + 1],
                        prelim, o, layer, e->p<SiftCand>(B_SCAND) + (size_t)ccap * b, cnt + 2 * b, ccap, st);
        }
        int hc[2 * kChunk];
        CK(cudaMemcpyAsync(hc, cnt, sizeof(int) * 2 * nb, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int b = 0; b < nb; ++b) {
            if (hc[2 * b] > ccap) return set_err(XA_ECAPACITY, "detect_dog: candidate capacity");
            if (!P[b].noct || !hc[2 * b]) continue;
            e->last_launches += launch_sift_keypoints(
                S0 + soff[b], tab<SiftImg>(e, P[b].og), tab<SiftImg>(e, P[b].od),
                e->p<SiftCand>(B_SCAND) + (size_t)ccap * b, cnt + 2 * b, hc[2 * b],
                e->p<xa_kp>(B_SKP) + (size_t)kcap * b, cnt + 2 * b + 1, kcap, st);
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hc, cnt, sizeof(int) * 2 * nb, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<std::vector<xa_keypoint>> K(nb);
        for (int b = 0; b < nb; ++b) {
            if (hc[2 * b + 1] > kcap) return set_err(XA_ECAPACITY, "detect_dog: keypoint capacity");
            K[b].resize(hc[2 * b + 1]);
            if (!K[b].empty())
                CK(cudaMemcpyAsync(K[b].data(), e->p<xa_kp>(B_SKP) + (size_t)kcap * b,
                                   sizeof(xa_kp) * K[b].size(), cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
        // sort_and_cap (sift.cpp:279-286), filter_to_content (pipeline.cpp:28-40,
        // not on the identity view), describe jobs (sift.cpp:360-379)
        std::vector<SiftJob> jobs;
        std::vector<int> jstart(nb + 1, 0);
        for (int b = 0; b < nb; ++b) {
            const int i = v0 + b;
            const xa_params& p = g[i];
            const bool identity = p.tilt == 1.0 && p.phi == 0.0 && p.scale == 1.0;
            SimView& v = views[i];
            v.back = V.frames[i].back;
            std::vector<xa_keypoint>& k = K[b];
            std::sort(k.begin(), k.end(), [](const xa_keypoint& x, const xa_keypoint& y) {
                if (x.response != y.response) return x.response > y.response;
                if (x.y != y.y) return x.y < y.y;
                if (x.x != y.x) return x.x < y.x;
                return x.orientation < y.orientation;
            });
            k.resize(std::min<size_t>(k.size(), (size_t)max_points));
            if (!identity) {
                std::vector<xa_keypoint> kept;
                for (const auto& kp : k) {
                    double sx, sy;
                    map_pt_h(v.back, kp.x, kp.y, sx, sy);
                    if (sx >= a && sx <= w - 1 - a && sy >= a && sy <= h - 1 - a) kept.push_back(kp);
                }
                k.swap(kept);
            }
            std::vector<int> src;
            if (P[b].noct) describe_jobs(P[b], k.data(), (int)k.size(), jobs, src);
            for (const int q : src) v.kps.push_back(k[q]);
            jstart[b + 1] = (int)jobs.size();
        }
        if (!jobs.empty()) {
            RET(e->ensure(B_SJOB, sizeof(SiftJob) * jobs.size()));
            RET(e->ensure_staging(sizeof(SiftJob) * jobs.size()));
            std::memcpy(e->staging, jobs.data(), sizeof(SiftJob) * jobs.size());
            CK(cudaMemcpyAsync(e->buf[B_SJOB], e->staging, sizeof(SiftJob) * jobs.size(),
                               cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(e->staging_done, st));
        }
        for (int b = 0; b < nb; ++b) {
            SimView& v = views[v0 + b];
            v.desc_off = ndesc;
            const int m = jstart[b + 1] - jstart[b];
            if (m)
                e->last_launches += launch_sift_describe(
                    S0 + soff[b], tab<SiftImg>(e, P[b].og), e->p<SiftJob>(B_SJOB) + jstart[b], m,
                    e->p<float>(desc_buf) + 128 * (size_t)ndesc, st);
            ndesc += m;
        }
        CK(cudaGetLastError());
    }
    clk.lap(st, "sift");
    return XA_OK;
}

// Duplicate suppression of the baseline's merged list (pipeline.cpp:268-296):
// a correspondence repeats an earlier one when both endpoints lie within 2 px.
// Earlier ones are bucketed by the 2-px cell of their first endpoint, so only
// the 3x3 neighbouring cells can hold a repeat.
class Repeats {
public:
    explicit Repeats(const std::vector<xa_correspondence>& all) : all_(all) {}
    bool seen(const xa_correspondence& c) const {
        const long long cx = cell(c.x1), cy = cell(c.y1);
        for (long long gy = cy - 1; gy <= cy + 1; ++gy)
            for (long long gx = cx - 1; gx <= cx + 1; ++gx) {
                const auto it = grid_.find(pack(gx, gy));
                if (it == grid_.end()) continue;
                for (const int k : it->second) {
                    const xa_correspondence& o = all_[k];
                    if (std::hypot(o.x1 - c.x1, o.y1 - c.y1) <= 2.0 &&
                        std::hypot(o.x2 - c.x2, o.y2 - c.y2) <= 2.0)
                        return true;
                }
            }
        return false;
    }
    void add(int k) { grid_[pack(cell(all_[k].x1), cell(all_[k].y1))].push_back(k); }

private:
    static long long cell(double v) { return (long long)std::floor(v / 2.0); }
    static uint64_t pack(long long x, long long y) {
        return ((uint64_t)(uint32_t)x << 32) | (uint64_t)(uint32_t)y;
    }
    const std::vector<xa_correspondence>& all_;
    std::unordered_map<uint64_t, std::vector<int>> grid_;
};

}  // namespace

// =================================================================== C ABI

extern "C" {

const char* xa_last_error(void) { return g_err.c_str(); }
int xa_version(void) { return 1; }
uint64_t xa_pattern_checksum(void) { return pattern_checksum_host(); }
int xa_trig_fixups(void) { return trig_fixup_count(); }

int xa_engine_create(int device, xa_engine** out) {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return set_err(XA_EINVAL, "no such CUDA device");
    CK(cudaSetDevice(device));
    xa_engine* e = new xa_engine();
    e->device = device;
    CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&e->staging_done, cudaEventDisableTiming));
    CK(cudaMalloc(&e->d_flags, 64));
    CK(cudaMemset(e->d_flags, 0, 64));
    if (orb_init_constants() || warp_init_attributes() || match_umma_init())
        return set_err(XA_ECUDA, "constant upload / kernel attribute setup failed");
    *out = e;
    return XA_OK;
}

int xa_engine_destroy(xa_engine* e) {
    if (!e) return XA_OK;
    cudaSetDevice(e->device);
    cudaStreamSynchronize(e->stream);
    for (int b = 0; b < B_COUNT; ++b)
        if (e->buf[b]) cudaFree(e->buf[b]);
    if (e->staging) cudaFreeHost(e->staging);
    if (e->staging_done) cudaEventDestroy(e->staging_done);
    if (e->d_flags) cudaFree(e->d_flags);
    delete e->cc;
    for (cudaEvent_t ev : e->marks) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->pair_ready) cudaEventDestroy(ev);
    if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
    cudaStreamDestroy(e->stream);
    delete e;
    return XA_OK;
}

void* xa_engine_stream(xa_engine* e) { return e ? (void*)e->stream : nullptr; }

size_t xa_engine_workspace_bytes(xa_engine* e) {
    size_t s = 0;
    for (int b = 0; b < B_COUNT; ++b) s += e->cap[b];
    return s;
}

int xa_engine_last_launches(xa_engine* e) { return e ? e->last_launches : 0; }

}  // extern "C" (reopened below)

namespace xa {
// error reporting for the host-only translation units (xa_image_io.cpp)
int host_error(int code, const std::string& msg) { return set_err(code, msg); }
}  // namespace xa

extern "C" {

// Diagnostics: copy the first `floats` floats of the ORB pyramid buffer (the
// levels of the last detect/describe/coarse call) to the host.
int xa_engine_read_pyramid(xa_engine* e, float* out, size_t floats) {
    if (!e->buf[B_PYR] || floats * sizeof(float) > e->cap[B_PYR]) return set_err(XA_EINVAL, "pyramid size");
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, e->buf[B_PYR], floats * sizeof(float), cudaMemcpyDeviceToHost));
    return XA_OK;
}

// Per-image ORB counters of the last detect/coarse call: for image i (0 = the
// coarse target, 1..n = views) out[5*i..] = candidates, thr-20 survivors,
// thr-7 survivors (auto-relaxed images only), detected keypoints, described keypoints.
int xa_engine_orb_counters(xa_engine* e, int cap_images, int32_t* out, int* n_images) {
    *n_images = 0;
    const Buf b = e->cnt_all ? B_CNTALL : B_CNT;
    if (!e->buf[b]) return XA_OK;
    const int n = std::min<int>({cap_images, e->orb_images, (int)(e->cap[b] / sizeof(ImgCounters))});
    std::vector<ImgCounters> h(n);
    CK(cudaDeviceSynchronize());  // the coarse call may have run on a caller stream
    CK(cudaMemcpy(h.data(), e->buf[b], sizeof(ImgCounters) * n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) {
        out[5 * i] = h[i].n_cand;
        out[5 * i + 1] = h[i].n20;
        out[5 * i + 2] = h[i].n7;
        out[5 * i + 3] = h[i].n_det;
        out[5 * i + 4] = h[i].n_desc;
    }
    *n_images = n;
    return XA_OK;
}

int xa_engine_set_profiling(xa_engine* e, int on) {
    e->profiling = on ? 1 : 0;
    e->nmarks = 0;
    return XA_OK;
}

int xa_engine_stage_times(xa_engine* e, int cap, float* ms, const char** names, int* n) {
    *n = 0;
    if (e->nmarks < 2) return XA_OK;
    CK(cudaEventSynchronize(e->marks[e->nmarks - 1]));
    int k = 0;
    for (int i = 1; i < e->nmarks && k < cap; ++i, ++k) {
        CK(cudaEventElapsedTime(&ms[k], e->marks[i - 1], e->marks[i]));
        names[k] = e->mark_names[i];
    }
    *n = k;
    return XA_OK;
}

// Reads (and clears) the overflow flag raised by earlier _device calls.
int xa_engine_check(xa_engine* e) {
    int f = 0;
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&f, e->d_flags, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(e->d_flags, 0, sizeof(int)));
    if (f) {
        // the next coarse plan sizes the candidate buffers with a larger factor
        e->cand_factor = std::min(0.5, e->cand_factor * 4);
        return set_err(XA_ECAPACITY, "ORB capacity exceeded in a device call");
    }
    return XA_OK;
}

int xa_simulation_from_params(const xa_params* p, double m[9]) {
    RET(check_params(*p, "simulation_from_params"));
    const Mat3 r = compose_params(&p->psi, true);
    std::memcpy(m, r.m, sizeof r.m);
    return XA_OK;
}

int xa_affine_from_params(const xa_params* p, double m[9]) {
    RET(check_params(*p, "affine_from_params"));
    const Mat3 r = compose_params(&p->psi, false);
    std::memcpy(m, r.m, sizeof r.m);
    return XA_OK;
}

int xa_invert(const double m[9], double out[9]) {
    Mat3 a, r;
    std::memcpy(a.m, m, sizeof a.m);
    if (!mat_inv(a, r)) return set_err(XA_ESINGULAR, "invert: singular matrix");
    std::memcpy(out, r.m, sizeof r.m);
    return XA_OK;
}

int xa_build_param_grid(double a, int n, double b_deg, double delta_s, xa_params* out, int cap,
                        int* count) {
    if (a <= 1.0) return set_err(XA_EINVAL, "build_param_grid: a must be > 1");
    if (n < 0) return set_err(XA_EINVAL, "build_param_grid: n must be >= 0");
    const std::vector<double> g = param_grid(a, n, b_deg, delta_s);
    const int cnt = (int)(g.size() / 6);
    *count = cnt;
    if (out) {
        if (cap < cnt) return set_err(XA_ECAPACITY, "build_param_grid: output capacity");
        std::memcpy(out, g.data(), sizeof(double) * g.size());
    }
    return XA_OK;
}

int xa_warp_frame(const double m[9], int w, int h, int* W, int* H, double* tx, double* ty,
                  double forward[9]) {
    Mat3 a;
    std::memcpy(a.m, m, sizeof a.m);
    Frame f;
    if (warp_frame(a, w, h, false, f)) return set_err(XA_ESINGULAR, "invert: singular matrix");
    *W = f.W;
    *H = f.H;
    *tx = f.tx;
    *ty = f.ty;
    if (forward) std::memcpy(forward, f.forward.m, sizeof f.forward.m);
    return XA_OK;
}

int xa_gaussian_blur(xa_engine* e, const float* img, int w, int h, double sigma, float* out) {
    const size_t n = (size_t)w * h;
    if (sigma <= 0 || n == 0) {
        if (n) std::memcpy(out, img, sizeof(float) * n);
        return XA_OK;
    }
    CK(cudaSetDevice(e->device));
    const int r = std::max(1, static_cast<int>(std::ceil(3.0 * sigma)));
    std::vector<float> k(2 * r + 1);
    double sum = 0;
    for (int i = -r; i <= r; ++i) {
        const double v = std::exp(-0.5 * i * i / (sigma * sigma));
        k[i + r] = static_cast<float>(v);
        sum += v;
    }
    for (auto& v : k) v = static_cast<float>(v / sum);
    e->last_launches = 0;
    RET(upload(e, B_IN0, img, sizeof(float) * n));
    RET(upload(e, B_SCRATCH, k.data(), sizeof(float) * k.size()));
    RET(e->ensure(B_TMP0, sizeof(float) * n));
    RET(e->ensure(B_TMP1, sizeof(float) * n));
    e->last_launches += launch_gauss(e->p<float>(B_IN0), e->p<float>(B_TMP0), e->p<float>(B_TMP1), w,
                                     h, e->p<float>(B_SCRATCH), r, e->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, e->buf[B_TMP1], sizeof(float) * n, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return XA_OK;
}

int xa_resize_bilinear(xa_engine* e, const float* img, int w, int h, int nw, int nh, float* out) {
    if (nw <= 0 || nh <= 0) return XA_OK;
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    RET(e->ensure(B_TMP0, sizeof(float) * (size_t)nw * nh));
    e->last_launches += launch_resize(e->p<float>(B_IN0), w, h, e->p<float>(B_TMP0), nw, nh, e->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, e->buf[B_TMP0], sizeof(float) * (size_t)nw * nh, cudaMemcpyDeviceToHost,
                       e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return XA_OK;
}

int xa_antialias_tilt(xa_engine* e, const float* img, int w, int h, double t, double phi,
                      float* out) {
    if (t < 1.0) return set_err(XA_EINVAL, "antialias_tilt: tilt must be >= 1");
    const size_t n = (size_t)w * h;
    if (t == 1.0 || n == 0) {
        if (n) std::memcpy(out, img, sizeof(float) * n);
        return XA_OK;
    }
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    std::vector<BlurView> bv(1);
    std::vector<BlurTap> taps;
    RET(blur_taps(t, phi, bv[0], taps));
    bv[0].out_off = 0;
    RET(upload(e, B_IN0, img, sizeof(float) * n));
    RET(e->ensure(B_TMP0, sizeof(float) * n));
    Tables T;
    const size_t ob = T.add(bv), ot = T.add(taps);
    RET(upload_tables(e, T, e->stream));
    e->last_launches += launch_antialias(tab<BlurView>(e, ob), tab<BlurTap>(e, ot), 1, e->buf[B_IN0],
                                         XA_PIX_F32, w, h, e->p<float>(B_TMP0), e->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, e->buf[B_TMP0], sizeof(float) * n, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return XA_OK;
}

int xa_warp(xa_engine* e, int mode, const float* img, int w, int h, const double m[9], int a,
            float* out, size_t out_cap, int* W, int* H, double* tx, double* ty, double forward[9]) {
    if (mode == XA_LANCZOS && a != 4)
        return set_err(XA_EINVAL, "warp_lanczos: the device resampler implements a = 4 only");
    Mat3 mm;
    std::memcpy(mm.m, m, sizeof mm.m);
    Frame f;
    if (warp_frame(mm, w, h, mode == XA_NEAREST, f)) return set_err(XA_ESINGULAR, "invert: singular matrix");
    *W = f.W;
    *H = f.H;
    *tx = f.tx;
    *ty = f.ty;
    if (forward) std::memcpy(forward, f.forward.m, sizeof f.forward.m);
    const size_t no = (size_t)f.W * f.H;
    if (!out) return XA_OK;  // frame query
    if (out_cap < no) return set_err(XA_ECAPACITY, "warp: output capacity");
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    RET(e->ensure(B_TMP0, sizeof(float) * no));
    ViewPlan V;
    V.frames.push_back(f);
    V.blur_of.push_back(-1);
    WarpView wv;
    std::memset(&wv, 0, sizeof wv);
    for (int k = 0; k < 6; ++k) wv.back[k] = f.back.m[k];
    wv.W = f.W;
    wv.H = f.H;
    wv.sw = w;
    wv.sh = h;
    wv.src = e->buf[B_IN0];
    wv.src_type = XA_PIX_F32;
    RET(warp_tiling(wv, w, h, mode, V.warp_smem));
    V.warp_tiles = wv.tiles_x * ((f.H + wv.tile_h - 1) / wv.tile_h);
    V.warp.push_back(wv);
    RET(run_views(e, V, e->buf[B_IN0], XA_PIX_F32, w, h, mode, XA_PIX_F32, e->buf[B_TMP0], e->stream));
    CK(cudaMemcpyAsync(out, e->buf[B_TMP0], sizeof(float) * no, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return XA_OK;
}

int xa_synth_warp_case(xa_engine* e, const float* img, int w, int h, const double hm[9], int out_type,
                       void* out, size_t out_cap, int* W, int* H, double composed[9]) {
    if (w <= 0 || h <= 0) return set_err(XA_EINVAL, "synth_warp_case: empty image");
    if (out_type != XA_U8 && out_type != XA_F32) return set_err(XA_EINVAL, "synth_warp_case: out_type");
    Mat3 mm;
    std::memcpy(mm.m, hm, sizeof mm.m);
    Frame f;
    switch (synth_frame(mm, w, h, f)) {
        case 1: return set_err(XA_EEVAL, "degenerate homography for synthetic warp");
        case 2: return set_err(XA_EEVAL, "degenerate homography: unbounded warp target");
        case 3: return set_err(XA_EEVAL, "degenerate homography: not invertible");
        default: break;
    }
    *W = f.W;
    *H = f.H;
    if (composed) std::memcpy(composed, f.forward.m, sizeof f.forward.m);
    const size_t no = (size_t)f.W * f.H;
    if (!out) return XA_OK;  // frame query
    if (out_cap < no) return set_err(XA_ECAPACITY, "synth_warp_case: output capacity");
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    const size_t esz = out_type == XA_U8 ? 1 : sizeof(float);
    RET(e->ensure(B_TMP0, esz * no));
    ProjView pv;
    std::memcpy(pv.back, f.back.m, sizeof pv.back);
    pv.W = f.W;
    pv.H = f.H;
    e->last_launches += launch_warp_projective((const float*)e->buf[B_IN0], w, h, pv,
                                               out_type == XA_U8 ? XA_PIX_U8 : XA_PIX_F32,
                                               e->buf[B_TMP0], e->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, e->buf[B_TMP0], esz * no, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return XA_OK;
}

int xa_detect_oriented_corners(xa_engine* e, const float* img, int w, int h, int max_points,
                               xa_keypoint* out, int cap, int* n) {
    *n = 0;
    if (w < kMinSide || h < kMinSide || max_points <= 0) return XA_OK;  // orb.cpp:183
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    std::vector<OrbSrc> srcs = {{e->buf[B_IN0], XA_PIX_F32, w, h, false, 0, 0, Mat3()}};
    for (double factor = 0.125;; factor *= 4) {
        OrbPlan P = plan_orb(srcs, max_points, std::min(factor, 1.0));
        RET(ensure_orb(e, P));
        Tables T;
        OrbDev D;
        D.imgs_off = T.add(P.imgs);
        D.pyr_off = T.add(P.pyr_segs);
        D.fast_off = T.add(P.fast_segs);
        D.rng_off = T.add(P.fast_rng);
        std::vector<TMap> maps;
        RET(encode_level_maps(P.imgs, e->p<float>(B_PYR), maps));
        D.maps_off = T.add(maps);
        RET(upload_tables(e, T, e->stream));
        RET(run_detect(e, P, D, e->stream));
        std::vector<ImgCounters> hc;
        const int rc = check_counters(e, 1, hc);
        if (rc == XA_ECAPACITY && hc[0].overflow == 1 && factor < 1.0) continue;
        RET(rc);
        if (hc[0].n_det > cap) return set_err(XA_ECAPACITY, "detect: output capacity");
        CK(cudaMemcpy(out, e->buf[B_DET], sizeof(xa_kp) * hc[0].n_det, cudaMemcpyDeviceToHost));
        *n = hc[0].n_det;
        return XA_OK;
    }
}

int xa_detect_dog_keypoints(xa_engine* e, const float* img, int w, int h, int max_points,
                            xa_keypoint* out, int cap, int* n) {
    *n = 0;
    if (w < 64 || h < 64 || max_points <= 0) return XA_OK;  // sift.cpp:291
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    cudaStream_t st = e->stream;
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    Tables T;
    SiftPyr P;
    RET(sift_pyramid(e, e->p<float>(B_IN0), w, h, P, T, st));
    const int ccap = 1 << 20, kcap = 1 << 20;
    RET(e->ensure(B_SCAND, sizeof(SiftCand) * ccap));
    RET(e->ensure(B_SKP, sizeof(xa_kp) * kcap));
    RET(e->ensure(B_OUT, 64));
    int* cnt = e->p<int>(B_OUT);
    CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), st));
    const float prelim = static_cast<float>(0.5 * 0.03 / 3 * 255.0);
    const float* S = e->p<float>(B_SIFT);
    for (int o = 0; o < P.noct; ++o)
        for (int layer = 1; layer <= 3; ++layer)
            e->last_launches += launch_dog_extrema(S, P.dog[5 * o + layer - 1], P.dog[5 * o + layer],
                                                   P.dog[5 * o + layer + 1], prelim, o, layer,
                                                   e->p<SiftCand>(B_SCAND), cnt, ccap, st);
    int hc[2] = {0, 0};
    CK(cudaMemcpyAsync(hc, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hc[0] > ccap) return set_err(XA_ECAPACITY, "detect_dog: candidate capacity");
    e->last_launches += launch_sift_keypoints(S, tab<SiftImg>(e, P.og), tab<SiftImg>(e, P.od),
                                              e->p<SiftCand>(B_SCAND), cnt, hc[0], e->p<xa_kp>(B_SKP),
                                              cnt + 1, kcap, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(hc + 1, cnt + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hc[1] > kcap) return set_err(XA_ECAPACITY, "detect_dog: keypoint capacity");
    std::vector<xa_kp> k(hc[1]);
    if (hc[1]) CK(cudaMemcpy(k.data(), e->buf[B_SKP], sizeof(xa_kp) * hc[1], cudaMemcpyDeviceToHost));
    // sort_and_cap (sift.cpp:279-286); keypoints equal in (response, y, x)
    // (orientations of one extremum) have no defined order in the reference's
    // std::sort: they are ordered by orientation here
    std::sort(k.begin(), k.end(), [](const xa_kp& a, const xa_kp& b) {
        if (a.response != b.response) return a.response > b.response;
        if (a.y != b.y) return a.y < b.y;
        if (a.x != b.x) return a.x < b.x;
        return a.orientation < b.orientation;
    });
    const int m = std::min<int>((int)k.size(), max_points);
    if (m > cap) return set_err(XA_ECAPACITY, "detect_dog: output capacity");
    std::memcpy(out, k.data(), sizeof(xa_kp) * m);
    *n = m;
    return XA_OK;
}

int xa_describe_gradient(xa_engine* e, const float* img, int w, int h, const xa_keypoint* kps, int n,
                         xa_keypoint* out_kps, float* out_desc, int* n_out) {
    *n_out = 0;
    if (w < 64 || h < 64 || n <= 0) return XA_OK;  // sift.cpp:363
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    cudaStream_t st = e->stream;
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    Tables T;
    SiftPyr P;
    RET(sift_pyramid(e, e->p<float>(B_IN0), w, h, P, T, st));
    std::vector<SiftJob> jobs;
    std::vector<int> src;
    describe_jobs(P, kps, n, jobs, src);
    const int m = (int)jobs.size();
    if (!m) return XA_OK;
    RET(e->ensure(B_SJOB, sizeof(SiftJob) * m));
    RET(e->ensure(B_SDESC, sizeof(float) * 128 * (size_t)m));
    CK(cudaMemcpyAsync(e->buf[B_SJOB], jobs.data(), sizeof(SiftJob) * m, cudaMemcpyHostToDevice, st));
    e->last_launches += launch_sift_describe(e->p<float>(B_SIFT), tab<SiftImg>(e, P.og),
                                             e->p<SiftJob>(B_SJOB), m, e->p<float>(B_SDESC), st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_desc, e->buf[B_SDESC], sizeof(float) * 128 * (size_t)m, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int j = 0; j < m; ++j) out_kps[j] = kps[src[j]];
    *n_out = m;
    return XA_OK;
}

int xa_describe_binary(xa_engine* e, const float* img, int w, int h, const xa_keypoint* kps, int n,
                       xa_keypoint* out_kps, uint64_t* out_desc, int* n_out) {
    *n_out = 0;
    if (n <= 0 || w <= 0 || h <= 0) return XA_OK;
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    RET(upload(e, B_IN0, img, sizeof(float) * (size_t)w * h));
    RET(upload(e, B_IN1, kps, sizeof(xa_kp) * n));
    std::vector<OrbSrc> srcs = {{e->buf[B_IN0], XA_PIX_F32, w, h, false, 0, 0, Mat3()}};
    OrbPlan P = plan_orb(srcs, n, 0.0);
    RET(ensure_orb(e, P));
    Tables T;
    OrbDev D;
    D.imgs_off = T.add(P.imgs);
    D.pyr_off = T.add(P.pyr_segs);
    RET(upload_tables(e, T, e->stream));
    const OrbImage* imgs = tab<OrbImage>(e, D.imgs_off);
    CK(cudaMemsetAsync(e->buf[B_CNT], 0, sizeof(ImgCounters), e->stream));
    e->orb_images = 1;
    e->cnt_all = false;
    int L = 0;
    L += launch_pyramid(imgs, tab<LevelSeg>(e, D.pyr_off), (int)P.pyr_segs.size(), P.pyr_blocks,
                        e->p<float>(B_PYR), e->stream);
    L += launch_describe_prep(imgs, e->p<xa_kp>(B_IN1), n, e->p<ImgCounters>(B_CNT),
                              e->p<DescKp>(B_DESCIN), e->p<xa_kp>(B_DESCKP), e->stream);
    L += launch_describe(imgs, 1, e->p<float>(B_PYR), e->p<ImgCounters>(B_CNT), e->p<DescKp>(B_DESCIN),
                         e->p<uint64_t>(B_DESC), e->stream);
    CK(cudaGetLastError());
    e->last_launches = L;
    std::vector<ImgCounters> hc;
    RET(check_counters(e, 1, hc));
    const int m = hc[0].n_desc;
    CK(cudaMemcpy(out_kps, e->buf[B_DESCKP], sizeof(xa_kp) * m, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_desc, e->buf[B_DESC], 32 * (size_t)m, cudaMemcpyDeviceToHost));
    *n_out = m;
    return XA_OK;
}

int xa_match_hamming_device(xa_engine* e, const uint64_t* d_a, int na, const uint64_t* d_b, int nb,
                            double ratio, uint32_t* d_best_idx, uint16_t* d_best,
                            uint16_t* d_second, int32_t* d_count, void* stream) {
    cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    RET(e->set_ratio(ratio, st));
    if (d_count) CK(cudaMemsetAsync(d_count, 0, sizeof(int32_t), st));
    if (na <= 0 || nb <= 0) return XA_OK;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
    const int qblocks = (na + 511) / 512;
    int nsplit = std::max(1, std::min((sms * 8 + qblocks - 1) / qblocks, (nb + 1023) / 1024));
    RET(e->ensure(B_SCRATCH, match_large_scratch(na, nsplit)));
    int* cnt = d_count;
    if (!cnt) {
        RET(e->ensure(B_OUT, 64));
        cnt = e->p<int>(B_OUT);
        CK(cudaMemsetAsync(cnt, 0, sizeof(int), st));
    }
    if (use_umma() && (long long)na + nb < (1LL << 22)) {
        // tcgen05 matcher: queries as rows [0, na), train as rows [na, na + nb)
        // of one expanded +-1 buffer; train slices so every SM gets >= 8 items
        RET(e->ensure(B_PM1, 256 * ((size_t)na + nb)));
        const int qb = (na + 255) / 256;
        // train slices: the fewest waves per unit of work over 1..4 slices
        // (ceil(items / SMs) / slices; fewer slices on ties: each item reloads
        // its query block), at least 1024 train rows per slice
        int split = 1;
        double best_cost = 1e30;
        for (int sp = 1; sp <= 4 && (sp == 1 || nb / sp >= 1024); ++sp) {
            const double cost = (double)((qb * sp + sms - 1) / sms) / sp;
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                split = sp;
            }
        }
        if (const char* sv = std::getenv("XA_UMMA_SPLIT")) split = std::max(1, std::atoi(sv));  // A/B
        RET(e->ensure(B_SCRATCH, sizeof(uint2) * (size_t)na * split));
        TMap map[2];
        RET(encode_pm1_maps(map, e->buf[B_PM1], (long long)na + nb));
        MatchJob one{};
        one.na = na;
        one.nb = nb;
        one.b_off = na;
        one.count_out = cnt;
        e->mark_begin(st);
        int L = launch_desc_pm1(d_a, na, e->buf[B_PM1], st);
        L += launch_desc_pm1(d_b, nb, static_cast<char*>(e->buf[B_PM1]) + 256 * (size_t)na, st);
        L += launch_match_umma(nullptr, one, 1, na, split, map, e->p<uint16_t>(B_KEEP), d_best_idx, d_best,
                               d_second, split > 1 ? e->buf[B_SCRATCH] : nullptr, sms, st);
        if (split > 1)
            L += launch_match_tc_merge(e->buf[B_SCRATCH], na, split, e->p<uint16_t>(B_KEEP), d_best_idx, d_best,
                                       d_second, cnt, st);
        e->last_launches += L;
        e->mark(st, "hamming");
        CK(cudaGetLastError());
        return XA_OK;
    }
    e->mark_begin(st);
    e->last_launches += launch_match_large(d_a, na, d_b, nb, e->p<uint16_t>(B_KEEP), d_best_idx, d_best,
                                           d_second, cnt, e->buf[B_SCRATCH], nsplit, st);
    e->mark(st, "hamming");
    CK(cudaGetLastError());
    return XA_OK;
}

int xa_match_hamming(xa_engine* e, const uint64_t* a, int na, const uint64_t* b, int nb,
                     double ratio, xa_match* out, int* n_out) {
    *n_out = 0;
    if (na <= 0 || nb <= 0) return XA_OK;  // orb.cpp:254
    CK(cudaSetDevice(e->device));
    RET(upload(e, B_IN0, a, 32 * (size_t)na));
    RET(upload(e, B_IN1, b, 32 * (size_t)nb));
    RET(e->ensure(B_MIDX, sizeof(uint32_t) * na));
    RET(e->ensure(B_MBEST, sizeof(uint16_t) * na));
    RET(e->ensure(B_MSEC, sizeof(uint16_t) * na));
    RET(xa_match_hamming_device(e, e->p<uint64_t>(B_IN0), na, e->p<uint64_t>(B_IN1), nb, ratio,
                                e->p<uint32_t>(B_MIDX), e->p<uint16_t>(B_MBEST), e->p<uint16_t>(B_MSEC),
                                nullptr, e->stream));
    std::vector<uint32_t> idx(na);
    std::vector<uint16_t> best(na), sec(na);
    CK(cudaMemcpyAsync(idx.data(), e->buf[B_MIDX], 4 * (size_t)na, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(best.data(), e->buf[B_MBEST], 2 * (size_t)na, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(sec.data(), e->buf[B_MSEC], 2 * (size_t)na, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    int m = 0;
    for (int i = 0; i < na; ++i)
        if (best[i] < ratio * sec[i]) out[m++] = {i, (int32_t)idx[i], (float)best[i]};
    *n_out = m;
    return XA_OK;
}

int xa_match_ratio_device(xa_engine* e, const float* d_a, int na, const float* d_b, int nb,
                          double ratio, int32_t* d_best_idx, float* d_dist, uint8_t* d_keep,
                          int32_t* d_count, void* stream) {
    cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    if (d_count) CK(cudaMemsetAsync(d_count, 0, sizeof(int32_t), st));
    if (na <= 0 || nb <= 0) return XA_OK;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
    const int nsplit = match_l2_split(na, nb, sms);
    if (nsplit > 1) RET(e->ensure(B_SCRATCH, match_l2_scratch(na, nsplit)));
    e->mark_begin(st);
    e->last_launches += launch_match_l2(d_a, na, d_b, nb, ratio, d_best_idx, d_dist, d_keep, d_count,
                                        e->buf[B_SCRATCH], nsplit, st);
    e->mark(st, "l2_ratio");
    CK(cudaGetLastError());
    return XA_OK;
}

int xa_match_ratio(xa_engine* e, const float* a, int na, const float* b, int nb, double ratio,
                   xa_match* out, int* n_out) {
    *n_out = 0;
    if (na <= 0 || nb <= 0) return XA_OK;  // sift.cpp:392
    CK(cudaSetDevice(e->device));
    RET(upload(e, B_IN0, a, sizeof(float) * 128 * (size_t)na));
    RET(upload(e, B_IN1, b, sizeof(float) * 128 * (size_t)nb));
    RET(e->ensure(B_MIDX, sizeof(int32_t) * na));
    RET(e->ensure(B_MBEST, sizeof(float) * na));
    RET(e->ensure(B_MSEC, na));
    RET(xa_match_ratio_device(e, e->p<float>(B_IN0), na, e->p<float>(B_IN1), nb, ratio,
                              e->p<int32_t>(B_MIDX), e->p<float>(B_MBEST), e->p<uint8_t>(B_MSEC),
                              nullptr, e->stream));
    std::vector<int32_t> idx(na);
    std::vector<float> dist(na);
    std::vector<uint8_t> keep(na);
    CK(cudaMemcpyAsync(idx.data(), e->buf[B_MIDX], 4 * (size_t)na, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(dist.data(), e->buf[B_MBEST], 4 * (size_t)na, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(keep.data(), e->buf[B_MSEC], (size_t)na, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    int m = 0;
    for (int i = 0; i < na; ++i)
        if (keep[i]) out[m++] = {i, idx[i], dist[i]};
    *n_out = m;
    return XA_OK;
}

int xa_coarse_search_device(xa_engine* e, int pixel_type, const void* d_ref, int w, int h,
                            const void* d_target, int tw, int th, const xa_params* grid, int n,
                            int max_points, double ratio, int warp_mode, int32_t* d_counts,
                            int32_t* d_kp_counts, void* stream) {
    CK(cudaSetDevice(e->device));
    return coarse_device(e, pixel_type, &d_ref, w, h, &d_target, tw, th, 1, grid, n, max_points, ratio,
                         warp_mode, d_counts, d_kp_counts, stream ? (cudaStream_t)stream : e->stream);
}

int xa_coarse_search_batch_device(xa_engine* e, int pixel_type, const void* const* d_refs, int w, int h,
                                  const void* const* d_targets, int tw, int th, int n_pairs,
                                  const xa_params* grid, int n, int max_points, double ratio,
                                  int warp_mode, int32_t* d_counts, int32_t* d_kp_counts, void* stream) {
    CK(cudaSetDevice(e->device));
    return coarse_device(e, pixel_type, d_refs, w, h, d_targets, tw, th, n_pairs, grid, n, max_points,
                         ratio, warp_mode, d_counts, d_kp_counts, stream ? (cudaStream_t)stream : e->stream);
}

int xa_coarse_search_batch(xa_engine* e, int pixel_type, const void* const* refs, int w, int h,
                           const void* const* targets, int tw, int th, int n_pairs, const xa_params* grid,
                           int n, int max_points, double ratio, int warp_mode, int32_t* counts,
                           int32_t* kp_counts, int32_t* best) {
    if (n <= 0 || !grid) return set_err(XA_EPIPELINE, "coarse: empty parameter grid");
    if (n_pairs <= 0 || !refs || !targets) return set_err(XA_EINVAL, "coarse: no image pairs");
    CK(cudaSetDevice(e->device));
    const size_t px = pixel_type == XA_U8 ? 1 : 4;
    const size_t rb = align_up(px * (size_t)w * h, 256), tb = align_up(px * (size_t)tw * th, 256);
    RET(e->ensure(B_IN0, rb * n_pairs));
    RET(e->ensure(B_IN1, tb * n_pairs));
    RET(e->ensure(B_MBEST, sizeof(int32_t) * 2 * (size_t)n * n_pairs));
    // H2D of every pair on the copy stream, one event per pair; the replayed
    // graph waits for a chunk's last pair before that chunk's first kernel, so
    // the copies of later chunks overlap the compute of earlier ones
    if (!e->copy_stream) CK(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    while ((int)e->pair_ready.size() < n_pairs) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        e->pair_ready.push_back(ev);
    }
    CK(cudaStreamSynchronize(e->stream));  // the buffers are free (previous calls are done)
    std::vector<const void*> dr(n_pairs), dt(n_pairs);
    for (int p = 0; p < n_pairs; ++p) {
        dr[p] = static_cast<char*>(e->buf[B_IN0]) + rb * p;
        dt[p] = static_cast<char*>(e->buf[B_IN1]) + tb * p;
        CK(cudaMemcpyAsync((void*)dr[p], refs[p], px * (size_t)w * h, cudaMemcpyHostToDevice, e->copy_stream));
        CK(cudaMemcpyAsync((void*)dt[p], targets[p], px * (size_t)tw * th, cudaMemcpyHostToDevice,
                           e->copy_stream));
        CK(cudaEventRecord(e->pair_ready[p], e->copy_stream));
    }
    const size_t nc = (size_t)n * n_pairs;
    std::vector<int32_t> hc(2 * nc);
    for (int attempt = 0;; ++attempt) {
        int32_t* dc = e->p<int32_t>(B_MBEST);
        CK(cudaMemsetAsync(e->d_flags, 0, sizeof(int), e->stream));
        RET(coarse_device(e, pixel_type, dr.data(), w, h, dt.data(), tw, th, n_pairs, grid, n, max_points,
                          ratio, warp_mode, dc, dc + nc, e->stream, e->pair_ready.data()));
        CK(cudaMemcpyAsync(hc.data(), dc, sizeof(int32_t) * 2 * nc, cudaMemcpyDeviceToHost, e->stream));
        int flag = 0;
        CK(cudaMemcpyAsync(&flag, e->d_flags, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        if (!flag) break;
        // an image had more NMS survivors than its candidate capacity: grow
        // the capacity (the next plan re-sizes the buffers) and run again
        if (e->cand_factor >= 0.5 || attempt >= 6)
            return set_err(XA_ECAPACITY, "coarse: ORB capacity exceeded");
        e->cand_factor = std::min(0.5, e->cand_factor * 4);
    }
    for (int p = 0; p < n_pairs; ++p) {
        int bc = -1, bi = 0;
        for (int i = 0; i < n; ++i) {
            const int32_t v = hc[(size_t)p * n + i];
            if (counts) counts[(size_t)p * n + i] = v;
            if (kp_counts) kp_counts[(size_t)p * n + i] = hc[nc + (size_t)p * n + i];
            if (v > bc) {  // pipeline.cpp:142-150
                bc = v;
                bi = i;
            }
        }
        if (best) best[p] = bi;
    }
    return XA_OK;
}

int xa_coarse_search(xa_engine* e, int pixel_type, const void* ref, int w, int h,
                     const void* target, int tw, int th, const xa_params* grid, int n,
                     int max_points, double ratio, int warp_mode, int32_t* counts,
                     int32_t* kp_counts, int32_t* best) {
    return xa_coarse_search_batch(e, pixel_type, &ref, w, h, &target, tw, th, 1, grid, n, max_points,
                                  ratio, warp_mode, counts, kp_counts, best);
}

int xa_simulate_views_device(xa_engine* e, const uint8_t* d_src, int w, int h, const xa_params* views,
                             int n, int warp_mode, uint8_t* d_out, int64_t* offsets, int* widths,
                             int* heights, size_t* out_bytes, void* stream) {
    cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    ViewPlan V;
    RET(plan_views(views, n, w, h, warp_mode, d_src, XA_PIX_U8, V));
    if (out_bytes) *out_bytes = V.out_elems;
    for (int i = 0; i < n; ++i) {
        if (offsets) offsets[i] = V.warp[i].out_off;
        if (widths) widths[i] = V.frames[i].W;
        if (heights) heights[i] = V.frames[i].H;
    }
    if (!d_out) return XA_OK;
    return run_views(e, V, d_src, XA_PIX_U8, w, h, warp_mode, XA_PIX_U8, d_out, st);
}

// asift_baseline (pipeline.cpp:298-343) up to the RANSAC screen: dual view
// simulation + SIFT on both images, one L2 ratio matching per view pair (all
// views of image 1 as one query set against each view of image 2), then the
// merge with duplicate suppression in the reference's pair order.
int xa_asift_correspondences(xa_engine* e, const float* img1, int w1, int h1, const float* img2,
                             int w2, int h2, const xa_params* grid, int n, int max_points,
                             double ratio, int lanczos_a, xa_correspondence* out, int cap,
                             int* n_out) {
    *n_out = 0;
    if (n <= 0) return set_err(XA_EINVAL, "asift: empty parameter grid");
    if (lanczos_a != 4) return set_err(XA_EINVAL, "warp_lanczos: the device resampler implements a = 4 only");
    CK(cudaSetDevice(e->device));
    e->last_launches = 0;
    cudaStream_t st = e->stream;
    std::vector<SimView> v1, v2;
    long long n1 = 0, n2 = 0;
    RET(asift_side(e, img1, w1, h1, grid, n, max_points, lanczos_a, B_ADESC1, v1, n1, st));
    RET(asift_side(e, img2, w2, h2, grid, n, max_points, lanczos_a, B_ADESC2, v2, n2, st));
    std::vector<xa_correspondence> merged;
    if (n1 > 0 && n2 > 0) {
        // per view j of image 2: (best index, distance, keep) for every query
        const size_t per = (size_t)n1 * n;
        RET(e->ensure(B_AMATCH, per * 9 + 64));
        int32_t* d_idx = e->p<int32_t>(B_AMATCH);
        float* d_dist = reinterpret_cast<float*>(d_idx + per);
        uint8_t* d_keep = reinterpret_cast<uint8_t*>(d_dist + per);
        CK(cudaMemsetAsync(d_keep, 0, per, st));
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
        for (int j = 0; j < n; ++j) {
            const int nb = (int)v2[j].kps.size();
            if (!nb) continue;
            const int nsplit = match_l2_split((int)n1, nb, sms);
            if (nsplit > 1) RET(e->ensure(B_SCRATCH, match_l2_scratch((int)n1, nsplit)));
            e->last_launches += launch_match_l2(e->p<float>(B_ADESC1), (int)n1,
                                                e->p<float>(B_ADESC2) + 128 * (size_t)v2[j].desc_off, nb,
                                                ratio, d_idx + (size_t)j * n1, d_dist + (size_t)j * n1,
                                                d_keep + (size_t)j * n1, nullptr, e->buf[B_SCRATCH],
                                                nsplit, st);
            CK(cudaGetLastError());
        }
        PhaseClock clk;
        std::vector<int32_t> idx(per);
        std::vector<float> dist(per);
        std::vector<uint8_t> keep(per);
        CK(cudaMemcpyAsync(idx.data(), d_idx, 4 * per, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(dist.data(), d_dist, 4 * per, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(keep.data(), d_keep, per, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        clk.lap(st, "match+d2h");
        Repeats rep(merged);
        std::vector<xa_correspondence> fresh;
        for (int i = 0; i < n; ++i) {
            const SimView& a = v1[i];
            for (int j = 0; j < n; ++j) {
                const SimView& b = v2[j];
                if (a.kps.empty() || b.kps.empty()) continue;
                fresh.clear();
                const size_t base = (size_t)j * n1 + a.desc_off;
                for (size_t q = 0; q < a.kps.size(); ++q) {
                    if (!keep[base + q]) continue;
                    const xa_keypoint& ka = a.kps[q];
                    const xa_keypoint& kb = b.kps[idx[base + q]];
                    xa_correspondence c;
                    map_pt_h(a.back, ka.x, ka.y, c.x1, c.y1);
                    map_pt_h(b.back, kb.x, kb.y, c.x2, c.y2);
                    c.distance = dist[base + q];
                    if (!rep.seen(c)) fresh.push_back(c);
                }
                for (const auto& c : fresh) {
                    merged.push_back(c);
                    rep.add((int)merged.size() - 1);
                }
            }
        }
        clk.lap(st, "merge");
    }
    *n_out = (int)merged.size();
    if ((int)merged.size() > cap) return set_err(XA_ECAPACITY, "asift: output capacity");
    if (!merged.empty()) std::memcpy(out, merged.data(), sizeof(xa_correspondence) * merged.size());
    return XA_OK;
}

}  // extern "C"
