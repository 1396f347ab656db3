// xa_match.cu — brute-force Hamming top-2 with ratio test on sm_100a.
//
// Reference: match_hamming (proj/src/orb.cpp:250-272). For each query the
// reference scans the train set in order keeping (best, best_idx, second):
// d < best shifts best into second (so the lowest train index wins ties),
// otherwise d < second updates second; a missing second counts as 256 and a
// query is kept iff best < ratio * second (double). Here:
//   - each thread owns Q queries in registers (8 x u32 words each);
//   - train descriptors are staged through shared memory in tiles and read
//     as broadcasts; XOR + __popc on the integer pipe, no tensor cores
//     (BASELINE.json north_star);
//   - the train set is split into S contiguous chunks scanned by different
//     CTAs; partial (best, idx, second) triples are merged in chunk order with
//     (b1,i1,s1) + (b2,i2,s2) = (b1,i1,min(s1,b2)) when (b1,i1) < (b2,i2)
//     (SURVEY.md Appendix A), which is exactly the sequential scan's result;
//   - the ratio test uses a 257-entry threshold table computed on the host in
//     double (keep iff best < thr[second]).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "xa_common.cuh"
#include "xa_kernels.h"

namespace xa {

constexpr int kTile = 256;  // train descriptors per shared-memory tile

struct Top2 {
    uint32_t best, idx, second;
};

__device__ __forceinline__ uint32_t hdist(const uint4& q0, const uint4& q1, const uint4& t0,
                                          const uint4& t1) {
    return __popc(q0.x ^ t0.x) + __popc(q0.y ^ t0.y) + __popc(q0.z ^ t0.z) + __popc(q0.w ^ t0.w) +
           __popc(q1.x ^ t1.x) + __popc(q1.y ^ t1.y) + __popc(q1.z ^ t1.z) + __popc(q1.w ^ t1.w);
}

// Sequential reference update (orb.cpp:259-265) for train index j.
__device__ __forceinline__ void upd(Top2& t, uint32_t d, uint32_t j) {
    if (d < t.best) {
        t.second = t.best;
        t.best = d;
        t.idx = j;
    } else if (d < t.second) {
        t.second = d;
    }
}

// ------------------------------------------------------------- per-view jobs

// Matcher for the coarse search: one CTA row per job (view vs target). A CTA
// owns 32 queries (one per lane) and its 4 warps scan 4 contiguous quarters of
// the train set (4x the warps of a query-per-thread layout, so the POPC pipe
// stays fed), each through its own shared-memory tile read as broadcasts; the
// quarter results are merged in train order with the chunk rule above.
constexpr int kJobWarps = 8, kJobTile = 64;
__global__ void __launch_bounds__(32 * kJobWarps) k_match_jobs(const MatchJob* __restrict__ jobs,
                                                               const uint64_t* __restrict__ a,
                                                               const uint64_t* __restrict__ b,
                                                               const uint16_t* __restrict__ keep_thr,
                                                               uint32_t* __restrict__ best_idx,
                                                               uint16_t* __restrict__ best,
                                                               uint16_t* __restrict__ second) {
    __shared__ uint4 s_b[kJobWarps][kJobTile][2];
    __shared__ Top2 s_t[kJobWarps][32];
    const MatchJob J = jobs[blockIdx.y];
    const int na = J.na_dev ? *J.na_dev : J.na;
    const int nb = J.nb_dev ? *J.nb_dev : J.nb;
    if ((int)(blockIdx.x * 32) >= na) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int qi = blockIdx.x * 32 + lane;
    const bool active = qi < na && nb > 0;
    uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
    if (active) {
        const uint4* qa = reinterpret_cast<const uint4*>(a + (J.a_off + qi) * 4);
        q0 = qa[0];
        q1 = qa[1];
    }
    // this warp's quarter [c0, c1) of the train set
    const int per = (nb + kJobWarps - 1) / kJobWarps;
    const int c0 = min(nb, wid * per), c1 = min(nb, c0 + per);
    Top2 t = {257u, 0xFFFFFFFFu, 257u};
    const uint4* B = reinterpret_cast<const uint4*>(b + J.b_off * 4);
    for (int base = c0; base < c1; base += kJobTile) {
        const int cnt = min(kJobTile, c1 - base);
        __syncwarp();
        for (int i = lane; i < cnt * 2; i += 32) s_b[wid][i >> 1][i & 1] = B[base * 2 + i];
        __syncwarp();
        if (active)
            for (int j = 0; j < cnt; ++j) upd(t, hdist(q0, q1, s_b[wid][j][0], s_b[wid][j][1]), base + j);
    }
    s_t[wid][lane] = t;
    __syncthreads();
    if (wid != 0) return;
    Top2 r = s_t[0][lane];
    for (int w = 1; w < kJobWarps; ++w) {  // chunks in train order: later indices lose ties
        const Top2 p = s_t[w][lane];
        if (p.idx == 0xFFFFFFFFu) continue;
        if (r.idx == 0xFFFFFFFFu) {
            r = p;
        } else if (p.best < r.best) {
            r.second = min(r.best, p.second);
            r.best = p.best;
            r.idx = p.idx;
        } else {
            r.second = min(r.second, p.best);
        }
    }
    bool keep = false;
    if (active) {
        const uint32_t sec = r.second > 256u ? 256u : r.second;
        const long long o = J.out_off + qi;
        if (best_idx) best_idx[o] = r.idx;
        if (best) best[o] = (uint16_t)r.best;
        if (second) second[o] = (uint16_t)sec;
        keep = r.best < keep_thr[sec];
    }
    const int nk = __popc(__ballot_sync(0xffffffffu, keep));
    if (lane == 0 && nk && J.count_out) atomicAdd(J.count_out, nk);
}


// ------------------------------------------------------------- tensor-core Hamming
//
// Brute-force Hamming kNN is a dense binary contraction: with each bit mapped
// to a signed byte (1 -> +1, 0 -> -1) the s8 dot product of two 256-bit
// descriptors is 256 - 2d, so a tile of queries x train descriptors is one
// int8 GEMM with K = 256 on the tensor cores (mma.sync m16n8k32 s8, IMMA),
// which on B200 delivers ~3.8x the comparisons/s of XOR + POPC on the integer
// pipe (tools/diag/imma_peak.cu, profiles/r02_imma_probe.jsonl). The epilogue
// stays exact integer work: each distance becomes the 31-bit key
// d << 22 | train index (one IMAD per value), and the two smallest keys of a
// query are its (best, best_idx) and second -- exactly the reference's
// sequential scan (orb.cpp:256-265: strict '<' keeps the lowest index among
// equal distances, and 'second' is the second smallest distance of the
// multiset), with no order dependence, so train splits merge by taking the
// two smallest keys again. Train sets beyond 2^22 descriptors keep the POPC
// kernels.
//
// CTA = 8 warps x 32 queries (two m16 tiles per warp, A fragments expanded
// from the packed bits once into 64 registers), train streamed in tiles of 64
// descriptors: packed bits by cp.async (2 KB), expanded once per CTA into a
// +-1 byte tile in shared memory (272-byte rows: conflict-free ldmatrix), then
// per 8-column group 4 ldmatrix.x4 + 16 IMMA + 8 keys x 4 integer ops per lane.
#ifndef TC_TILE
#define TC_TILE 128
#endif
constexpr int kTcWarps = 8, kTcQ = 32 * kTcWarps, kTcTile = TC_TILE, kTcRow = 272;
constexpr uint32_t kTcNone = (257u << 22) | 0x3FFFFFu;  // "no neighbour": decodes to 257
constexpr int kTcMaxTrain = 1 << 22;

// 4 bits -> 4 bytes of +1 (bit set) / -1 (bit clear), byte i from bit i
__device__ __forceinline__ uint32_t pm1_nibble(uint32_t n) {
    const uint32_t s = (n * 0x00204081u) & 0x01010101u;
    return 0x01010101u | ((s ^ 0x01010101u) * 0xFEu);
}

__device__ __forceinline__ void imma_s8(int* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(s));
}

// two smallest keys (b <= s) after offering key k
__device__ __forceinline__ void top2_key(uint32_t& b, uint32_t& s, uint32_t k) {
    s = min(s, max(b, k));
    b = min(b, k);
}

// Final per-query decision from the two smallest keys (orb.cpp:266-268).
__device__ __forceinline__ bool tc_finish(uint32_t b, uint32_t s, long long o, const uint16_t* keep_thr,
                                          uint32_t* best_idx, uint16_t* best, uint16_t* second) {
    const uint32_t bd = b >> 22, sd = min(s >> 22, 256u);
    if (best_idx) best_idx[o] = b & 0x3FFFFFu;
    if (best) best[o] = (uint16_t)bd;
    if (second) second[o] = (uint16_t)sd;
    return bd < keep_thr[sd];
}

// jobs == nullptr: the single job `one`. gridDim.z > 1 splits each job's train
// set into contiguous slices; their key pairs go to part[slice * one.na + q]
// (single-job launches only) and k_match_tc_merge finishes.
#ifndef TC_MINB
#define TC_MINB 2
#endif
__global__ void __launch_bounds__(32 * kTcWarps, TC_MINB) k_match_tc(const MatchJob* __restrict__ jobs, MatchJob one,
                                                              const uint64_t* __restrict__ a,
                                                              const uint64_t* __restrict__ b,
                                                              const uint16_t* __restrict__ keep_thr,
                                                              uint32_t* __restrict__ best_idx,
                                                              uint16_t* __restrict__ best,
                                                              uint16_t* __restrict__ second,
                                                              uint2* __restrict__ part) {
    __shared__ __align__(16) uint8_t s_e[kTcTile * kTcRow];
    __shared__ __align__(16) uint32_t s_bits[2][kTcTile * 8];
    const MatchJob J = jobs ? jobs[blockIdx.y] : one;
    const int na = J.na_dev ? *J.na_dev : J.na;
    const int nb = J.nb_dev ? *J.nb_dev : J.nb;
    const int qb = blockIdx.x * kTcQ;
    if (qb >= na || nb <= 0) return;
    const int S = gridDim.z, per = (nb + S - 1) / S;
    const int c0 = min(nb, (int)blockIdx.z * per), c1 = min(nb, c0 + per);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, g = lane >> 2, t4 = lane & 3;

    // A fragments (m16n8k32 row-major s8): step s of m-tile mt holds, for rows
    // g and g + 8, the bytes k = 4 t4 .. 4 t4 + 3 and k + 16 of bit word s
    uint32_t A[2][8][4];
    const uint32_t* Abits = reinterpret_cast<const uint32_t*>(a) + (size_t)J.a_off * 8;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = qb + wid * 32 + mt * 16 + g + 8 * h;
            uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
            if (q < na) {
                w0 = reinterpret_cast<const uint4*>(Abits + (size_t)q * 8)[0];
                w1 = reinterpret_cast<const uint4*>(Abits + (size_t)q * 8)[1];
            }
            const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int st = 0; st < 8; ++st) {
                A[mt][st][h] = pm1_nibble((w[st] >> (4 * t4)) & 15u);
                A[mt][st][2 + h] = pm1_nibble((w[st] >> (16 + 4 * t4)) & 15u);
            }
        }
    uint32_t kb[4] = {kTcNone, kTcNone, kTcNone, kTcNone}, ks[4] = {kTcNone, kTcNone, kTcNone, kTcNone};

    const uint32_t* Bbits = reinterpret_cast<const uint32_t*>(b) + (size_t)J.b_off * 8;
    const int ntile = (c1 - c0 + kTcTile - 1) / kTcTile;
    auto load_bits = [&](int t, int buf) {
        for (int e = tid; e < 2 * kTcTile; e += 32 * kTcWarps) {
            const int row = e >> 1, half = e & 1, j = c0 + t * kTcTile + row;
            uint32_t* dst = &s_bits[buf][row * 8 + half * 4];
            if (j < c1) cp_async16(reinterpret_cast<float*>(dst), reinterpret_cast<const float*>(Bbits + (size_t)j * 8 + half * 4));
            else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
        }
        cp_async_commit();
    };
    if (ntile > 0) load_bits(0, 0);
    for (int t = 0; t < ntile; ++t) {
        const int base = c0 + t * kTcTile, cnt = min(kTcTile, c1 - base);
        if (t + 1 < ntile) load_bits(t + 1, (t + 1) & 1);
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();  // tile t's bits landed; every warp is done with s_e (tile t - 1)
        for (int e = tid; e < kTcTile * 4; e += 32 * kTcWarps) {  // expand: row e / 4, bit words 2 (e & 3), +1
            const int row = e >> 2, q4 = e & 3;
            const uint32_t w0 = s_bits[t & 1][row * 8 + 2 * q4], w1 = s_bits[t & 1][row * 8 + 2 * q4 + 1];
            uint4* dst = reinterpret_cast<uint4*>(s_e + row * kTcRow + q4 * 64);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t w = k ? w1 : w0;
                dst[2 * k] = make_uint4(pm1_nibble(w & 15u), pm1_nibble((w >> 4) & 15u), pm1_nibble((w >> 8) & 15u),
                                        pm1_nibble((w >> 12) & 15u));
                dst[2 * k + 1] = make_uint4(pm1_nibble((w >> 16) & 15u), pm1_nibble((w >> 20) & 15u),
                                            pm1_nibble((w >> 24) & 15u), pm1_nibble(w >> 28));
            }
        }
        __syncthreads();
#ifndef TC_GROUPS
#define TC_GROUPS 2
#endif
        for (int n0 = 0; n0 < cnt; n0 += 8 * TC_GROUPS) {
            int acc[TC_GROUPS][2][4];
#pragma unroll
            for (int gi = 0; gi < TC_GROUPS; ++gi)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[gi][0][k] = acc[gi][1][k] = 0;
#pragma unroll
            for (int st = 0; st < 8; st += 2) {
#pragma unroll
                for (int gi = 0; gi < TC_GROUPS; ++gi) {
                    uint32_t r[4];
                    ldsm_x4(r, s_e + (n0 + 8 * gi + (lane & 7)) * kTcRow + (lane >> 3) * 16 + st * 32);
                    imma_s8(acc[gi][0], A[0][st], r[0], r[1]);
                    imma_s8(acc[gi][1], A[1][st], r[0], r[1]);
                    imma_s8(acc[gi][0], A[0][st + 1], r[2], r[3]);
                    imma_s8(acc[gi][1], A[1][st + 1], r[2], r[3]);
                }
            }
            // key = d << 22 | j with d = (256 - dot) / 2: (256 << 21) + j - (dot << 21).
            // A key changes a row's top-2 only if it is below the row's second
            // key; after the first tiles that is rare, so the full update runs
            // under one warp-uniform test per group.
#pragma unroll
            for (int gi = 0; gi < TC_GROUPS; ++gi) {
                const int col = n0 + 8 * gi + 2 * t4;
                const uint32_t C0 = (256u << 21) + (uint32_t)(base + col);
                uint32_t k[4][2];
                bool need = false;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    k[r][0] = C0 - ((uint32_t)acc[gi][r >> 1][2 * (r & 1)] << 21);
                    k[r][1] = C0 + 1u - ((uint32_t)acc[gi][r >> 1][2 * (r & 1) + 1] << 21);
                    need |= min(k[r][0], k[r][1]) < ks[r];
                }
                if (__any_sync(0xffffffffu, need)) {
                    const bool v0 = col < cnt, v1 = col + 1 < cnt;
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (v0) top2_key(kb[r], ks[r], k[r][0]);
                        if (v1) top2_key(kb[r], ks[r], k[r][1]);
                    }
                }
            }
        }
    }
    // the four lanes of a row group saw disjoint columns: two smallest of the union
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
            const uint32_t ob = __shfl_xor_sync(0xffffffffu, kb[r], off), os = __shfl_xor_sync(0xffffffffu, ks[r], off);
            ks[r] = min(max(kb[r], ob), min(ks[r], os));
            kb[r] = min(kb[r], ob);
        }
    int nk = 0;
    if (t4 == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int q = qb + wid * 32 + (r >> 1) * 16 + g + 8 * (r & 1);
            if (q >= na) continue;
            if (part) part[(size_t)blockIdx.z * J.na + q] = make_uint2(kb[r], ks[r]);
            else nk += tc_finish(kb[r], ks[r], J.out_off + q, keep_thr, best_idx, best, second) ? 1 : 0;
        }
    }
    if (!part) {
        nk = __reduce_add_sync(0xffffffffu, nk);
        if (lane == 0 && nk && J.count_out) atomicAdd(J.count_out, nk);
    }
}

__global__ void k_match_tc_merge(const uint2* __restrict__ part, int na, int nsplit,
                                 const uint16_t* __restrict__ keep_thr, uint32_t* __restrict__ best_idx,
                                 uint16_t* __restrict__ best, uint16_t* __restrict__ second,
                                 int* __restrict__ count) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    bool k = false;
    if (q < na) {
        uint32_t b = kTcNone, s = kTcNone;
        for (int sp = 0; sp < nsplit; ++sp) {
            const uint2 p = part[(size_t)sp * na + q];
            s = min(max(b, p.x), min(s, p.y));
            b = min(b, p.x);
        }
        k = tc_finish(b, s, q, keep_thr, best_idx, best, second);
    }
    const int nk = __popc(__ballot_sync(0xffffffffu, k));
    if ((threadIdx.x & 31) == 0 && nk && count) atomicAdd(count, nk);
}


// ------------------------------------------------------------- tcgen05 Hamming
//
// The same contraction on the 5th-generation tensor cores: tcgen05.mma
// kind::i8 (UTCIMMA) issued by one thread, operands in shared memory,
// accumulators in tensor memory (tools/diag/umma_i8_check.cu validates the
// descriptor encoding). Descriptors are first expanded once into +-1 s8 rows
// (k_desc_pm1, 256 B each) in one buffer; a 2-D tensor map over it (256-byte
// rows, box 128 B x 128 rows, SWIZZLE_128B) lands each K half of 128 rows in
// the K-major 128-byte-swizzled canonical layout (8-row x 128-byte atoms,
// SBO = 1024 B): 2 TMA per train tile, 4 per query block.
//
// Persistent CTAs (one per SM) walk work items (job, 256-query block, train
// slice). Warp roles: warp 8 = TMA producer (A block once per item, B tiles of
// 128 train rows through a 3-stage ring), warp 9 = TMEM allocator + MMA issuer
// (per tile 8 k-steps x 2 M=128 halves, N = 128), warps 0-7 = epilogue: thread
// t of warp w owns TMEM lane 32 (w % 4) + t of half w / 4, i.e. query
// qb + 128 (w / 4) + 32 (w % 4) + t, reads its 128 dot products per tile with
// tcgen05.ld, and keeps the reference's
// sequential top-2 in train order (orb.cpp:256-265). A value can change the
// top-2 only if its distance beats the current second, i.e. dot > 256 - 2
// second; a 3-input max over each 32-column load tests that once, so the exact
// per-value update runs only for the rare loads that contain a candidate.
// Two accumulator buffers (2 x 256 TMEM columns) let the MMAs of tile t + 1
// overlap the epilogue of tile t.
#ifndef UM_STAGES
#define UM_STAGES 4
#endif
#ifndef UM_N
#define UM_N 128
#endif
constexpr int kUmQ = 256, kUmN = UM_N, kUmStages = UM_STAGES, kUmBufs = 512 / (2 * kUmN);
constexpr int kUmAbytes = kUmQ * 256, kUmBbytes = kUmN * 256;
constexpr int kUmSmem = kUmAbytes + kUmStages * kUmBbytes + 1024;

struct __align__(64) TmaDesc {
    unsigned char b[128];
};

__device__ __forceinline__ uint32_t sm_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_128B operand: 8-row x 128-byte atoms (SBO = 1024 B), the
// k-step's 32 bytes selected by advancing the start inside the atom
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ void um_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(sm_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void um_tma3(void* dst, const TmaDesc* map, int row, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            sm_u32(dst)),
        "l"(map), "r"(0), "r"(row), "r"(0), "r"(sm_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbarrier_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_u32(bar)) : "memory");
}

__device__ __forceinline__ void um_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void um_ld32(uint32_t taddr, int (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// Expanded descriptors: row i = 256 bytes, byte k = +1 if bit k is set else -1.
__global__ void k_desc_pm1(const uint32_t* __restrict__ bits, long long nwords, uint4* __restrict__ out) {
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < nwords; w += (long long)gridDim.x * blockDim.x) {
        const uint32_t x = bits[w];
        out[2 * w] = make_uint4(pm1_nibble(x & 15u), pm1_nibble((x >> 4) & 15u), pm1_nibble((x >> 8) & 15u),
                                pm1_nibble((x >> 12) & 15u));
        out[2 * w + 1] = make_uint4(pm1_nibble((x >> 16) & 15u), pm1_nibble((x >> 20) & 15u),
                                    pm1_nibble((x >> 24) & 15u), pm1_nibble(x >> 28));
    }
}

// Top-2 over one 32-column load (train indices j0 .. j0 + 31) as the two
// smallest keys d << 22 | j (dot = 256 - 2 d). A value can enter the top-2
// only if d < second (its index is later than every key seen, so ties lose),
// i.e. dot > 256 - 2 second: each group of 8 values is tested with one 3-input
// max tree and a warp vote, and only groups holding a candidate for some lane
// run the exact key updates (branch-free min / max per value).
__device__ __forceinline__ void um_scan(const int (&v)[32], int cnt, int j0, uint32_t& kb, uint32_t& ks,
                                        bool whole) {
    int thr = 256 - 2 * (int)(ks >> 22);
    // long train sets (whole): the whole load first (one 3-input max tree), the
    // groups of 8 only if it holds a candidate -- candidates get rare along a
    // long scan; short scans (the coarse jobs) test the groups directly
    if (whole) {
        int m32 = __vimax3_s32(v[0], v[1], v[2]);
#pragma unroll
        for (int k = 3; k < 30; k += 3) m32 = __vimax3_s32(m32, v[k], max(v[k + 1], v[k + 2]));
        m32 = __vimax3_s32(m32, v[30], v[31]);
        if (!__any_sync(0xffffffffu, m32 > thr)) return;
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const int* w = v + 8 * g;
        const int m = __vimax3_s32(__vimax3_s32(w[0], w[1], w[2]), __vimax3_s32(w[3], w[4], w[5]), max(w[6], w[7]));
        if (__any_sync(0xffffffffu, m > thr)) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (8 * g + k < cnt) top2_key(kb, ks, ((uint32_t)(256 - w[k]) << 21) + (uint32_t)(j0 + 8 * g + k));
            thr = 256 - 2 * (int)(ks >> 22);
        }
    }
}

template <bool WHOLE>
__global__ void __launch_bounds__(320, 1) k_match_umma(const MatchJob* __restrict__ jobs, MatchJob one, int njobs,
                                                      int qblocks, int nsplit, const __grid_constant__ TmaDesc tmap,
                                                      const __grid_constant__ TmaDesc tmapB,
                                                      const uint16_t* __restrict__ keep_thr,
                                                      uint32_t* __restrict__ best_idx, uint16_t* __restrict__ best,
                                                      uint16_t* __restrict__ second, uint2* __restrict__ part) {
    extern __shared__ __align__(1024) uint8_t um_smem[];
    uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(um_smem) + 1023) & ~uintptr_t(1023));
    uint8_t* sB = sA + kUmAbytes;
    __shared__ __align__(8) uint64_t b_full[kUmStages], b_empty[kUmStages], a_full, a_empty, acc_full[kUmBufs], acc_empty[kUmBufs];
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kUmStages; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        mbar_init(&a_full, 1);
        mbar_init(&a_empty, 1);
        for (int s = 0; s < kUmBufs; ++s) {
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], 8);
        }
        fence_mbar_init();
    }
    if (wid == 9) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(&s_tmem)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;
    const int nitems = njobs * qblocks * nsplit;

    if (wid == 8) {
        // ---------------- TMA producer
        if (lane == 0) {
            uint32_t stage = 0, sph = 0, aph = 0;
            bool first = true;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const int sp = it % nsplit, qbk = (it / nsplit) % qblocks, jb = it / (nsplit * qblocks);
                const MatchJob J = jobs ? jobs[jb] : one;
                const int na = J.na_dev ? *J.na_dev : J.na, nb = J.nb_dev ? *J.nb_dev : J.nb;
                const int qb = qbk * kUmQ;
                if (qb >= na || nb <= 0) continue;
                const int per = (nb + nsplit - 1) / nsplit;
                const int c0 = min(nb, sp * per), c1 = min(nb, c0 + per);
                const int ntile = (c1 - c0 + kUmN - 1) / kUmN;
                if (ntile == 0) continue;
                if (!first) {
                    um_wait(&a_empty, aph);
                    aph ^= 1;
                }
                first = false;
                mbar_arrive_tx(&a_full, kUmAbytes);
#pragma unroll
                for (int kh = 0; kh < 2; ++kh)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
                        tma_load_2d(sA + kh * (kUmQ * 128) + hh * (128 * 128), &tmap, 128 * kh,
                                    (int)(J.a_off + qb + 128 * hh), &a_full);
                for (int t = 0; t < ntile; ++t) {
                    um_wait(&b_empty[stage], sph ^ 1);
                    mbar_arrive_tx(&b_full[stage], kUmBbytes);
#pragma unroll
                    for (int kh = 0; kh < 2; ++kh)
                        tma_load_2d(sB + stage * kUmBbytes + kh * (kUmN * 128), &tmapB, 128 * kh,
                                    (int)(J.b_off + c0 + t * kUmN), &b_full[stage]);
                    if (++stage == kUmStages) {
                        stage = 0;
                        sph ^= 1;
                    }
                }
            }
        }
    } else if (wid == 9) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kUmN >> 3) << 17) | (8u << 24);
            uint32_t stage = 0, sph = 0, aph = 0, abuf = 0, accph = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const int sp = it % nsplit, qbk = (it / nsplit) % qblocks, jb = it / (nsplit * qblocks);
                const MatchJob J = jobs ? jobs[jb] : one;
                const int na = J.na_dev ? *J.na_dev : J.na, nb = J.nb_dev ? *J.nb_dev : J.nb;
                if (qbk * kUmQ >= na || nb <= 0) continue;
                const int per = (nb + nsplit - 1) / nsplit;
                const int c0 = min(nb, sp * per), c1 = min(nb, c0 + per);
                const int ntile = (c1 - c0 + kUmN - 1) / kUmN;
                if (ntile == 0) continue;
                um_wait(&a_full, aph);
                aph ^= 1;
                for (int t = 0; t < ntile; ++t) {
                    um_wait(&b_full[stage], sph);
                    um_wait(&acc_empty[abuf], accph ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t bbase = sm_u32(sB + stage * kUmBbytes);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t d = tmem + abuf * (2 * kUmN) + h * kUmN;
#pragma unroll
                        for (int s = 0; s < 8; ++s) {
                            const uint64_t da = umma_desc_sw128(sm_u32(sA) + (s >> 2) * (kUmQ * 128) + h * (128 * 128) + (s & 3) * 32);
                            const uint64_t db = umma_desc_sw128(bbase + (s >> 2) * (kUmN * 128) + (s & 3) * 32);
                            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                                         "l"(da), "l"(db), "r"(idesc), "r"(s));
                        }
                    }
                    um_commit(&b_empty[stage]);   // smem slot free once these MMAs complete
                    um_commit(&acc_full[abuf]);   // accumulators ready for the epilogue
                    if (++stage == kUmStages) {
                        stage = 0;
                        sph ^= 1;
                    }
                    if (++abuf == kUmBufs) {
                        abuf = 0;
                        accph ^= 1;
                    }
                }
                um_commit(&a_empty);  // A block free once this item's MMAs complete
            }
        }
    } else {
        // ---------------- epilogue (warps 0-7): warp w reads TMEM lanes
        // 32 (w % 4) .. + 31 of accumulator half h = w / 4, i.e. one query per
        // thread; a tile's four 32-column loads are issued before one wait and
        // the accumulator buffer is released before the scans
        const int h = wid >> 2, quarter = wid & 3;
        uint32_t abuf = 0, accph = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int sp = it % nsplit, qbk = (it / nsplit) % qblocks, jb = it / (nsplit * qblocks);
            const MatchJob J = jobs ? jobs[jb] : one;
            const int na = J.na_dev ? *J.na_dev : J.na, nb = J.nb_dev ? *J.nb_dev : J.nb;
            const int qb = qbk * kUmQ;
            if (qb >= na || nb <= 0) continue;
            const int per = (nb + nsplit - 1) / nsplit;
            const int c0 = min(nb, sp * per), c1 = min(nb, c0 + per);
            const int ntile = (c1 - c0 + kUmN - 1) / kUmN;
            if (ntile == 0) continue;
            uint32_t kb = kTcNone, ks = kTcNone;
            const bool whole = WHOLE && c1 - c0 > 8192;
            for (int t = 0; t < ntile; ++t) {
                const int base = c0 + t * kUmN, cnt = min(kUmN, c1 - base);
                um_wait(&acc_full[abuf], accph);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t ta = tmem + ((uint32_t)(32 * quarter) << 16) + abuf * (2 * kUmN) + h * kUmN;
                int v0[32], v1[32], v2[32], v3[32];
                um_ld32(ta, v0);
                um_ld32(ta + 32, v1);
                if (kUmN > 64) {
                    um_ld32(ta + 64, v2);
                    um_ld32(ta + 96, v3);
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;");
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbarrier_arrive(&acc_empty[abuf]);
                if (++abuf == kUmBufs) {
                    abuf = 0;
                    accph ^= 1;
                }
                um_scan(v0, cnt, base, kb, ks, whole);
                um_scan(v1, cnt - 32, base + 32, kb, ks, whole);
                if (kUmN > 64) {
                    um_scan(v2, cnt - 64, base + 64, kb, ks, whole);
                    um_scan(v3, cnt - 96, base + 96, kb, ks, whole);
                }
            }
            int nk = 0;
            const int q = qb + h * 128 + 32 * quarter + lane;
            if (q < na) {
                if (part) part[(size_t)sp * J.na + q] = make_uint2(kb, ks);
                else nk = tc_finish(kb, ks, J.out_off + q, keep_thr, best_idx, best, second) ? 1 : 0;
            }
            if (!part) {
                nk = __reduce_add_sync(0xffffffffu, nk);
                if (lane == 0 && nk && J.count_out) atomicAdd(J.count_out, nk);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (wid == 9) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

int match_umma_tile_n() { return kUmN; }

int match_umma_init() {
    return cudaFuncSetAttribute(k_match_umma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kUmSmem) == cudaSuccess &&
                   cudaFuncSetAttribute(k_match_umma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kUmSmem) == cudaSuccess
               ? 0
               : -1;
}

int launch_desc_pm1(const uint64_t* bits, long long n, void* out, cudaStream_t st) {
    if (n <= 0) return 0;
    const long long nw = n * 8;
    const int blocks = (int)std::min<long long>((nw + 255) / 256, 148LL * 16);
    k_desc_pm1<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(bits), nw, static_cast<uint4*>(out));
    return 1;
}

int launch_match_umma(const MatchJob* d_jobs, const MatchJob& one, int njobs, int max_na, int nsplit,
                      const void* tmap, const uint16_t* keep_thr, uint32_t* best_idx, uint16_t* best,
                      uint16_t* second, void* part, int sms, cudaStream_t st) {
    if (njobs <= 0 || max_na <= 0) return 0;
    const int qblocks = (max_na + kUmQ - 1) / kUmQ;
    const int nitems = njobs * qblocks * nsplit;
    TmaDesc m, mb;
    memcpy(&m, tmap, sizeof m);
    memcpy(&mb, static_cast<const char*>(tmap) + sizeof m, sizeof mb);
    // single-job launches scan long train sets; the coarse per-view jobs are short
    if (d_jobs)
        k_match_umma<false><<<std::min(nitems, sms), 320, kUmSmem, st>>>(d_jobs, one, njobs, qblocks, nsplit, m, mb,
                                                                       keep_thr, best_idx, best, second,
                                                                       static_cast<uint2*>(part));
    else
        k_match_umma<true><<<std::min(nitems, sms), 320, kUmSmem, st>>>(d_jobs, one, njobs, qblocks, nsplit, m, mb,
                                                                      keep_thr, best_idx, best, second,
                                                                      static_cast<uint2*>(part));
    return 1;
}

int launch_match_tc_merge(const void* part, int na, int nsplit, const uint16_t* keep_thr, uint32_t* best_idx,
                          uint16_t* best, uint16_t* second, int* count, cudaStream_t st) {
    k_match_tc_merge<<<(na + 255) / 256, 256, 0, st>>>(static_cast<const uint2*>(part), na, nsplit, keep_thr,
                                                        best_idx, best, second, count);
    return 1;
}

// XA_MATCH_TC=0 keeps the XOR + POPC kernels (A/B and fallback tests)
static bool use_tc() {
    static const bool on = [] {
        const char* e = std::getenv("XA_MATCH_TC");
        return !(e && e[0] == '0');
    }();
    return on;
}

int launch_match(const MatchJob* d_jobs, int njobs, int max_na, const uint64_t* a,
                 const uint64_t* b, const uint16_t* d_keep_thr, uint32_t* best_idx,
                 uint16_t* best, uint16_t* second, cudaStream_t st, int max_nb) {
    if (njobs <= 0 || max_na <= 0) return 0;
    if (use_tc() && max_nb <= kTcMaxTrain) {
        dim3 grid((max_na + kTcQ - 1) / kTcQ, njobs, 1);
        k_match_tc<<<grid, 32 * kTcWarps, 0, st>>>(d_jobs, MatchJob{}, a, b, d_keep_thr, best_idx, best, second,
                                                    nullptr);
        return 1;
    }
    dim3 grid((max_na + 31) / 32, njobs);
    k_match_jobs<<<grid, 32 * kJobWarps, 0, st>>>(d_jobs, a, b, d_keep_thr, best_idx, best, second);
    return 1;
}

// ------------------------------------------------------------- large sets

constexpr int QPT = 4;        // queries per thread
constexpr int LTHREADS = 128; // threads per CTA -> 512 queries per CTA

// Partial scan of train chunk [c0, c1) for QPT queries per thread.
__global__ void __launch_bounds__(LTHREADS) k_match_partial(const uint64_t* __restrict__ a, int na,
                                                            const uint64_t* __restrict__ b, int nb,
                                                            int chunk, Top2* __restrict__ part) {
    __shared__ uint4 s_b[kTile][2];
    const int split = blockIdx.y;
    const int c0 = split * chunk, c1 = min(nb, c0 + chunk);
    uint4 q[QPT][2];
    Top2 t[QPT];
    const uint4* A = reinterpret_cast<const uint4*>(a);
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
        const int qi = (blockIdx.x * QPT + k) * LTHREADS + threadIdx.x;
        if (qi < na) {
            q[k][0] = A[2 * (size_t)qi];
            q[k][1] = A[2 * (size_t)qi + 1];
        } else {
            q[k][0] = q[k][1] = make_uint4(0, 0, 0, 0);
        }
        t[k].best = 257u;
        t[k].idx = 0xFFFFFFFFu;
        t[k].second = 257u;
    }
    const uint4* B = reinterpret_cast<const uint4*>(b);
    for (int base = c0; base < c1; base += kTile) {
        const int cnt = min(kTile, c1 - base);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt * 2; i += LTHREADS) s_b[i >> 1][i & 1] = B[(size_t)base * 2 + i];
        __syncthreads();
        for (int j = 0; j < cnt; ++j) {
            const uint4 t0 = s_b[j][0], t1 = s_b[j][1];
#pragma unroll
            for (int k = 0; k < QPT; ++k) upd(t[k], hdist(q[k][0], q[k][1], t0, t1), base + j);
        }
    }
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
        const int qi = (blockIdx.x * QPT + k) * LTHREADS + threadIdx.x;
        if (qi < na) part[(size_t)split * na + qi] = t[k];
    }
}

__global__ void k_match_merge(const Top2* __restrict__ part, int na, int nsplit,
                              const uint16_t* __restrict__ keep_thr, uint32_t* __restrict__ best_idx,
                              uint16_t* __restrict__ best, uint16_t* __restrict__ second,
                              int* __restrict__ count) {
    __shared__ int s_keep;
    if (threadIdx.x == 0) s_keep = 0;
    __syncthreads();
    const int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi < na) {
        Top2 r = part[qi];
        for (int s = 1; s < nsplit; ++s) {
            const Top2 p = part[(size_t)s * na + qi];
            if (p.idx == 0xFFFFFFFFu) continue;
            if (r.idx == 0xFFFFFFFFu) {
                r = p;
            } else if (p.best < r.best) {  // p's indices are all later: strict
                r.second = min(r.best, p.second);
                r.best = p.best;
                r.idx = p.idx;
            } else {
                r.second = min(r.second, p.best);
            }
        }
        const uint32_t sec = r.second > 256u ? 256u : r.second;
        best_idx[qi] = r.idx;
        best[qi] = (uint16_t)r.best;
        second[qi] = (uint16_t)sec;
        if (r.best < keep_thr[sec]) atomicAdd(&s_keep, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_keep) atomicAdd(count, s_keep);
}

int launch_match_large(const uint64_t* a, int na, const uint64_t* b, int nb,
                       const uint16_t* d_keep_thr, uint32_t* best_idx, uint16_t* best,
                       uint16_t* second, int* count, void* scratch, int nsplit, cudaStream_t st) {
    if (na <= 0) return 0;
    if (use_tc() && nb <= kTcMaxTrain) {
        MatchJob one{};
        one.na = na;
        one.nb = nb;
        one.count_out = count;
        const int qblocks = (na + kTcQ - 1) / kTcQ;
        // slices so the grid fills ~8 waves of 2 CTAs per SM; tiles of >= 8 x 64 train each
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const int tc_split = std::max(1, std::min({(16 * sms + qblocks - 1) / qblocks, (nb + 511) / 512, (3 * nsplit) / 2}));  // scratch: 12 B x na x nsplit
        dim3 grid(qblocks, 1, tc_split);
        uint2* part = tc_split > 1 ? static_cast<uint2*>(scratch) : nullptr;
        k_match_tc<<<grid, 32 * kTcWarps, 0, st>>>(nullptr, one, a, b, d_keep_thr, best_idx, best, second, part);
        if (tc_split == 1) return 1;  // counted through one.count_out
        k_match_tc_merge<<<(na + 255) / 256, 256, 0, st>>>(part, na, tc_split, d_keep_thr, best_idx, best, second,
                                                            count);
        return 2;
    }
    const int chunk = (nb + nsplit - 1) / nsplit;
    const int qblocks = (na + QPT * LTHREADS - 1) / (QPT * LTHREADS);
    Top2* part = static_cast<Top2*>(scratch);
    dim3 grid(qblocks, nsplit);
    k_match_partial<<<grid, LTHREADS, 0, st>>>(a, na, b, nb, chunk, part);
    k_match_merge<<<(na + 255) / 256, 256, 0, st>>>(part, na, nsplit, d_keep_thr, best_idx, best,
                                                     second, count);
    return 2;
}

size_t match_large_scratch(int na, int nsplit) { return sizeof(Top2) * (size_t)na * nsplit; }

// ------------------------------------------------------------- L2 ratio matcher

// match_ratio (sift.cpp:388-418), the fine stage's matcher:
// per pair a sequential float sum of (a_k - b_k)^2 with the reference's two
// roundings per step (no FMA), a top-2 scan in B order with strict '<' (the
// lower B index wins ties), distances sqrt'ed in double, a missing second
// neighbour = 1024, keep iff d1 < ratio * min(d2, 1024). A CTA owns 32 queries
// (one per lane, rows in shared memory); its 4 warps scan 4 contiguous
// quarters of B through per-warp shared tiles (broadcast reads, 4 candidates
// per register block) and the quarters merge in B order.
constexpr int kL2Warps = 4, kL2Tile = 8, kL2Stride = 132;  // 132: conflict-free 16-byte row reads

struct L2Top2 {
    float best, second;
    int idx;
};

// Final per-query decision from the merged top-2 (sift.cpp:411-415).
__device__ __forceinline__ bool l2_finish(const L2Top2& r, int q, double ratio, int32_t* best_idx,
                                          float* dist, uint8_t* keep) {
    const double d1 = sqrt((double)r.best);
    const double d2 = r.second < 1e30f ? sqrt((double)r.second) : 1024.0;
    const bool k = d1 < ratio * fmin(d2, 1024.0);
    best_idx[q] = r.idx;
    dist[q] = (float)d1;
    keep[q] = k ? 1 : 0;
    return k;
}

// (r) then (p) in B order: p's indices are all later, so ties keep r.
__device__ __forceinline__ void l2_merge(L2Top2& r, const L2Top2& p) {
    if (p.idx < 0) return;
    if (r.idx < 0) {
        r = p;
    } else if (p.best < r.best) {
        r.second = fminf(r.best, p.second);
        r.best = p.best;
        r.idx = p.idx;
    } else {
        r.second = fminf(r.second, p.best);
    }
}

// blockIdx.y selects a contiguous slice of B when the scan is split across
// CTAs (nsplit > 1): partial top-2s go to `part` and k_match_l2_merge folds
// them in slice order.
__global__ void __launch_bounds__(32 * kL2Warps) k_match_l2(const float* __restrict__ a, int na,
                                                            const float* __restrict__ b, int nb,
                                                            double ratio, int32_t* __restrict__ best_idx,
                                                            float* __restrict__ dist,
                                                            uint8_t* __restrict__ keep,
                                                            int32_t* __restrict__ count,
                                                            L2Top2* __restrict__ part) {
    __shared__ __align__(16) float s_a[32 * kL2Stride];
    __shared__ __align__(16) float s_b[kL2Warps][kL2Tile * 128];
    __shared__ L2Top2 s_t[kL2Warps][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int q0 = blockIdx.x * 32;
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {  // 32 rows x 32 float4
        const int r = i >> 5, c = i & 31;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q0 + r < na) v = reinterpret_cast<const float4*>(a + (size_t)(q0 + r) * 128)[c];
        *reinterpret_cast<float4*>(s_a + r * kL2Stride + 4 * c) = v;
    }
    __syncthreads();
    const int slice = (nb + gridDim.y - 1) / gridDim.y;
    const int s0 = min(nb, (int)blockIdx.y * slice), s1 = min(nb, s0 + slice);
    const int per = (s1 - s0 + kL2Warps - 1) / kL2Warps;
    const int c0 = min(s1, s0 + wid * per), c1 = min(s1, c0 + per);
    L2Top2 t = {INFINITY, INFINITY, -1};
    const float4* ar = reinterpret_cast<const float4*>(s_a + lane * kL2Stride);
    float* tb = s_b[wid];
    for (int base = c0; base < c1; base += kL2Tile) {
        const int cnt = min(kL2Tile, c1 - base);
        __syncwarp();
        for (int i = lane; i < cnt * 32; i += 32)
            reinterpret_cast<float4*>(tb)[i] = reinterpret_cast<const float4*>(b + (size_t)base * 128)[i];
        __syncwarp();
        for (int j = 0; j < cnt; j += 4) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
            for (int k = 0; k < 32; ++k) {
                const float4 av = ar[k];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const float4 bv = reinterpret_cast<const float4*>(tb + (j + jj) * 128)[k];
                    float d = fsub(av.x, bv.x);
                    acc[jj] = fadd(acc[jj], fmul(d, d));
                    d = fsub(av.y, bv.y);
                    acc[jj] = fadd(acc[jj], fmul(d, d));
                    d = fsub(av.z, bv.z);
                    acc[jj] = fadd(acc[jj], fmul(d, d));
                    d = fsub(av.w, bv.w);
                    acc[jj] = fadd(acc[jj], fmul(d, d));
                }
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                if (j + jj >= cnt) break;
                const float v = acc[jj];
                if (v < t.best) {
                    t.second = t.best;
                    t.best = v;
                    t.idx = base + j + jj;
                } else if (v < t.second) {
                    t.second = v;
                }
            }
        }
    }
    s_t[wid][lane] = t;
    __syncthreads();
    if (wid != 0) return;
    L2Top2 r = s_t[0][lane];
    for (int w = 1; w < kL2Warps; ++w) l2_merge(r, s_t[w][lane]);  // warp quarters in B order
    const int q = q0 + lane;
    if (gridDim.y > 1) {
        if (q < na) part[(size_t)blockIdx.y * na + q] = r;
        return;
    }
    bool k = false;
    if (q < na && nb > 0) k = l2_finish(r, q, ratio, best_idx, dist, keep);
    const int nk = __popc(__ballot_sync(0xffffffffu, k));
    if (lane == 0 && nk && count) atomicAdd(count, nk);
}

__global__ void k_match_l2_merge(const L2Top2* __restrict__ part, int na, int nsplit, double ratio,
                                 int32_t* __restrict__ best_idx, float* __restrict__ dist,
                                 uint8_t* __restrict__ keep, int32_t* __restrict__ count) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    bool k = false;
    if (q < na) {
        L2Top2 r = part[q];
        for (int sp = 1; sp < nsplit; ++sp) l2_merge(r, part[(size_t)sp * na + q]);
        k = l2_finish(r, q, ratio, best_idx, dist, keep);
    }
    const int nk = __popc(__ballot_sync(0xffffffffu, k));
    if ((threadIdx.x & 31) == 0 && nk && count) atomicAdd(count, nk);
}

size_t match_l2_scratch(int na, int nsplit) { return sizeof(L2Top2) * (size_t)na * nsplit; }

int match_l2_split(int na, int nb, int sms) {
    const int qblocks = (na + 31) / 32;  // enough CTAs for ~4 per SM, slices of >= 256 rows of B
    return std::max(1, std::min((4 * sms + qblocks - 1) / qblocks, (nb + 255) / 256));
}

int launch_match_l2(const float* a, int na, const float* b, int nb, double ratio, int32_t* best_idx,
                    float* dist, uint8_t* keep, int32_t* count, void* scratch, int nsplit,
                    cudaStream_t st) {
    if (na <= 0 || nb <= 0) return 0;
    dim3 grid((na + 31) / 32, nsplit);
    L2Top2* part = static_cast<L2Top2*>(scratch);
    k_match_l2<<<grid, 32 * kL2Warps, 0, st>>>(a, na, b, nb, ratio, best_idx, dist, keep, count, part);
    if (nsplit == 1) return 1;
    k_match_l2_merge<<<(na + 255) / 256, 256, 0, st>>>(part, na, nsplit, ratio, best_idx, dist, keep, count);
    return 2;
}

}  // namespace xa
