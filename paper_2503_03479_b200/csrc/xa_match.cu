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

int launch_match(const MatchJob* d_jobs, int njobs, int max_na, const uint64_t* a,
                 const uint64_t* b, const uint16_t* d_keep_thr, uint32_t* best_idx,
                 uint16_t* best, uint16_t* second, cudaStream_t st) {
    if (njobs <= 0 || max_na <= 0) return 0;
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

}  // namespace xa
