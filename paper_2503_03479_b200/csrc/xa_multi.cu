// xa_multi.cu — multi-GPU sharding of the batched coarse search.
//
// The reference parallelises coarse_search with a std::thread parallel_for
// over grid entries on one host (proj/include/xaffine/parallel.hpp:22-36,
// proj/src/pipeline.cpp:130). Here the unit of sharding is the image pair
// (BASELINE config 5): pairs are split into contiguous blocks, one block per
// GPU, each block runs through that GPU's batched pipeline, and the only
// exchange is gathering the per-pair counts.
//
//   xa_coarse_search_multi   one process, a list of engines (one per device):
//                            one host thread per engine, results land in the
//                            caller's arrays at the block offsets;
//   xa_coarse_search_nccl    one process per GPU (MPI / torchrun ranks): each
//                            rank runs its block, then the counts of every
//                            rank are all-gathered over the caller's NCCL
//                            communicator (NVLink / NVSwitch), so every rank
//                            returns the whole job.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, the library the
// process already loaded -- e.g. torch's -- when there is one), so the C-ABI
// library has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/xaffine_b200.h"

namespace {

// Contiguous block [lo, hi) of n items for rank r of w (bench.py / dist.py block_range).
void block_range(int n, int w, int r, int& lo, int& hi) {
    const int base = n / w, rem = n % w;
    lo = r * base + std::min(r, rem);
    hi = lo + base + (r < rem ? 1 : 0);
}

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.get_unique_id = (decltype(n.get_unique_id))dlsym(h, "ncclGetUniqueId");
        n.comm_init_rank = (decltype(n.comm_init_rank))dlsym(h, "ncclCommInitRank");
        n.comm_destroy = (decltype(n.comm_destroy))dlsym(h, "ncclCommDestroy");
        n.all_gather = (decltype(n.all_gather))dlsym(h, "ncclAllGather");
        n.error_string = (decltype(n.error_string))dlsym(h, "ncclGetErrorString");
        n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather && n.error_string;
    });
    return n;
}

thread_local std::string g_merr;

int fail(int code, const std::string& m) {
    g_merr = m;
    return code;
}

}  // namespace

extern "C" {

const char* xa_multi_last_error(void) { return g_merr.c_str(); }

int xa_coarse_search_multi(xa_engine* const* engines, int n_engines, int pixel_type, const void* const* refs,
                           int w, int h, const void* const* targets, int tw, int th, int n_pairs,
                           const xa_params* grid, int n, int max_points, double ratio, int warp_mode,
                           int32_t* counts, int32_t* kp_counts, int32_t* best) {
    if (n_engines <= 0 || !engines) return fail(XA_EINVAL, "coarse_multi: no engines");
    if (n_pairs <= 0 || !refs || !targets) return fail(XA_EINVAL, "coarse: no image pairs");
    if (n <= 0 || !grid) return fail(XA_EPIPELINE, "coarse: empty parameter grid");
    std::vector<int> rc(n_engines, XA_OK);
    std::vector<std::string> err(n_engines);
    std::vector<std::thread> workers;
    for (int r = 0; r < n_engines; ++r) {
        int lo, hi;
        block_range(n_pairs, n_engines, r, lo, hi);
        if (hi <= lo) continue;
        workers.emplace_back([&, r, lo, hi] {
            rc[r] = xa_coarse_search_batch(engines[r], pixel_type, refs + lo, w, h, targets + lo, tw, th,
                                           hi - lo, grid, n, max_points, ratio, warp_mode,
                                           counts ? counts + (size_t)lo * n : nullptr,
                                           kp_counts ? kp_counts + (size_t)lo * n : nullptr,
                                           best ? best + lo : nullptr);
            if (rc[r] != XA_OK) err[r] = xa_last_error();
        });
    }
    for (auto& t : workers) t.join();
    for (int r = 0; r < n_engines; ++r)
        if (rc[r] != XA_OK) return fail(rc[r], "engine " + std::to_string(r) + ": " + err[r]);
    return XA_OK;
}

int xa_nccl_unique_id(void* id, size_t bytes) {
    const Nccl& N = nccl();
    if (!N.ok) return fail(XA_ECUDA, "NCCL not loadable (libnccl.so.2)");
    if (bytes < sizeof(ncclUniqueId)) return fail(XA_EINVAL, "nccl id buffer too small");
    ncclUniqueId u;
    const ncclResult_t r = N.get_unique_id(&u);
    if (r != ncclSuccess) return fail(XA_ECUDA, std::string("ncclGetUniqueId: ") + N.error_string(r));
    std::memcpy(id, &u, sizeof u);
    return XA_OK;
}

int xa_nccl_comm_init(void** comm, int world, const void* id, int rank, int device) {
    const Nccl& N = nccl();
    if (!N.ok) return fail(XA_ECUDA, "NCCL not loadable (libnccl.so.2)");
    if (cudaSetDevice(device) != cudaSuccess) return fail(XA_ECUDA, "cudaSetDevice");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    const ncclResult_t r = N.comm_init_rank(&c, world, u, rank);
    if (r != ncclSuccess) return fail(XA_ECUDA, std::string("ncclCommInitRank: ") + N.error_string(r));
    *comm = c;
    return XA_OK;
}

int xa_nccl_comm_destroy(void* comm) {
    const Nccl& N = nccl();
    if (!N.ok || !comm) return XA_OK;
    N.comm_destroy(static_cast<ncclComm_t>(comm));
    return XA_OK;
}

int xa_coarse_search_nccl(xa_engine* e, void* comm, int rank, int world, int pixel_type,
                          const void* const* refs, int w, int h, const void* const* targets, int tw, int th,
                          int n_pairs, const xa_params* grid, int n, int max_points, double ratio,
                          int warp_mode, int32_t* counts, int32_t* kp_counts, int32_t* best) {
    const Nccl& N = nccl();
    if (!N.ok) return fail(XA_ECUDA, "NCCL not loadable (libnccl.so.2)");
    if (!comm || world <= 0 || rank < 0 || rank >= world) return fail(XA_EINVAL, "coarse_nccl: communicator");
    if (n_pairs <= 0 || !refs || !targets) return fail(XA_EINVAL, "coarse: no image pairs");
    if (n <= 0 || !grid) return fail(XA_EPIPELINE, "coarse: empty parameter grid");
    int lo, hi;
    block_range(n_pairs, world, rank, lo, hi);
    const int blk = (n_pairs + world - 1) / world;  // padded block (all-gather needs equal sizes)
    const size_t rec = (size_t)2 * n + 1;           // counts, kp counts, best per pair
    std::vector<int32_t> mine((size_t)blk * rec, -1);
    if (hi > lo) {
        std::vector<int32_t> c((size_t)(hi - lo) * n), k((size_t)(hi - lo) * n), b(hi - lo);
        const int rc = xa_coarse_search_batch(e, pixel_type, refs + lo, w, h, targets + lo, tw, th, hi - lo, grid,
                                              n, max_points, ratio, warp_mode, c.data(), k.data(), b.data());
        if (rc != XA_OK) return fail(rc, xa_last_error());
        for (int p = 0; p < hi - lo; ++p) {
            int32_t* r = mine.data() + (size_t)p * rec;
            std::memcpy(r, c.data() + (size_t)p * n, sizeof(int32_t) * n);
            std::memcpy(r + n, k.data() + (size_t)p * n, sizeof(int32_t) * n);
            r[2 * n] = b[p];
        }
    }
    cudaStream_t st = static_cast<cudaStream_t>(xa_engine_stream(e));
    int32_t* d = nullptr;
    const size_t per = (size_t)blk * rec;
    if (cudaMalloc(&d, sizeof(int32_t) * per * (world + 1)) != cudaSuccess)
        return fail(XA_ENOMEM, "coarse_nccl: gather buffer");
    std::vector<int32_t> all(per * world);
    int rc = XA_OK;
    if (cudaMemcpyAsync(d, mine.data(), sizeof(int32_t) * per, cudaMemcpyHostToDevice, st) != cudaSuccess) {
        rc = fail(XA_ECUDA, "coarse_nccl: upload");
    } else {
        const ncclResult_t r = N.all_gather(d, d + per, per, ncclInt32, static_cast<ncclComm_t>(comm), st);
        if (r != ncclSuccess) rc = fail(XA_ECUDA, std::string("ncclAllGather: ") + N.error_string(r));
        else if (cudaMemcpyAsync(all.data(), d + per, sizeof(int32_t) * per * world, cudaMemcpyDeviceToHost,
                                 st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
            rc = fail(XA_ECUDA, "coarse_nccl: readback");
    }
    cudaFree(d);
    if (rc != XA_OK) return rc;
    for (int r = 0; r < world; ++r) {
        int a, z;
        block_range(n_pairs, world, r, a, z);
        for (int p = a; p < z; ++p) {
            const int32_t* src = all.data() + per * r + (size_t)(p - a) * rec;
            if (counts) std::memcpy(counts + (size_t)p * n, src, sizeof(int32_t) * n);
            if (kp_counts) std::memcpy(kp_counts + (size_t)p * n, src + n, sizeof(int32_t) * n);
            if (best) best[p] = src[2 * n];
        }
    }
    return XA_OK;
}

}  // extern "C"
