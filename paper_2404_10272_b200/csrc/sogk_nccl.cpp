// sogk_nccl.cpp — the multi-GPU setup step: one broadcast of the dense grid over
// the caller's NCCL communicator (NVLink 5 / NVSwitch), then every rank holds the same grid
// and builds its VDB / distance grid locally (deterministic, so byte-identical).  Rays shard
// with no data-path collective (ray_index_base gives global ray_indices).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2", preferring a copy the process already
// loaded -- e.g. torch's -- so a communicator created there is usable here); the library has
// no link-time NCCL dependency and returns SOGK_INVALID_ARG when NCCL is absent.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "sogk.h"

namespace {
using ncclResult = int;
using ncclComm = void*;
using BcastFn = ncclResult (*)(const void*, void*, size_t, int /*ncclDataType_t*/, int, ncclComm, cudaStream_t);
using RankFn = ncclResult (*)(ncclComm, int*);
using ErrFn = const char* (*)(ncclResult);
constexpr int kNcclUint8 = 1; // ncclUint8 (nccl.h)

struct Nccl {
    BcastFn bcast = nullptr;
    RankFn rank = nullptr;
    ErrFn err = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.bcast = reinterpret_cast<BcastFn>(dlsym(h, "ncclBroadcast"));
        n.rank = reinterpret_cast<RankFn>(dlsym(h, "ncclCommUserRank"));
        n.err = reinterpret_cast<ErrFn>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.bcast && n.rank && n.err;
    });
    return n;
}
} // namespace

extern "C" int sogk_last_error_set(int status, const char* msg); // sogk_api.cpp

extern "C" int sogk_grid_create_dense_broadcast(const sogk_transform* t, const uint8_t* h_bits,
                                                 size_t nbytes, int root, void* nccl_comm, void* stream,
                                                 sogk_grid** out) {
    if (!out) return sogk_last_error_set(SOGK_INVALID_ARG, "out is NULL");
    *out = nullptr;
    const Nccl& N = nccl();
    if (!N.ok) return sogk_last_error_set(SOGK_INVALID_ARG, "NCCL (libnccl.so.2) is not available");
    if (!nccl_comm) return sogk_last_error_set(SOGK_INVALID_ARG, "NCCL communicator is NULL");
    int rank = -1;
    ncclResult r = N.rank(nccl_comm, &rank);
    if (r != 0) return sogk_last_error_set(SOGK_CUDA_ERROR, (std::string("ncclCommUserRank: ") + N.err(r)).c_str());
    const bool is_root = rank == root;
    if (is_root && (!t || !h_bits))
        return sogk_last_error_set(SOGK_INVALID_ARG, "the root rank passes the transform and the payload");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // 1) the transform (fixed size), so that ranks need not know the grid in advance
    sogk_transform* d_t = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d_t), sizeof(sogk_transform));
    if (e != cudaSuccess) return sogk_last_error_set(SOGK_OOM, "broadcast scratch");
    // the root validates its arguments before any collective; an invalid grid is broadcast as
    // a zero transform so every rank fails the same way instead of waiting on the payload
    sogk_transform ht{};
    const char* root_err = nullptr;
    if (is_root) {
        const uint64_t v = uint64_t(t->res[0] > 0 ? t->res[0] : 0) * uint64_t(t->res[1] > 0 ? t->res[1] : 0) *
                           uint64_t(t->res[2] > 0 ? t->res[2] : 0);
        if (t->res[0] < 1 || t->res[1] < 1 || t->res[2] < 1 || !(t->voxel_size > 0.0))
            root_err = "broadcast transform is invalid";
        else if (nbytes != size_t((v + 7) / 8))
            root_err = "payload size must be ceil(voxel_count / 8) bytes";
        if (!root_err) ht = *t;
    }
    if (is_root) e = cudaMemcpyAsync(d_t, &ht, sizeof ht, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        r = N.bcast(d_t, d_t, sizeof(sogk_transform), kNcclUint8, root, nccl_comm, st);
        if (r != 0) {
            cudaFree(d_t);
            return sogk_last_error_set(SOGK_CUDA_ERROR, (std::string("ncclBroadcast: ") + N.err(r)).c_str());
        }
        e = cudaMemcpyAsync(&ht, d_t, sizeof ht, cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_t);
    if (e != cudaSuccess) return sogk_last_error_set(SOGK_CUDA_ERROR, cudaGetErrorString(e));
    const uint64_t vox = uint64_t(ht.res[0]) * uint64_t(ht.res[1]) * uint64_t(ht.res[2]);
    const size_t need = size_t((vox + 7) / 8);
    if (root_err) return sogk_last_error_set(SOGK_INVALID_ARG, root_err);
    if (ht.res[0] < 1 || ht.res[1] < 1 || ht.res[2] < 1 || !(ht.voxel_size > 0.0))
        return sogk_last_error_set(SOGK_INVALID_ARG, "broadcast transform is invalid (the root's arguments)");
    // 2) the payload, once, NCCL over NVLink
    uint8_t* d_bits = nullptr;
    e = cudaMalloc(reinterpret_cast<void**>(&d_bits), need);
    if (e != cudaSuccess) return sogk_last_error_set(SOGK_OOM, "broadcast payload");
    if (is_root) e = cudaMemcpyAsync(d_bits, h_bits, need, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        r = N.bcast(d_bits, d_bits, need, kNcclUint8, root, nccl_comm, st);
        if (r != 0) {
            cudaFree(d_bits);
            return sogk_last_error_set(SOGK_CUDA_ERROR, (std::string("ncclBroadcast: ") + N.err(r)).c_str());
        }
    }
    if (e != cudaSuccess) {
        cudaFree(d_bits);
        return sogk_last_error_set(SOGK_CUDA_ERROR, cudaGetErrorString(e));
    }
    const int rc = sogk_grid_create_dense_device(&ht, d_bits, need, stream, out); // ordered on `stream`, synced
    cudaFree(d_bits);
    return rc;
}
