// sogk_vdb.cu — K1: dense occupancy bits -> VDB hierarchy on the GPU.
//
// Replaces build_sparse + read_leaf_block (sparse.hpp:283-371).  One CTA per
// 128^3 region (internal node), 512 threads, 8 children of the 16^3 node per
// thread:
//   classify: each child reads its 8^3 block (64 row bytes on the aligned fast
//             path, :291-310; per-voxel padded path otherwise, :312-323),
//             warp ballots form the child (mixed) and value (full) masks, CTA
//             popcounts decide the root-tile collapse (:360-367).
//   fill:     CTA-wide exclusive scan of the region leaf counts gives the
//             node's leaf base; a 64-word popcount prefix gives every mixed
//             child its slot (ci order, the order SOG1 walks, io.hpp:174-178);
//             mixed children copy their 64 bytes into the leaf pool.
// Both kernels read the dense payload once (256 KiB at 128^3, 16 MiB at
// 512^3); no host round trip, the leaf pool is sized for the worst case.
#include <cuda_runtime.h>

#include "sogk_device.cuh"
#include "sogk_internal.h"

namespace sogk {

constexpr int kBuildThreads = 512;

// 8^3 block at `bo` as 8 leaf words (word z = bytes z*8+y, bit x); out-of-grid voxels read empty
__device__ __forceinline__ void read_block(const GridDev& d, const int bo[3], uint64_t w[8]) {
    const bool aligned = (d.res[0] % 8 == 0) && bo[0] >= 0 && bo[0] + 8 <= d.res[0] &&
                         bo[1] >= 0 && bo[1] + 8 <= d.res[1] && bo[2] >= 0 &&
                         bo[2] + 8 <= d.res[2];
    if (aligned) {
        const uint64_t row_bytes = (uint64_t)d.res[0] / 8;
        const uint64_t xb = (uint64_t)bo[0] / 8;
#pragma unroll
        for (int lz = 0; lz < 8; ++lz) {
            uint64_t word = 0;
#pragma unroll
            for (int ly = 0; ly < 8; ++ly) {
                const uint64_t row =
                    ((uint64_t)(bo[2] + lz) * (uint64_t)d.res[1] + (uint64_t)(bo[1] + ly)) *
                        row_bytes +
                    xb;
                word |= (uint64_t)__ldg(d.bits + row) << (8 * ly);
            }
            w[lz] = word;
        }
        return;
    }
    for (int lz = 0; lz < 8; ++lz) {
        uint64_t word = 0;
        for (int ly = 0; ly < 8; ++ly)
            for (int lx = 0; lx < 8; ++lx) {
                const int ijk[3] = {bo[0] + lx, bo[1] + ly, bo[2] + lz};
                if (dense_voxel(d, ijk)) word |= 1ull << (ly * 8 + lx);
            }
        w[lz] = word;
    }
}

__device__ __forceinline__ void child_origin(int r, const int R[3], int ci, int bo[3]) {
    const int rx = r % R[0], ry = (r / R[0]) % R[1], rz = r / (R[0] * R[1]);
    bo[0] = rx * 128 + (ci & 15) * 8;
    bo[1] = ry * 128 + ((ci >> 4) & 15) * 8;
    bo[2] = rz * 128 + (ci >> 8) * 8;
}

__global__ void __launch_bounds__(kBuildThreads) vdb_classify_kernel(const VdbBuildArgs a) {
    __shared__ int s_mixed, s_full;
    const int r = blockIdx.x;
    if (threadIdx.x == 0) s_mixed = s_full = 0;
    __syncthreads();
    int my_mixed = 0, my_full = 0;
    uint32_t* cm32 = reinterpret_cast<uint32_t*>(a.child_mask) + (int64_t)r * 128;
    uint32_t* vm32 = reinterpret_cast<uint32_t*>(a.value_mask) + (int64_t)r * 128;
#pragma unroll 1
    for (int k = 0; k < 4096 / kBuildThreads; ++k) {
        const int ci = threadIdx.x + kBuildThreads * k;
        int bo[3];
        child_origin(r, a.R, ci, bo);
        uint64_t w[8];
        read_block(a.dense, bo, w);
        uint64_t and_ = ~0ull, or_ = 0;
#pragma unroll
        for (int z = 0; z < 8; ++z) {
            and_ &= w[z];
            or_ |= w[z];
        }
        const bool full = and_ == ~0ull, empty = or_ == 0;
        const bool mixed = !(full || empty); // uniform leaves collapse to tiles (:353-355)
        const unsigned bm = __ballot_sync(0xffffffffu, mixed);
        const unsigned bv = __ballot_sync(0xffffffffu, full);
        if ((threadIdx.x & 31) == 0) {
            cm32[ci >> 5] = bm;
            vm32[ci >> 5] = bv;
            my_mixed += __popc(bm);
            my_full += __popc(bv);
        }
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_mixed, my_mixed);
        atomicAdd(&s_full, my_full);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a.region_leaves[r] = (uint32_t)s_mixed;
        // InternalNode::uniform_tiles (:92-99) -> root tile; else an internal node (:360-367)
        int32_t node = r;
        if (s_mixed == 0 && s_full == 0) node = kRootEmpty;
        if (s_mixed == 0 && s_full == 4096) node = kRootOccupied;
        a.root[r] = node;
    }
}

__global__ void __launch_bounds__(kBuildThreads) vdb_fill_kernel(const VdbBuildArgs a, int nreg) {
    __shared__ uint32_t s_part[kBuildThreads / 32];
    __shared__ uint32_t s_base;
    const int r = blockIdx.x;
    // leaf base = sum of the leaf counts of all preceding regions (z, y, x order)
    uint32_t part = 0;
    for (int j = threadIdx.x; j < r; j += kBuildThreads) part += a.region_leaves[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t b = 0;
        for (int i = 0; i < kBuildThreads / 32; ++i) b += s_part[i];
        s_base = b;
        if (r == nreg - 1) *a.total_leaves = b + a.region_leaves[r];
    }
    __syncthreads();
    if (a.root[r] < 0) return;
    const uint64_t* cm = a.child_mask + (int64_t)r * 64;
    if (threadIdx.x == 0) { // 64-word exclusive popcount prefix
        uint32_t acc = s_base;
        for (int w = 0; w < 64; ++w) {
            a.prefix[(int64_t)r * 64 + w] = acc;
            acc += (uint32_t)__popcll(cm[w]);
        }
    }
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k < 4096 / kBuildThreads; ++k) {
        const int ci = threadIdx.x + kBuildThreads * k;
        const uint64_t m = cm[ci >> 6];
        const int b = ci & 63;
        if (!((m >> b) & 1ull)) continue;
        const uint64_t leaf =
            (uint64_t)a.prefix[(int64_t)r * 64 + (ci >> 6)] + __popcll(m & ((1ull << b) - 1ull));
        int bo[3];
        child_origin(r, a.R, ci, bo);
        uint64_t w[8];
        read_block(a.dense, bo, w);
        uint2* dst = reinterpret_cast<uint2*>(a.leaves + leaf * 8);
#pragma unroll
        for (int z = 0; z < 8; ++z) dst[z] = make_uint2((uint32_t)w[z], (uint32_t)(w[z] >> 32));
    }
}

// child table: one CTA per node, every child's leaf index (prefix + popcount, as K1 placed
// the leaves) or its tile value
__global__ void __launch_bounds__(kBuildThreads) vdb_table_kernel(const VdbBuildArgs a) {
    const int r = blockIdx.x;
    if (a.root[r] < 0) return; // collapsed regions have no node
    const uint64_t* cm = a.child_mask + (int64_t)r * 64;
    const uint64_t* vm = a.value_mask + (int64_t)r * 64;
    const uint32_t* pf = a.prefix + (int64_t)r * 64;
    for (int ci = threadIdx.x; ci < 4096; ci += kBuildThreads) {
        const uint64_t m = cm[ci >> 6];
        const int b = ci & 63;
        int32_t v;
        if ((m >> b) & 1ull) v = (int32_t)(pf[ci >> 6] + __popcll(m & ((1ull << b) - 1ull)));
        else v = ((vm[ci >> 6] >> b) & 1ull) ? kTileOccupied : kTileEmpty;
        a.table[(int64_t)r * 4096 + ci] = v;
    }
}

cudaError_t launch_vdb_table(const VdbBuildArgs& a, cudaStream_t st) {
    const int nreg = a.R[0] * a.R[1] * a.R[2];
    vdb_table_kernel<<<nreg, kBuildThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_vdb_build(const VdbBuildArgs& a, cudaStream_t st) {
    const int nreg = a.R[0] * a.R[1] * a.R[2];
    vdb_classify_kernel<<<nreg, kBuildThreads, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    vdb_fill_kernel<<<nreg, kBuildThreads, 0, st>>>(a, nreg);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_vdb_table(a, st);
}

// to_dense (sparse.hpp:374-383): one thread per payload byte (8 consecutive voxels)
__global__ void vdb_to_dense_kernel(const GridDev g, uint8_t* bits, int64_t nbytes) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nbytes) return;
    const int64_t nvox = (int64_t)g.res[0] * g.res[1] * g.res[2];
    VdbCursor c;
    c.reset();
    uint8_t out = 0;
    for (int b = 0; b < 8; ++b) {
        const int64_t idx = i * 8 + b;
        if (idx >= nvox) break;
        const int ijk[3] = {(int)(idx % g.res[0]), (int)((idx / g.res[0]) % g.res[1]),
                            (int)(idx / ((int64_t)g.res[0] * g.res[1]))};
        if (c.query(g, ijk).occ) out |= (uint8_t)(1u << b);
    }
    bits[i] = out;
}

cudaError_t launch_vdb_to_dense(const GridDev& vdb, uint8_t* bits, int64_t nbytes,
                                cudaStream_t st) {
    if (nbytes <= 0) return cudaSuccess;
    vdb_to_dense_kernel<<<(unsigned)((nbytes + 255) / 256), 256, 0, st>>>(vdb, bits, nbytes);
    return cudaGetLastError();
}

} // namespace sogk
