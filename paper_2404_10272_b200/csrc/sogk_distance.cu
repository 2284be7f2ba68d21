// sogk_distance.cu — build_distance (distance.hpp:45-103) on the GPU.
//
// The reference runs a two-pass 26-neighbour chamfer, inherently sequential in raster order.
// The chessboard distance is also separable: with g0 = 0 on occupied voxels and +inf
// elsewhere,
//     D(p) = min_q max(|px-qx|, |py-qy|, |pz-qz|)
//          = min_qz max(|pz-qz|, min_qy max(|py-qy|, min_qx max(|px-qx|, g0(q))))
// (max(c, .) distributes over min when c does not depend on the minimised index), so three
// 1-D passes  out[i] = min_j max(|i - j|, g[j])  along x, y, z give the exact distances --
// the values the chamfer produces, since both are exact (distance.hpp:12-14).
// One CTA per line: the line sits in shared memory with a sparse table of range minima and
// every thread binary-searches the smallest k with  min g[i-k .. i+k] <= k.
#include <cuda_runtime.h>

#include "sogk_internal.h"

namespace sogk {

constexpr int32_t kDistInf = 1 << 29;

__device__ __forceinline__ int ilog2(int x) { return 31 - __clz(x); }

// axis 0: input is the bit payload; axes 1, 2: the previous pass
__global__ void distance_pass_kernel(int axis, const uint8_t* __restrict__ bits,
                                     const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                     int rx, int ry, int rz, int32_t sentinel,
                                     unsigned* __restrict__ any_occupied) {
    extern __shared__ int32_t sm[]; // [kDistMaxLog][N]
    const int N = axis == 0 ? rx : (axis == 1 ? ry : rz);
    // line id -> the two fixed coordinates
    const int64_t line = blockIdx.x;
    int64_t base, stride;
    if (axis == 0) { // line (y, z)
        const int64_t y = line % ry, z = line / ry;
        base = (z * ry + y) * rx;
        stride = 1;
    } else if (axis == 1) { // line (x, z)
        const int64_t x = line % rx, z = line / rx;
        base = z * ry * rx + x;
        stride = rx;
    } else { // line (x, y)
        base = line;
        stride = (int64_t)rx * ry;
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int64_t v = base + i * stride;
        int32_t g;
        if (axis == 0) {
            const bool occ = (__ldg(bits + (v >> 3)) >> (v & 7)) & 1u;
            g = occ ? 0 : kDistInf;
            if (occ) *any_occupied = 1u; // benign race: all writers store 1
        } else {
            g = in[v];
        }
        sm[i] = g;
    }
    __syncthreads();
    int levels = 1;
    for (int l = 1; (1 << l) <= N; ++l, ++levels) { // sparse table of range minima
        const int half = 1 << (l - 1);
        for (int i = threadIdx.x; i + (1 << l) <= N; i += blockDim.x) {
            const int32_t a = sm[(l - 1) * N + i], b = sm[(l - 1) * N + i + half];
            sm[l * N + i] = a < b ? a : b;
        }
        __syncthreads();
    }
    auto rmin = [&](int a, int b) { // min over [a, b]
        const int l = ilog2(b - a + 1);
        const int32_t x = sm[l * N + a], y = sm[l * N + b - (1 << l) + 1];
        return x < y ? x : y;
    };
    const int32_t all = rmin(0, N - 1);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        int32_t r;
        if (all > N - 1) {
            r = all; // every |i - j| <= N - 1 < g[j]: max(|i - j|, g[j]) = g[j]
        } else {     // smallest k in [0, N-1] with min g[i-k .. i+k] <= k (monotone in k)
            int lo = 0, hi = N - 1;
            while (lo < hi) {
                const int k = (lo + hi) >> 1;
                const int a = i - k < 0 ? 0 : i - k, b = i + k > N - 1 ? N - 1 : i + k;
                if (rmin(a, b) <= k) hi = k;
                else lo = k + 1;
            }
            r = lo;
        }
        if (axis == 2 && r >= kDistInf) r = sentinel; // nothing occupied (distance.hpp:67-71)
        out[base + i * stride] = r;
    }
}

cudaError_t launch_distance_build(const GridDev& dense, int32_t* dist, int32_t* scratch,
                                  unsigned* any_occupied, cudaStream_t st) {
    const int rx = dense.res[0], ry = dense.res[1], rz = dense.res[2];
    int32_t sentinel = rx > ry ? rx : ry;
    if (rz > sentinel) sentinel = rz;
    cudaError_t e = cudaMemsetAsync(any_occupied, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    const int n[3] = {rx, ry, rz};
    const int64_t lines[3] = {(int64_t)ry * rz, (int64_t)rx * rz, (int64_t)rx * ry};
    // ping-pong so that the last pass lands in `dist`: x -> dist, y -> scratch, z -> dist
    int32_t* const bufs[3] = {dist, scratch, dist};
    const int32_t* in = nullptr;
    for (int axis = 0; axis < 3; ++axis) {
        int levels = 1;
        while ((1 << levels) <= n[axis]) ++levels;
        const size_t smem = size_t(levels) * n[axis] * sizeof(int32_t);
        const int threads = n[axis] < 1024 ? ((n[axis] + 31) / 32) * 32 : 1024;
        if (smem > 48 * 1024) {
            e = cudaFuncSetAttribute(distance_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            if (e != cudaSuccess) return e;
        }
        distance_pass_kernel<<<(unsigned)lines[axis], threads, smem, st>>>(
            axis, dense.bits, in, bufs[axis], rx, ry, rz, sentinel, any_occupied);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        in = bufs[axis];
    }
    return cudaSuccess;
}

} // namespace sogk
