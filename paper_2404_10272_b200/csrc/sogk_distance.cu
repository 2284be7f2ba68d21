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
//
// Each 1-D transform is two O(N) sweeps.  Sweeping left to right, L(i) = min_{j<=i} term_j(i)
// with term_j(i) = max(i - j, g[j]): a term is flat at g[j] until i = j + g[j] and then grows
// by one per step, so L(i) is L(i-1) if some term of value v = L(i-1) is still flat at i --
// i.e. the last j with g[j] = v has j + v >= i -- and v + 1 otherwise, then min'ed with g[i].
// `last[v]` per line is all the state; the right-to-left sweep is the mirror and the result
// is min(L, R).  Values g[j] >= N are flat over the whole line and fold into one line
// constant.  The x pass reads the bit payload (binary input: distance to the nearest set bit).
// Loads and stores are coalesced: the x pass stages 32 consecutive rows (one warp, one row
// per lane) in shared memory; the y / z passes give adjacent lanes adjacent x.
#include <cuda_runtime.h>

#include "sogk_internal.h"

namespace sogk {

constexpr int32_t kDistInf = 1 << 29;
constexpr int kRowsPerWarp = 32;

// x pass: one warp = 32 consecutive rows; tile[row][i] (uint16, stride N + 1) holds L then
// the result; bits of the 32 rows are staged first (they are contiguous in the payload)
__global__ void __launch_bounds__(32) distance_x_kernel(const uint8_t* __restrict__ bits,
                                                        int32_t* __restrict__ out, int rx,
                                                        int64_t nrows,
                                                        unsigned* __restrict__ any_occupied) {
    extern __shared__ uint16_t tile[]; // [32][N + 1], then the staged bits
    const int N = rx, lane = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsPerWarp;
    const int rows = nrows - r0 < kRowsPerWarp ? (int)(nrows - r0) : kRowsPerWarp;
    uint8_t* sb = reinterpret_cast<uint8_t*>(tile + kRowsPerWarp * (N + 1));
    // staged bits: voxel (r0 * N + e) for e in [0, rows * N); the first byte may be unaligned
    const int64_t v0 = r0 * N, v1 = v0 + (int64_t)rows * N;
    const int64_t b0 = v0 >> 3, b1 = (v1 + 7) >> 3;
    for (int64_t b = b0 + lane; b < b1; b += 32) sb[b - b0] = __ldg(bits + b);
    __syncwarp();
    const int sh = (int)(v0 & 7);
    auto bit = [&](int row, int i) {
        const int64_t e = (int64_t)row * N + i + sh;
        return (sb[e >> 3] >> (e & 7)) & 1;
    };
    bool any = false;
    if (lane < rows) {
        uint16_t* t = tile + lane * (N + 1);
        constexpr int kInf16 = 0xFFFF;
        int last = -kDistInf;
        for (int i = 0; i < N; ++i) {
            if (bit(lane, i)) last = i;
            const int d = i - last;
            t[i] = (uint16_t)(d < kInf16 ? d : kInf16);
        }
        any = last >= 0;
        int next = kDistInf;
        for (int i = N - 1; i >= 0; --i) {
            if (bit(lane, i)) next = i;
            const int d = next - i;
            const int l = t[i];
            const int m = d < l ? d : l;
            t[i] = (uint16_t)(m < kInf16 ? m : kInf16);
        }
    }
    if (__any_sync(0xffffffffu, any) && lane == 0) *any_occupied = 1u;
    __syncwarp();
    const int64_t n = (int64_t)rows * N;
    for (int64_t e = lane; e < n; e += 32) {
        const int row = (int)(e / N), i = (int)(e - (int64_t)row * N);
        const int v = tile[row * (N + 1) + i];
        out[v0 + e] = v == 0xFFFF ? kDistInf : v;
    }
}

// y / z pass: one thread per line, adjacent lanes adjacent x; last[v] per line in shared
// memory as int16 ([N + 1][blockDim]), lines of length N <= 2047
template <int AXIS>
__global__ void distance_line_kernel(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                     int rx, int ry, int rz, int32_t sentinel) {
    extern __shared__ int16_t lastv[];
    const int N = AXIS == 1 ? ry : rz;
    const int64_t nlines = AXIS == 1 ? (int64_t)rx * rz : (int64_t)rx * ry;
    const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int bd = blockDim.x, t = threadIdx.x;
    if (line >= nlines) return;
    const int64_t slab = (int64_t)rx * ry;
    const int64_t x = line % rx, o = line / rx;
    const int64_t base = AXIS == 1 ? o * slab + x : o * rx + x;
    const int64_t stride = AXIS == 1 ? rx : slab;
    auto L = [&](int v) -> int16_t& { return lastv[v * bd + t]; };
    constexpr int kNone = -32768;
    constexpr int kChunk = 8; // loads of a chunk are issued together, ahead of the recurrence
    for (int v = 0; v <= N; ++v) L(v) = kNone;
    int cst = kDistInf; // min of the values >= N (flat across the line)
    int cur = kDistInf;
    for (int i0 = 0; i0 < N; i0 += kChunk) {
        int gv[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            gv[k] = i0 + k < N ? __ldg(in + base + (int64_t)(i0 + k) * stride) : 0;
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            const int i = i0 + k, g = gv[k];
            if (i >= N) break;
            if (cur < kDistInf) cur = (cur < N && L(cur) + cur >= i) ? cur : cur + 1;
            if (g < N) {
                L(g) = (int16_t)i;
                cur = g < cur ? g : cur;
            } else if (g < cst) {
                cst = g;
            }
            gv[k] = cur;
        }
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            if (i0 + k < N) out[base + (int64_t)(i0 + k) * stride] = gv[k];
    }
    for (int v = 0; v <= N; ++v) L(v) = kNone; // now "first j >= i with g[j] = v"
    cur = kDistInf;
    const int top = ((N + kChunk - 1) / kChunk) * kChunk;
    for (int i0 = top - kChunk; i0 >= 0; i0 -= kChunk) {
        int gv[kChunk], lv[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            const bool ok = i0 + k < N;
            const int64_t p = base + (int64_t)(i0 + k) * stride;
            gv[k] = ok ? __ldg(in + p) : 0;
            lv[k] = ok ? out[p] : 0;
        }
#pragma unroll
        for (int k = kChunk - 1; k >= 0; --k) {
            const int i = i0 + k, g = gv[k];
            if (i >= N) continue;
            if (cur < kDistInf) cur = (cur < N && L(cur) != kNone && L(cur) - cur <= i) ? cur : cur + 1;
            if (g < N) {
                L(g) = (int16_t)i;
                cur = g < cur ? g : cur;
            }
            int r = lv[k];
            r = cur < r ? cur : r;
            r = cst < r ? cst : r;
            if (AXIS == 2 && r >= kDistInf) r = sentinel; // nothing occupied (distance.hpp:67-71)
            lv[k] = r;
        }
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            if (i0 + k < N) out[base + (int64_t)(i0 + k) * stride] = lv[k];
    }
}

template <int AXIS>
static cudaError_t launch_line(const int32_t* in, int32_t* out, int rx, int ry, int rz,
                               int32_t sentinel, cudaStream_t st) {
    const int N = AXIS == 1 ? ry : rz;
    const int64_t nlines = AXIS == 1 ? (int64_t)rx * rz : (int64_t)rx * ry;
    int bd = 128;
    while (bd > 32 && size_t(N + 1) * bd * sizeof(int16_t) > 96 * 1024) bd >>= 1;
    const size_t smem = size_t(N + 1) * bd * sizeof(int16_t);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(distance_line_kernel<AXIS>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    distance_line_kernel<AXIS><<<(unsigned)((nlines + bd - 1) / bd), bd, smem, st>>>(in, out, rx, ry,
                                                                                  rz, sentinel);
    return cudaGetLastError();
}

cudaError_t launch_distance_build(const GridDev& dense, int32_t* dist, int32_t* scratch,
                                  unsigned* any_occupied, cudaStream_t st) {
    const int rx = dense.res[0], ry = dense.res[1], rz = dense.res[2];
    int32_t sentinel = rx > ry ? rx : ry;
    if (rz > sentinel) sentinel = rz;
    cudaError_t e = cudaMemsetAsync(any_occupied, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    // x -> dist, y -> scratch, z -> dist
    const int64_t nrows = (int64_t)ry * rz;
    const size_t smem_x = size_t(kRowsPerWarp) * (rx + 1) * sizeof(uint16_t) + size_t(kRowsPerWarp) * rx / 8 + 16;
    if (smem_x > 48 * 1024) {
        e = cudaFuncSetAttribute(distance_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x);
        if (e != cudaSuccess) return e;
    }
    distance_x_kernel<<<(unsigned)((nrows + kRowsPerWarp - 1) / kRowsPerWarp), 32, smem_x, st>>>(
        dense.bits, dist, rx, nrows, any_occupied);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_line<1>(dist, scratch, rx, ry, rz, sentinel, st)) != cudaSuccess) return e;
    return launch_line<2>(scratch, dist, rx, ry, rz, sentinel, st);
}

} // namespace sogk
