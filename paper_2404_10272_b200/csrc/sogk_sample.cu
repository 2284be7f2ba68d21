// sogk_sample.cu — K2/K3/K5 sampling kernels (count + write) and K6 raygen.
//
// Pass 1 (count): one thread per ray runs the analyzer + ladder exactly like
// run_sampler / run_cascade_sampler (sampling.hpp:166-196, 440-455) but only
// counts samples.  The per-ray counts are exclusive-scanned inside the same
// kernel with a single-pass decoupled look-back over 256-ray tiles, so
// packed_info = {offset, count} and the total come out of one launch.
// Pass 2 (write): one thread per ray with count > 0 replays the same
// traversal and writes its samples at packed_info.offset, stopping as soon as
// `count` samples are out (the tail of the ray is never traversed).
#include <cuda_runtime.h>

#include "sogk_device.cuh"
#include "sogk_internal.h"

namespace sogk {

constexpr int kBlock = 256;

// ---------------------------------------------------------------------------
// ray sources
// ---------------------------------------------------------------------------
struct RaysFromBuffer {
    const double* rays;
    __device__ __forceinline__ Ray load(int64_t i) const {
        const double2* p = reinterpret_cast<const double2*>(rays + 8 * i);
        const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3);
        Ray r;
        r.o[0] = a.x;
        r.o[1] = a.y;
        r.o[2] = b.x;
        r.d[0] = b.y;
        r.d[1] = c.x;
        r.d[2] = c.y;
        r.tmin = d.x;
        r.tmax = d.y;
        return r;
    }
};

// Camera::pixel_ray, camera.hpp:167-179 (per-camera terms precomputed on the host)
__device__ __forceinline__ Ray pixel_ray(const CameraDev& c, int64_t pix) {
    const int px = (int)(pix % c.width);
    const int py = (int)(pix / c.width);
    const double u = (((double)px + 0.5) / (double)c.width * 2.0 - 1.0) * c.tan_half * c.aspect;
    const double v = (1.0 - ((double)py + 0.5) / (double)c.height * 2.0) * c.tan_half;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = c.forward[a] + c.right[a] * u + c.cam_up[a] * v;
    const double len = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    Ray r;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = c.position[a];
        r.d[a] = d[a] / len;
    }
    r.tmin = 0.0;
    r.tmax = c.t_far;
    return r;
}

struct RaysFromCamera {
    CameraDev cam;
    int64_t first;
    __device__ __forceinline__ Ray load(int64_t i) const { return pixel_ray(cam, first + i); }
};

// ---------------------------------------------------------------------------
// sinks
// ---------------------------------------------------------------------------
struct CountSink {
    int n;
    __device__ __forceinline__ bool emit(double, double, const Event&) {
        ++n;
        return true;
    }
};

struct WriteSink {
    int64_t off;
    int n, count;
    int32_t ray_index;
    double* t_starts;
    double* t_ends;
    int32_t* ray_indices;
    uint32_t* cells;
    uint8_t* levels;
    __device__ __forceinline__ bool emit(double t, double t_next, const Event& ev) {
        const int64_t k = off + n;
        t_starts[k] = t;
        if (t_ends) t_ends[k] = t_next;
        if (ray_indices) ray_indices[k] = ray_index;
        if (cells) cells[k] = pack_cell(ev.ijk);
        if (levels) levels[k] = (uint8_t)(ev.level | (ev.grid_level << 2));
        return ++n < count;
    }
};

template <int AN, bool CASC>
struct PickAn {
    using Sub = typename std::conditional<AN == SOGK_HDDA, HddaAn, DdaAn>::type;
    using type = AnyAn<Sub, CASC>;
};

// ---------------------------------------------------------------------------
// block scan + decoupled look-back
// ---------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ long long warp_incl_scan(long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// returns the exclusive prefix of v within the block; *total = block sum
__device__ __forceinline__ long long block_excl_scan(long long v, long long* total) {
    __shared__ long long warp_tot[kBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long incl = warp_incl_scan(v);
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long w = lane < kBlock / 32 ? warp_tot[lane] : 0;
        w = warp_incl_scan(w);
        if (lane < kBlock / 32) warp_tot[lane] = w; // inclusive over warps
    }
    __syncthreads();
    const long long before = wid > 0 ? warp_tot[wid - 1] : 0;
    *total = warp_tot[kBlock / 32 - 1];
    return before + incl - v;
}

__device__ __forceinline__ long long block_sum(long long v) {
    long long t;
    block_excl_scan(v, &t);
    __syncthreads();
    return t;
}

__device__ __forceinline__ void tile_publish(uint64_t* tiles, int64_t bid, uint64_t word) {
    atomicExch(reinterpret_cast<unsigned long long*>(tiles + bid), (unsigned long long)word);
}

// exclusive prefix of tile `bid` given its aggregate (called by one thread)
__device__ uint64_t tile_lookback(uint64_t* tiles, int64_t bid, uint64_t agg) {
    if (bid == 0) {
        tile_publish(tiles, 0, kFlagInc | agg);
        return 0;
    }
    tile_publish(tiles, bid, kFlagAgg | agg);
    uint64_t excl = 0;
    int64_t j = bid - 1;
    for (;;) {
        const uint64_t w = *reinterpret_cast<volatile uint64_t*>(tiles + j);
        const uint64_t f = w & ~kValMask;
        if (f == 0) continue; // predecessor still running
        excl += w & kValMask;
        if (f == kFlagInc) break;
        --j;
    }
    tile_publish(tiles, bid, kFlagInc | (excl + agg));
    return excl;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <int AN, bool CASC, bool BR, int SCH, class Src>
__global__ void __launch_bounds__(kBlock)
    count_kernel(const SamplerDev s, const Src src, int64_t n, int64_t* __restrict__ packed,
                 int64_t* __restrict__ stats, uint8_t* __restrict__ status,
                 int32_t* __restrict__ counters, uint64_t* __restrict__ tiles,
                 unsigned int* __restrict__ tile_ctr) {
    __shared__ int64_t s_bid;
    __shared__ uint64_t s_excl;
    if (threadIdx.x == 0) s_bid = atomicAdd(tile_ctr, 1u); // dynamic tile id: in-order look-back
    __syncthreads();
    const int64_t bid = s_bid;
    const int64_t r = bid * kBlock + threadIdx.x;

    int cnt = 0, st = SOGK_RAY_OK, lk = 0, sp = 0, klk = 0;
    if (r < n) {
        const Ray ray = src.load(r);
        if (!ray_valid(ray)) {
            st = SOGK_RAY_INVALID;
        } else {
            typename PickAn<AN, CASC>::type an;
            an.init(ray, s);
            CountSink sink{0};
            run_kernel<BR, SCH>(an, s, sink, klk);
            if (an.undefined()) {
                st = SOGK_RAY_UNDEFINED;
                klk = 0;
            } else {
                cnt = sink.n;
                lk = an.lookups();
                sp = an.steps();
            }
        }
        if (status) status[r] = (uint8_t)st;
        if (counters) {
            counters[3 * r] = lk;
            counters[3 * r + 1] = sp;
            counters[3 * r + 2] = klk;
        }
    }

    long long agg;
    const long long excl_in = block_excl_scan(cnt, &agg);
    if (threadIdx.x == 0) s_excl = tile_lookback(tiles, bid, (uint64_t)agg);
    __syncthreads();
    if (r < n) {
        longlong2 pi;
        pi.x = (long long)s_excl + excl_in;
        pi.y = cnt;
        reinterpret_cast<longlong2*>(packed)[r] = pi;
    }
    if (bid == (int64_t)gridDim.x - 1 && threadIdx.x == 0)
        stats[SOGK_STAT_TOTAL_SAMPLES] = (int64_t)(s_excl + agg);

    // block-reduced statistics (cheap: 5 reductions per 256 rays)
    const long long inv = block_sum(st == SOGK_RAY_INVALID);
    const long long und = block_sum(st == SOGK_RAY_UNDEFINED);
    const long long slk = block_sum(lk), ssp = block_sum(sp), sklk = block_sum(klk);
    if (threadIdx.x == 0) {
        unsigned long long* S = reinterpret_cast<unsigned long long*>(stats);
        if (inv) atomicAdd(S + SOGK_STAT_INVALID_RAYS, (unsigned long long)inv);
        if (und) atomicAdd(S + SOGK_STAT_UNDEFINED_RAYS, (unsigned long long)und);
        atomicAdd(S + SOGK_STAT_ANALYZER_LOOKUPS, (unsigned long long)slk);
        atomicAdd(S + SOGK_STAT_ANALYZER_STEPS, (unsigned long long)ssp);
        if (sklk) atomicAdd(S + SOGK_STAT_KERNEL_LOOKUPS, (unsigned long long)sklk);
    }
}

template <int AN, bool CASC, bool BR, int SCH, class Src>
__global__ void __launch_bounds__(kBlock)
    write_kernel(const SamplerDev s, const Src src, int64_t n, const int64_t* __restrict__ packed,
                 int64_t ray_index_base, double* __restrict__ t_starts, double* __restrict__ t_ends,
                 int32_t* __restrict__ ray_indices, uint32_t* __restrict__ cells,
                 uint8_t* __restrict__ levels) {
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (r >= n) return;
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
    if (pi.y == 0) return;
    const Ray ray = src.load(r);
    typename PickAn<AN, CASC>::type an;
    an.init(ray, s);
    WriteSink sink{pi.x,  0,           (int)pi.y, (int32_t)(ray_index_base + r), t_starts, t_ends,
                   ray_indices, cells, levels};
    int klk = 0;
    run_kernel<BR, SCH>(an, s, sink, klk);
}

__global__ void raygen_kernel(const CameraDev cam, int64_t first, int64_t n, double* rays) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Ray r = pixel_ray(cam, first + i);
    double2* p = reinterpret_cast<double2*>(rays + 8 * i);
    p[0] = make_double2(r.o[0], r.o[1]);
    p[1] = make_double2(r.o[2], r.d[0]);
    p[2] = make_double2(r.d[1], r.d[2]);
    p[3] = make_double2(r.tmin, r.tmax);
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
template <class Src>
struct Launch {
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t count(const SamplerDev& s, const Src& src, int64_t n, int64_t* packed,
                             int64_t* stats, uint8_t* status, int32_t* counters, uint64_t* tiles,
                             unsigned int* ctr, cudaStream_t st) {
        const int64_t blocks = (n + kBlock - 1) / kBlock;
        count_kernel<AN, CASC, BR, SCH, Src><<<(unsigned)blocks, kBlock, 0, st>>>(
            s, src, n, packed, stats, status, counters, tiles, ctr);
        return cudaGetLastError();
    }
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t write(const SamplerDev& s, const Src& src, int64_t n, const int64_t* packed,
                             int64_t base, double* ts, double* te, int32_t* ri, uint32_t* ce,
                             uint8_t* lv, cudaStream_t st) {
        const int64_t blocks = (n + kBlock - 1) / kBlock;
        write_kernel<AN, CASC, BR, SCH, Src>
            <<<(unsigned)blocks, kBlock, 0, st>>>(s, src, n, packed, base, ts, te, ri, ce, lv);
        return cudaGetLastError();
    }
};

#define SOGK_DISPATCH(FN, ...)                                                                    \
    do {                                                                                          \
        const int key = (v.analyzer << 3) | (v.cascade << 2) | (v.branch << 1) | v.linear;       \
        switch (key) {                                                                            \
            case 0: return L::template FN<0, false, false, 0>(__VA_ARGS__);                       \
            case 1: return L::template FN<0, false, false, 1>(__VA_ARGS__);                       \
            case 2: return L::template FN<0, false, true, 0>(__VA_ARGS__);                        \
            case 3: return L::template FN<0, false, true, 1>(__VA_ARGS__);                        \
            case 4: return L::template FN<0, true, false, 0>(__VA_ARGS__);                        \
            case 5: return L::template FN<0, true, false, 1>(__VA_ARGS__);                        \
            case 6: return L::template FN<0, true, true, 0>(__VA_ARGS__);                         \
            case 7: return L::template FN<0, true, true, 1>(__VA_ARGS__);                         \
            case 8: return L::template FN<1, false, false, 0>(__VA_ARGS__);                       \
            case 9: return L::template FN<1, false, false, 1>(__VA_ARGS__);                       \
            case 10: return L::template FN<1, false, true, 0>(__VA_ARGS__);                       \
            case 11: return L::template FN<1, false, true, 1>(__VA_ARGS__);                       \
            case 12: return L::template FN<1, true, false, 0>(__VA_ARGS__);                       \
            case 13: return L::template FN<1, true, false, 1>(__VA_ARGS__);                       \
            case 14: return L::template FN<1, true, true, 0>(__VA_ARGS__);                        \
            default: return L::template FN<1, true, true, 1>(__VA_ARGS__);                        \
        }                                                                                         \
    } while (0)

// Variant key: analyzer (0 dda / 1 hdda), cascade, kernel == branch, schedule == linear.
cudaError_t launch_count(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, int64_t* packed,
                         int64_t* stats, uint8_t* status, int32_t* counters, uint64_t* tiles,
                         unsigned int* ctr, cudaStream_t st) {
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        SOGK_DISPATCH(count, s, src, n, packed, stats, status, counters, tiles, ctr, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays};
        SOGK_DISPATCH(count, s, src, n, packed, stats, status, counters, tiles, ctr, st);
    }
}

cudaError_t launch_write(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, const int64_t* packed,
                         int64_t base, double* ts, double* te, int32_t* ri, uint32_t* ce,
                         uint8_t* lv, cudaStream_t st) {
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        SOGK_DISPATCH(write, s, src, n, packed, base, ts, te, ri, ce, lv, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays};
        SOGK_DISPATCH(write, s, src, n, packed, base, ts, te, ri, ce, lv, st);
    }
}

cudaError_t launch_raygen(const CameraDev& cam, int64_t first, int64_t n, double* rays,
                          cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    raygen_kernel<<<(unsigned)blocks, 256, 0, st>>>(cam, first, n, rays);
    return cudaGetLastError();
}

} // namespace sogk
