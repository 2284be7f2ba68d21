// sogk_render.cu — the compositing consumer (render.hpp) on the GPU.
//
// composite_kernel: composite_detailed (render.hpp:97-118) for every ray of a packed batch,
//   one thread per ray over its contiguous samples.
// render (sogk_render_camera): render_frame's per-pixel work (bench.hpp:424-461) as pass 1 +
//   scan + pass 2 on the camera rays, then shade_kernel (per sample, all samples of the frame
//   in parallel) and accumulate_kernel (per ray, the reference's sequential sums).  Shading (a
//   loop over the candidate primitives and an exp per sample) dominates; interleaved with the
//   divergent traversal loop it ran 4x slower, and thread-per-ray compositing made every warp
//   wait on its longest ray.
//
// FP64 with the reference's operation order (Ray::at, density/emission sums in primitive
// order, Vec3 operators); exp() is CUDA's (≤ 1 ulp), not glibc's, so results match the CPU
// within a tolerance, not bit for bit (tests/test_gpu_render.py states it).
#include <cuda_runtime.h>

#include <algorithm>

#include "sogk_device.cuh"
#include "sogk_internal.h"
#include "sogk_sources.cuh"

namespace sogk {

constexpr int kRenderBlock = 128;

__device__ __forceinline__ bool prim_contains(const sogk_primitive& q, const double p[3]) {
    if (q.shape == SOGK_SPHERE) { // Primitive::contains (render.hpp:44-51)
        const double dx = p[0] - q.center[0], dy = p[1] - q.center[1], dz = p[2] - q.center[2];
        return dx * dx + dy * dy + dz * dz <= q.radius * q.radius;
    }
    return p[0] >= q.lo[0] && p[1] >= q.lo[1] && p[2] >= q.lo[2] && p[0] < q.hi[0] &&
           p[1] < q.hi[1] && p[2] < q.hi[2];
}

// AnalyticScene::density_at / emission_at (render.hpp:72-91) at p, one pass over the
// primitives in order (both sums run in the same order as the reference's two loops).
// With the candidate grid only the primitives listed for p's cell are tested: every other
// primitive's (grown) box misses the cell, so it cannot contain p, and the list keeps
// index order -- the sums are the reference's.
__device__ __forceinline__ double scene_at(const SceneDev& sc, const double p[3], double e[3]) {
    double sigma = 0.0;
    e[0] = e[1] = e[2] = 0.0;
    int i0 = 0, i1 = sc.n;
    const int* list = nullptr;
    if (sc.gres > 0) {
        int c[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double g = (p[a] - sc.glo[a]) * sc.ginv;
            if (!(g > -1.0 && g < (double)(sc.gres + 1))) return 0.0; // outside every box
            const int ci = (int)floor(g);
            c[a] = ci < 0 ? 0 : (ci >= sc.gres ? sc.gres - 1 : ci);
        }
        const int cell = (c[2] * sc.gres + c[1]) * sc.gres + c[0];
        i0 = __ldg(sc.cstart + cell);
        i1 = __ldg(sc.cstart + cell + 1);
        list = sc.cand;
    }
    for (int k = i0; k < i1; ++k) {
        const sogk_primitive& q = sc.prims[list ? __ldg(list + k) : k];
        if (prim_contains(q, p)) {
            e[0] += q.color[0] * q.density;
            e[1] += q.color[1] * q.density;
            e[2] += q.color[2] * q.density;
            sigma += q.density;
        }
    }
    return sigma;
}

// composite_detailed's accumulator; a sample is shaded once its successor (its dt) is known
template <int SCH>
struct Compositor {
    double c[3], ws, T;
    double pt;
    bool pending;

    __device__ __forceinline__ void init() {
        c[0] = c[1] = c[2] = 0.0;
        ws = 0.0;
        T = 1.0;
        pending = false;
    }
    __device__ __forceinline__ void shade(const SceneDev& sc, const Ray& ray, double t, double dt) {
        double p[3], e[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) p[a] = ray.o[a] + ray.d[a] * t; // Ray::at (ray.hpp:35)
        const double sigma = scene_at(sc, p, e);
        if (sigma <= 0.0) return;
        const double alpha = 1.0 - exp(-sigma * dt);
        const double w = T * alpha;
#pragma unroll
        for (int a = 0; a < 3; ++a) c[a] += (e[a] / sigma) * w; // emission_at(p) * w
        ws += w;
        T *= 1.0 - alpha;
    }
    __device__ __forceinline__ void add(const SceneDev& sc, const Ray& ray, const SamplerDev& s,
                                        double t) {
        if (pending) shade(sc, ray, pt, t - pt); // samples[i + 1] - t (render.hpp:106)
        pt = t;
        pending = true;
    }
    __device__ __forceinline__ void finish(const SceneDev& sc, const Ray& ray, const SamplerDev& s) {
        if (pending) shade(sc, ray, pt, ladder_step<SCH>(pt, s.dt0, s.growth)); // sched.step(t)
        pending = false;
#pragma unroll
        for (int a = 0; a < 3; ++a) c[a] += sc.bg[a] * T; // background * transmittance
    }
    __device__ __forceinline__ void store(int64_t r, double* result, uint8_t* rgb8) const {
        if (result) {
            double* o = result + 5 * r;
            o[0] = c[0];
            o[1] = c[1];
            o[2] = c[2];
            o[3] = ws;
            o[4] = T;
        }
        if (rgb8) { // Image::set_pixel (render.hpp:133-139)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double lo = (0.0 < c[a]) ? c[a] : 0.0; // std::max(0.0, v)
                const double v = (lo < 1.0) ? lo : 1.0;      // std::min(1.0, .)
                rgb8[3 * r + a] = (uint8_t)llround(v * 255.0);
            }
        }
    }
};

template <int SCH>
__global__ void __launch_bounds__(kRenderBlock)
    composite_kernel(const __grid_constant__ SamplerDev s, const SceneDev sc, const double* rays,
                     int64_t n, const int64_t* __restrict__ packed, const double* __restrict__ ts,
                     double* __restrict__ result, uint8_t* __restrict__ rgb8) {
    const int64_t r = (int64_t)blockIdx.x * kRenderBlock + threadIdx.x;
    if (r >= n) return;
    const Ray ray = RaysFromBuffer{rays}.load(r);
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
    Compositor<SCH> comp;
    comp.init();
    for (long long k = 0; k < pi.y; ++k) comp.add(sc, ray, s, __ldg(ts + pi.x + k));
    comp.finish(sc, ray, s);
    comp.store(r, result, rgb8);
}

// ---------------------------------------------------------------------------
// render in three data-parallel steps after pass 1 + scan + gather (t_starts, ray_indices):
//   shade_kernel:      per sample (all samples of the frame in parallel): alpha and the
//                      emission colour (emission_at(p) = e / sigma); sigma <= 0 marked skip
//   accumulate_kernel: per ray, the reference's sequential front-to-back sums over them
// The arithmetic is the compositor's, operation for operation, so frames are bit-identical
// to composite_kernel's; shading no longer waits on the longest ray of a warp.
// ---------------------------------------------------------------------------
template <int SCH>
__global__ void __launch_bounds__(kRenderBlock)
    shade_kernel(const __grid_constant__ SamplerDev s, const SceneDev sc, const double* rays,
                 const int64_t* __restrict__ d_total, const int64_t* __restrict__ packed,
                 const double* __restrict__ ts, const int32_t* __restrict__ ri,
                 int64_t ray_index_base, double4* __restrict__ shaded) {
    // grid-stride over the frame's samples; the total comes from pass 1 on the device, so the
    // host never waits for it
    const int64_t total = *d_total;
    for (int64_t e = (int64_t)blockIdx.x * kRenderBlock + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * kRenderBlock) {
    const int64_t r = __ldg(ri + e) - ray_index_base;
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
    const double t = __ldg(ts + e);
    // samples[i + 1] - t, or sched.step(t) for the ray's last sample (render.hpp:106)
    const double dt = e + 1 < pi.x + pi.y ? __ldg(ts + e + 1) - t : ladder_step<SCH>(t, s.dt0, s.growth);
    const Ray ray = RaysFromBuffer{rays}.load(r);
    double p[3], em[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = ray.o[a] + ray.d[a] * t; // Ray::at (ray.hpp:35)
    const double sigma = scene_at(sc, p, em);
    double4 out;
    if (sigma <= 0.0) {
        out = make_double4(-1.0, 0.0, 0.0, 0.0); // skipped (render.hpp:109)
    } else {
        out = make_double4(1.0 - exp(-sigma * dt), em[0] / sigma, em[1] / sigma, em[2] / sigma);
    }
    shaded[e] = out;
    }
}

__global__ void __launch_bounds__(kRenderBlock)
    accumulate_kernel(const SceneDev sc, int64_t n, const int64_t* __restrict__ packed,
                      const double4* __restrict__ shaded, double* __restrict__ result,
                      uint8_t* __restrict__ rgb8) {
    const int64_t r = (int64_t)blockIdx.x * kRenderBlock + threadIdx.x;
    if (r >= n) return;
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
    Compositor<0> comp;
    comp.init();
    for (long long k = 0; k < pi.y; ++k) {
        const double4 v = shaded[pi.x + k];
        if (v.x < 0.0) continue; // sigma <= 0
        const double alpha = v.x;
        const double w = comp.T * alpha;
        comp.c[0] += v.y * w;
        comp.c[1] += v.z * w;
        comp.c[2] += v.w * w;
        comp.ws += w;
        comp.T *= 1.0 - alpha;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) comp.c[a] += sc.bg[a] * comp.T; // background * transmittance
    comp.store(r, result, rgb8);
}

cudaError_t launch_shade_accumulate(const Variant& v, const SamplerDev& s, const SceneDev& sc,
                                    const double* rays, int64_t n, const int64_t* packed,
                                    const double* ts, const int32_t* ri, const int64_t* d_total,
                                    int64_t total_hint, int64_t ray_index_base, void* shaded,
                                    double* result, uint8_t* rgb8, cudaStream_t st) {
    if (total_hint > 0) {
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (sms <= 0) sms = 148;
        }
        const int64_t want = (total_hint + kRenderBlock - 1) / kRenderBlock;
        const unsigned blocks = (unsigned)std::min<int64_t>(want, int64_t(sms) * 16);
        if (v.linear)
            shade_kernel<1><<<blocks, kRenderBlock, 0, st>>>(s, sc, rays, d_total, packed, ts, ri,
                                                            ray_index_base, static_cast<double4*>(shaded));
        else
            shade_kernel<0><<<blocks, kRenderBlock, 0, st>>>(s, sc, rays, d_total, packed, ts, ri,
                                                            ray_index_base, static_cast<double4*>(shaded));
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    accumulate_kernel<<<(unsigned)((n + kRenderBlock - 1) / kRenderBlock), kRenderBlock, 0, st>>>(
        sc, n, packed, static_cast<const double4*>(shaded), result, rgb8);
    return cudaGetLastError();
}

cudaError_t launch_composite(const Variant& v, const SamplerDev& s, const SceneDev& sc,
                             const double* rays, int64_t n, const int64_t* packed, const double* ts,
                             double* result, uint8_t* rgb8, cudaStream_t st) {
    const unsigned blocks = (unsigned)((n + kRenderBlock - 1) / kRenderBlock);
    if (v.linear)
        composite_kernel<1><<<blocks, kRenderBlock, 0, st>>>(s, sc, rays, n, packed, ts, result, rgb8);
    else
        composite_kernel<0><<<blocks, kRenderBlock, 0, st>>>(s, sc, rays, n, packed, ts, result, rgb8);
    return cudaGetLastError();
}

} // namespace sogk
