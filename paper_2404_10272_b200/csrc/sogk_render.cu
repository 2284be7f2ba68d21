// sogk_render.cu — the compositing consumer (render.hpp) on the GPU.
//
// composite_kernel: composite_detailed (render.hpp:97-118) for every ray of a packed batch,
//   one thread per ray over its contiguous samples.
// render (sogk_render_camera): render_frame's per-pixel work (bench.hpp:424-461) as
//   pass 1 (count_kernel on camera rays, samples into the per-ray slabs) followed by
//   composite_slab_kernel, which composites each ray straight from its slab row: no scan, no
//   packed sample arrays.  Shading (a loop over every primitive per sample) dominates; done
//   in its own kernel the lanes of a warp shade in step, where interleaving it with the
//   divergent traversal loop measured 4x slower.  Rays whose samples overflowed the slab are
//   finished by render_tail_kernel (slab part, then the resumed traversal, composited).
//
// FP64 with the reference's operation order (Ray::at, density/emission sums in primitive
// order, Vec3 operators); exp() is CUDA's (≤ 1 ulp), not glibc's, so results match the CPU
// within a tolerance, not bit for bit (tests/test_gpu_render.py states it).
#include <cuda_runtime.h>

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

// composite from the run slabs of pass 1 (rays whose runs all fit)
template <int SCH>
__device__ __forceinline__ long long composite_runs(Compositor<SCH>& comp, const SceneDev& sc,
                                                    const Ray& ray, const SamplerDev& s,
                                                    const RunRec* row, int nr, long long fill) {
    for (int j = 0; j < nr; ++j) {
        const RunRec a = row[j];
        const long long start = a.sl & kRunStartMax;
        const long long end = j + 1 < nr ? (long long)(row[j + 1].sl & kRunStartMax) : fill;
        double t = a.first;
        for (long long k = start; k < end; ++k) {
            comp.add(sc, ray, s, t);
            t = t + ladder_step<SCH>(t, s.dt0, s.growth);
        }
    }
    return fill;
}

template <int SCH, class Src>
__global__ void __launch_bounds__(kRenderBlock)
    composite_slab_kernel(const __grid_constant__ SamplerDev s, const SceneDev sc, const Src src,
                          int64_t n, const int64_t* __restrict__ packed, const SlabDev S,
                          double* __restrict__ result, uint8_t* __restrict__ rgb8) {
    const int64_t r = (int64_t)blockIdx.x * kRenderBlock + threadIdx.x;
    if (r >= n) return;
    const long long cnt = __ldg(reinterpret_cast<const longlong2*>(packed) + r).y;
    const int raw = cnt > 0 ? __ldg(S.nruns + r) : 0;
    if (raw < 0) return; // overflowed: render_tail_kernel
    const Ray ray = src.load(r);
    Compositor<SCH> comp;
    comp.init();
    composite_runs<SCH>(comp, sc, ray, s, S.runs + r * S.C, raw, cnt);
    comp.finish(sc, ray, s);
    comp.store(r, result, rgb8);
}

// rays whose runs overflowed the slab: the slab part, then the traversal resumed at the
// first event that did not fit, all composited in order
template <int AN, bool CASC, bool BR, int SCH, class Src>
__global__ void __launch_bounds__(kRenderBlock)
    render_tail_kernel(const __grid_constant__ SamplerDev s, const SceneDev sc, const Src src,
                       const int64_t* __restrict__ packed, const SlabDev S,
                       double* __restrict__ result, uint8_t* __restrict__ rgb8) {
    const unsigned cnt = *S.ovf_ctr;
    for (unsigned i = blockIdx.x * kRenderBlock + threadIdx.x; i < cnt; i += gridDim.x * kRenderBlock) {
        const int64_t r = S.ovf_list[i];
        const long long total = __ldg(reinterpret_cast<const longlong2*>(packed) + r).y;
        Resume res = S.resume[r];
        const long long fill = res.tag >> 8;
        res.tag &= 255;
        const Ray ray = src.load(r);
        Compositor<SCH> comp;
        comp.init();
        long long done = composite_runs<SCH>(comp, sc, ray, s, S.runs + r * S.C,
                                             S.nruns[r] & 0x7fffffff, fill);
        RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
        gen.init(ray, s);
        gen.resume(s, res);
        Run run;
        while (done < total) {
            const int st = gen.step(s, run);
            if (st == 0) break;
            if (st != 2) continue;
            double t = run.first;
            for (int k = 0; k < run.n && done < total; ++k, ++done) {
                comp.add(sc, ray, s, t);
                t = t + ladder_step<SCH>(t, s.dt0, s.growth);
            }
        }
        comp.finish(sc, ray, s);
        comp.store(r, result, rgb8);
    }
}

struct RenderLaunch {
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t tail(const SamplerDev& s, const SceneDev& sc, const RaysFromCamera& src,
                            const int64_t* packed, const SlabDev& S, double* result, uint8_t* rgb8,
                            unsigned grid, cudaStream_t st) {
        render_tail_kernel<AN, CASC, BR, SCH, RaysFromCamera>
            <<<grid, kRenderBlock, 0, st>>>(s, sc, src, packed, S, result, rgb8);
        return cudaGetLastError();
    }
};

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

cudaError_t launch_render_composite(const Variant& v, const SamplerDev& s, const SceneDev& sc,
                                    const CameraDev& cam, int64_t first, int64_t n,
                                    const int64_t* packed, const SlabDev& S, double* result,
                                    uint8_t* rgb8, cudaStream_t st) {
    const RaysFromCamera src{cam, first};
    const unsigned blocks = (unsigned)((n + kRenderBlock - 1) / kRenderBlock);
    if (v.linear)
        composite_slab_kernel<1, RaysFromCamera><<<blocks, kRenderBlock, 0, st>>>(s, sc, src, n, packed, S, result, rgb8);
    else
        composite_slab_kernel<0, RaysFromCamera><<<blocks, kRenderBlock, 0, st>>>(s, sc, src, n, packed, S, result, rgb8);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const unsigned tg = blocks < 148u * 8u ? (blocks ? blocks : 1u) : 148u * 8u;
    using L = RenderLaunch;
    SOGK_DISPATCH(tail, s, sc, src, packed, S, result, rgb8, tg, st);
}

} // namespace sogk
