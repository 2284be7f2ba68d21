// sogk_render.cu — the compositing consumer (render.hpp) on the GPU.
//
// composite_kernel: composite_detailed (render.hpp:97-118) for every ray of a packed batch,
//   one thread per ray over its contiguous samples.
// render_kernel:    render_frame's per-pixel work (bench.hpp:424-461) fused: the pixel's ray
//   is generated (Camera::pixel_ray), sampled with pass 1's loop and composited sample by
//   sample in registers; no sample ever reaches HBM.
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

// AnalyticScene::density_at / emission_at (render.hpp:72-91) at p, one pass over the
// primitives in order (both sums run in the same order as the reference's two loops)
__device__ __forceinline__ double scene_at(const SceneDev& sc, const double p[3], double e[3]) {
    double sigma = 0.0;
    e[0] = e[1] = e[2] = 0.0;
    for (int i = 0; i < sc.n; ++i) {
        const sogk_primitive& q = sc.prims[i]; // warp-uniform: one broadcast per field
        bool in;
        if (q.shape == SOGK_SPHERE) { // Primitive::contains (render.hpp:44-51)
            const double dx = p[0] - q.center[0], dy = p[1] - q.center[1], dz = p[2] - q.center[2];
            in = dx * dx + dy * dy + dz * dz <= q.radius * q.radius;
        } else {
            in = p[0] >= q.lo[0] && p[1] >= q.lo[1] && p[2] >= q.lo[2] && p[0] < q.hi[0] &&
                 p[1] < q.hi[1] && p[2] < q.hi[2];
        }
        if (in) {
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

template <int AN, bool CASC, bool BR, int SCH, class Src>
__global__ void __launch_bounds__(kRenderBlock)
    render_kernel(const __grid_constant__ SamplerDev s, const SceneDev sc, const Src src, int64_t n,
                  int64_t* __restrict__ stats, double* __restrict__ result,
                  uint8_t* __restrict__ rgb8) {
    const int64_t r = (int64_t)blockIdx.x * kRenderBlock + threadIdx.x;
    long long smp = 0, lk = 0, sp = 0, klk = 0, und = 0;
    if (r < n) {
        const Ray ray = src.load(r);
        Compositor<SCH> comp;
        comp.init();
        if (ray_valid(ray)) {
            RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
            gen.init(ray, s);
            for (;;) { // pass 1's loop, the samples go to the compositor
                Event ev;
                double t_last0;
                const int st = gen.step_event(s, ev, t_last0);
                if (st == 0) break;
                if (st == 1) continue;
                double t = gen.t_last;
                int k = 0;
                bool stuck = false;
                while (t <= ev.t1) { // while (t <= t1) { push(t); t += step(t); }
                    comp.add(sc, ray, s, t);
                    const double tn = t + ladder_step<SCH>(t, s.dt0, s.growth);
                    ++k;
                    if (!(tn > t)) { // t + step == t: the reference loops forever
                        stuck = true;
                        break;
                    }
                    t = tn;
                }
                gen.t_last = t;
                if (stuck) {
                    gen.stalled = true;
                    break;
                }
                if (BR) gen.kernel_lookups += k;
                smp += k;
            }
            if (gen.undefined()) { // the reference never returns: no samples, like pass 1
                comp.init();
                smp = 0;
                und = 1;
            } else {
                lk = gen.an.lookups();
                sp = gen.an.steps();
                klk = gen.kernel_lookups;
            }
        }
        comp.finish(sc, ray, s);
        comp.store(r, result, rgb8);
    }
    if (stats) { // warp-level reduction, one atomic per warp and counter
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            smp += __shfl_xor_sync(0xffffffffu, smp, o);
            lk += __shfl_xor_sync(0xffffffffu, lk, o);
            sp += __shfl_xor_sync(0xffffffffu, sp, o);
            klk += __shfl_xor_sync(0xffffffffu, klk, o);
            und += __shfl_xor_sync(0xffffffffu, und, o);
        }
        if ((threadIdx.x & 31) == 0) {
            unsigned long long* S = reinterpret_cast<unsigned long long*>(stats);
            if (smp) atomicAdd(S + SOGK_STAT_TOTAL_SAMPLES, (unsigned long long)smp);
            if (lk) atomicAdd(S + SOGK_STAT_ANALYZER_LOOKUPS, (unsigned long long)lk);
            if (sp) atomicAdd(S + SOGK_STAT_ANALYZER_STEPS, (unsigned long long)sp);
            if (klk) atomicAdd(S + SOGK_STAT_KERNEL_LOOKUPS, (unsigned long long)klk);
            if (und) atomicAdd(S + SOGK_STAT_UNDEFINED_RAYS, (unsigned long long)und);
        }
    }
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

struct RenderLaunch {
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t render(const SamplerDev& s, const SceneDev& sc, const RaysFromCamera& src,
                              int64_t n, int64_t* stats, double* result, uint8_t* rgb8,
                              cudaStream_t st) {
        const unsigned blocks = (unsigned)((n + kRenderBlock - 1) / kRenderBlock);
        render_kernel<AN, CASC, BR, SCH, RaysFromCamera>
            <<<blocks, kRenderBlock, 0, st>>>(s, sc, src, n, stats, result, rgb8);
        return cudaGetLastError();
    }
};

cudaError_t launch_render(const Variant& v, const SamplerDev& s, const SceneDev& sc,
                          const CameraDev& cam, int64_t first, int64_t n, int64_t* stats,
                          double* result, uint8_t* rgb8, cudaStream_t st) {
    using L = RenderLaunch;
    const RaysFromCamera src{cam, first};
    SOGK_DISPATCH(render, s, sc, src, n, stats, result, rgb8, st);
}

} // namespace sogk
