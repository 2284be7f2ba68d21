// sogk_sources.cuh — ray sources of the sampling kernels and the analyzer selection.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "sogk_device.cuh"
#include "sogk_internal.h"

namespace sogk {

// ---------------------------------------------------------------------------
// ray sources
// ---------------------------------------------------------------------------
struct RaysFromBuffer {
    const double* rays;
    const uint32_t* perm = nullptr; // processing order (ray binning), nullptr: as given
    // the ray a thread of pass 1 processes: every output stays indexed by this id
    __device__ __forceinline__ int64_t id(int64_t j) const { return perm ? (int64_t)__ldg(perm + j) : j; }
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
    __device__ __forceinline__ int64_t id(int64_t j) const { return j; }
    __device__ __forceinline__ Ray load(int64_t i) const { return pixel_ray(cam, first + i); }
};

// ONE: the HDDA query's single-region mode (VdbCursor::query): the count kernel is compiled for
// single-region grids (1) and for the rest (0); other kernels decide at run time (-1)
template <int AN, bool CASC, int ONE = -1>
struct PickAn {
    using Sub = typename std::conditional<
        AN == SOGK_HDDA, NodeAn<false, ONE>, typename std::conditional<AN == SOGK_CD, CdAn, DdaAn>::type>::type;
    using type = AnyAn<Sub, CASC>;
};

} // namespace sogk
