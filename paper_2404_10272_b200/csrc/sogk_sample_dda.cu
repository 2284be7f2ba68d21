// sogk_sample_dda.cu — the DDA analyzer's pass-1 / pass-2 kernels (8 variants: cascade x
// kernel x schedule), one translation unit per analyzer so the build compiles them in parallel.
#include "sogk_sample_kernels.cuh"

namespace sogk {

cudaError_t launch_count_dda(const Variant& v, const SamplerDev& s, const double* rays, const CameraDev* cam,
                            int64_t first, int64_t n, int64_t* packed, int64_t* stats, uint8_t* status,
                            int32_t* counters, const SlabDev& slab, cudaStream_t st, const uint32_t* perm) {
    return launch_count_an<0>(v, s, rays, cam, first, n, packed, stats, status, counters, slab, st, perm);
}

cudaError_t launch_write_dda(const Variant& v, const SamplerDev& s, const double* rays, const CameraDev* cam,
                            int64_t first, int64_t n, const int64_t* packed, const SlabDev* slab, int64_t base,
                            double* ts, double* te, int32_t* ri, uint32_t* ce, uint8_t* lv, cudaStream_t st) {
    return launch_write_an<0>(v, s, rays, cam, first, n, packed, slab, base, ts, te, ri, ce, lv, st);
}

} // namespace sogk
