// sogk_traverse.cu — the analyzers' event streams over a ray batch (the reference's
// traverse entry points: DdaTraversal / HddaTraversal / CdTraversal / CascadeTraversal
// next() drained by collect_events, traversal.hpp:120-359, sampling.hpp:305-415) and the
// point queries (SparseGrid::query, sparse.hpp:163-171; DenseGrid::voxel_at, grid.hpp:129-133).
//
// Two passes like the sampler: traverse_kernel<count> writes per-ray event counts (then the
// shared decoupled look-back scan turns them into offsets), traverse_kernel<write> walks the
// rays again and writes each event at its offset.  The analyzers are the sampler's own
// (sogk_device.cuh), so event boundaries, cells and counters are bit-identical to what the
// samplers consume.
#include <cuda_runtime.h>

#include "sogk_device.cuh"
#include "sogk_internal.h"
#include "sogk_sources.cuh"

namespace sogk {

constexpr int kTraverseBlock = kGeomBlock; // node analyzers keep per-thread smem columns

template <int AN, bool CASC, bool WRITE>
__global__ void __launch_bounds__(kTraverseBlock)
    traverse_kernel(const __grid_constant__ SamplerDev s, const double* __restrict__ rays, int64_t n,
                    int64_t* __restrict__ info, int64_t* __restrict__ stats, uint8_t* __restrict__ status,
                    int32_t* __restrict__ counters, sogk_event* __restrict__ events) {
    const int64_t r = (int64_t)blockIdx.x * kTraverseBlock + threadIdx.x;
    long long cnt = 0, lk = 0, sp = 0, inv = 0, und = 0;
    if (r < n) {
        const Ray ray = RaysFromBuffer{rays}.load(r);
        int sta = SOGK_RAY_OK;
        if (!ray_valid(ray)) { // sog::Ray's constructor would throw (ray.hpp:98-106)
            sta = SOGK_RAY_INVALID;
            inv = 1;
        } else {
            typename PickAn<AN, CASC>::type an;
            an.init(ray, s);
            long long base = 0, cap = 0;
            if (WRITE) { // only the counted events: a ray the count flagged (spin) has none
                const longlong2 pi = reinterpret_cast<const longlong2*>(info)[r];
                base = pi.x;
                cap = pi.y;
            }
            for (;;) { // collect_events: next() until the stream ends
                if (WRITE && cnt >= cap) break;
                Event ev;
                const int got = an.next(s, ev);
                if (got == 0) break;
                if (got < 0) continue;
                if (WRITE) {
                    sogk_event e;
                    e.ijk[0] = ev.ijk[0];
                    e.ijk[1] = ev.ijk[1];
                    e.ijk[2] = ev.ijk[2];
                    e.level = ev.level;
                    e.t0 = ev.t0;
                    e.t1 = ev.t1;
                    e.occupied = ev.occ ? 1 : 0;
                    e.grid_level = ev.grid_level;
                    events[base + cnt] = e;
                }
                ++cnt;
            }
            if (an.undefined()) { // the reference's next() never returns on this ray
                sta = SOGK_RAY_UNDEFINED;
                cnt = 0;
                und = 1;
            } else {
                lk = an.lookups();
                sp = an.steps();
            }
        }
        if (!WRITE) {
            reinterpret_cast<longlong2*>(info)[r] = make_longlong2(0, cnt);
            if (status) status[r] = (uint8_t)sta;
            if (counters) {
                counters[2 * r] = (int32_t)lk;
                counters[2 * r + 1] = (int32_t)sp;
            }
        }
    }
    if constexpr (!WRITE) { // warp sums into the stats block
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lk += __shfl_xor_sync(0xffffffffu, lk, o);
            sp += __shfl_xor_sync(0xffffffffu, sp, o);
            inv += __shfl_xor_sync(0xffffffffu, inv, o);
            und += __shfl_xor_sync(0xffffffffu, und, o);
        }
        if ((threadIdx.x & 31) == 0) {
            unsigned long long* S = reinterpret_cast<unsigned long long*>(stats);
            if (inv) atomicAdd(S + SOGK_STAT_INVALID_RAYS, (unsigned long long)inv);
            if (und) atomicAdd(S + SOGK_STAT_UNDEFINED_RAYS, (unsigned long long)und);
            if (lk) atomicAdd(S + SOGK_STAT_ANALYZER_LOOKUPS, (unsigned long long)lk);
            if (sp) atomicAdd(S + SOGK_STAT_ANALYZER_STEPS, (unsigned long long)sp);
        }
    }
}

template <bool WRITE>
static cudaError_t launch_traverse_impl(const Variant& v, const SamplerDev& s, const double* rays, int64_t n,
                                        int64_t* info, int64_t* stats, uint8_t* status, int32_t* counters,
                                        sogk_event* events, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + kTraverseBlock - 1) / kTraverseBlock);
#define SOGK_TRAV(A, C)                                                                               \
    traverse_kernel<A, C, WRITE><<<blocks, kTraverseBlock, 0, st>>>(s, rays, n, info, stats, status,  \
                                                                    counters, events)
    const int key = v.analyzer * 2 + (v.cascade ? 1 : 0);
    switch (key) {
        case 0: SOGK_TRAV(0, false); break;
        case 1: SOGK_TRAV(0, true); break;
        case 2: SOGK_TRAV(1, false); break;
        case 3: SOGK_TRAV(1, true); break;
        case 4: SOGK_TRAV(2, false); break;
        default: SOGK_TRAV(2, true); break;
    }
#undef SOGK_TRAV
    return cudaGetLastError();
}

cudaError_t launch_traverse_count(const Variant& v, const SamplerDev& s, const double* rays, int64_t n,
                                  int64_t* info, int64_t* stats, uint8_t* status, int32_t* counters,
                                  cudaStream_t st) {
    return launch_traverse_impl<false>(v, s, rays, n, info, stats, status, counters, nullptr, st);
}

cudaError_t launch_traverse_write(const Variant& v, const SamplerDev& s, const double* rays, int64_t n,
                                  const int64_t* info, sogk_event* events, cudaStream_t st) {
    return launch_traverse_impl<true>(v, s, rays, n, const_cast<int64_t*>(info), nullptr, nullptr, nullptr,
                                      events, st);
}

// SparseGrid::query (sparse.hpp:163-171) / DenseGrid::voxel_at (grid.hpp:129-133) per point
__global__ void query_kernel(const GridDev g, int vdb, const int32_t* __restrict__ ijk, int64_t n,
                             sogk_query* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int p[3] = {__ldg(ijk + 3 * i), __ldg(ijk + 3 * i + 1), __ldg(ijk + 3 * i + 2)};
    sogk_query q;
    if (vdb) {
        VdbCursor c;
        c.reset();
        const Query a = c.query(g, p);
        q.occupied = a.occ ? 1 : 0;
        q.level = a.level;
        q.extent = a.ext;
        // every answer is aligned to its extent; out of bounds: region_origin = floor_div(ijk, 128) * 128
        q.origin[0] = p[0] & -a.ext;
        q.origin[1] = p[1] & -a.ext;
        q.origin[2] = p[2] & -a.ext;
    } else {
        q.occupied = dense_voxel(g, p) ? 1 : 0;
        q.level = LV_VOXEL;
        q.extent = 1;
        q.origin[0] = p[0];
        q.origin[1] = p[1];
        q.origin[2] = p[2];
    }
    out[i] = q;
}

cudaError_t launch_query(const GridDev& g, int vdb, const int32_t* ijk, int64_t n, sogk_query* out,
                         cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    query_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, vdb, ijk, n, out);
    return cudaGetLastError();
}

} // namespace sogk
