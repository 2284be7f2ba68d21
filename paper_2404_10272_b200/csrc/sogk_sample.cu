// sogk_sample.cu — K2/K3/K5 sampling kernels and K6 raygen.
//
// Pass 1 (count_kernel): one thread per ray runs the analyzer with the
// reference kernel's control flow (sample_skip / sample_branch over
// Dda/Hdda/CascadeTraversal, sampling.hpp:87-122, 166-196, 305-455), advancing
// the ladder per event in closed form.  It writes the per-ray count, status and
// counters, and the ray's first samples (t, cell, level) into the ray's fixed
// slab; a ray whose runs do not all fit stores the resume state of the first
// run that did not.
// Scan (scan_kernel): packed_info offsets = exclusive scan of the counts.
// Pass 2 (gather_kernel): moves the slabs into the packed arrays, one output
// sample per thread, every store coalesced; tail_kernel resumes the traversal
// only for the rays whose slab overflowed.  write_kernel is the cold path (a
// write with no matching pass 1): it traverses from the ray's start.
// The pass-1 / pass-2 kernels live in sogk_sample_kernels.cuh and are instantiated per
// analyzer in sogk_sample_{dda,hdda,cd}.cu (parallel compilation); this file holds the scan,
// raygen, ray binning and the analyzer dispatch.
#include <cuda_runtime.h>

#include <climits>

#include "sogk_sample_kernels.cuh"

namespace sogk {

// ---------------------------------------------------------------------------
// scan: packed_info[r].offset = exclusive scan of counts (single pass,
// decoupled look-back over 1024-ray tiles, warp-parallel look-back window)
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kScanThreads)
    scan_kernel(int64_t n, int64_t* __restrict__ packed, int64_t* __restrict__ stats,
                uint64_t* __restrict__ tiles, unsigned int* __restrict__ tile_ctr) {
    __shared__ int64_t s_tile;
    __shared__ long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u); // in-order tile ids
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
    long long c[kScanItems];
    long long local = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        c[i] = (base + i < n) ? packed[2 * (base + i) + 1] : 0;
        local += c[i];
    }
    long long agg;
    const long long excl_in = block_excl_scan<kScanThreads>(local, &agg);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        long long excl = 0;
        if (tile == 0) {
            if (lane == 0)
                atomicExch(reinterpret_cast<unsigned long long*>(tiles), kFlagInc | (uint64_t)agg);
        } else {
            if (lane == 0)
                atomicExch(reinterpret_cast<unsigned long long*>(tiles + tile), kFlagAgg | (uint64_t)agg);
            int64_t j = tile - 1; // window [j - 31, j]
            for (;;) {
                const int64_t idx = j - lane;
                uint64_t w = kFlagInc; // tiles before 0 act as an inclusive zero
                if (idx >= 0) {
                    do {
                        w = *reinterpret_cast<volatile uint64_t*>(tiles + idx);
                    } while ((w & ~kValMask) == 0);
                }
                const unsigned inc_mask = __ballot_sync(0xffffffffu, (w & ~kValMask) == kFlagInc);
                const int stop = inc_mask ? __ffs(inc_mask) - 1 : 32; // nearest inclusive predecessor
                long long v = (lane <= stop && idx >= 0) ? (long long)(w & kValMask) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                excl += v;
                if (inc_mask) break;
                j -= 32;
            }
            if (lane == 0)
                atomicExch(reinterpret_cast<unsigned long long*>(tiles + tile),
                           kFlagInc | (uint64_t)(excl + agg));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    long long off = s_excl + excl_in;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) packed[2 * (base + i)] = off;
        off += c[i];
    }
    if (tile == (int64_t)gridDim.x - 1 && threadIdx.x == 0) stats[SOGK_STAT_TOTAL_SAMPLES] = s_excl + agg;
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


cudaError_t launch_scan(int64_t n, int64_t* packed, int64_t* stats, uint64_t* tiles,
                        unsigned int* ctr, cudaStream_t st) {
    const int64_t tiles_n = (n + kScanTile - 1) / kScanTile;
    scan_kernel<<<(unsigned)tiles_n, kScanThreads, 0, st>>>(n, packed, stats, tiles, ctr);
    return cudaGetLastError();
}

int64_t scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }
size_t resume_bytes(int64_t n) { return size_t(n) * sizeof(Resume); }

#define SOGK_AN_DECL(NAME)                                                                         \
    cudaError_t launch_count_##NAME(const Variant&, const SamplerDev&, const double*, const CameraDev*,   \
                                    int64_t, int64_t, int64_t*, int64_t*, uint8_t*, int32_t*,            \
                                    const SlabDev&, cudaStream_t, const uint32_t*);                       \
    cudaError_t launch_write_##NAME(const Variant&, const SamplerDev&, const double*, const CameraDev*,   \
                                    int64_t, int64_t, const int64_t*, const SlabDev*, int64_t, double*,  \
                                    double*, int32_t*, uint32_t*, uint8_t*, cudaStream_t);
SOGK_AN_DECL(dda)
SOGK_AN_DECL(hdda)
SOGK_AN_DECL(cd)
#undef SOGK_AN_DECL

// Variant key: analyzer (0 dda / 1 hdda / 2 cd), then cascade, kernel == branch, schedule == linear
// inside the analyzer's translation unit.
cudaError_t launch_count(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, int64_t* packed,
                         int64_t* stats, uint8_t* status, int32_t* counters, const SlabDev& slab,
                         cudaStream_t st, const uint32_t* perm) {
    switch (v.analyzer) {
        case 0: return launch_count_dda(v, s, rays, cam, first, n, packed, stats, status, counters, slab, st, perm);
        case 1: return launch_count_hdda(v, s, rays, cam, first, n, packed, stats, status, counters, slab, st, perm);
        default: return launch_count_cd(v, s, rays, cam, first, n, packed, stats, status, counters, slab, st, perm);
    }
}

cudaError_t launch_write(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, const int64_t* packed,
                         const SlabDev* slab, int64_t base, double* ts, double* te, int32_t* ri,
                         uint32_t* ce, uint8_t* lv, cudaStream_t st) {
    switch (v.analyzer) {
        case 0: return launch_write_dda(v, s, rays, cam, first, n, packed, slab, base, ts, te, ri, ce, lv, st);
        case 1: return launch_write_hdda(v, s, rays, cam, first, n, packed, slab, base, ts, te, ri, ce, lv, st);
        default: return launch_write_cd(v, s, rays, cam, first, n, packed, slab, base, ts, te, ri, ce, lv, st);
    }
}

// ---------------------------------------------------------------------------
// ray binning (opt-in, SOGK ray order 1): pass 1 processes incoherent rays grouped by where
// they enter the grid and where they head, so that a warp's rays walk nearby nodes in step.
// Key: 8^3 cells of the entry point into the (outermost) grid box x 16^3 direction bins
// (cfg4: 3 % faster than 16^3 x 8^3, 20 % faster than 32^3 x 4^3 -- direction coherence
// matters more than entry position; SOGK_BIN_* select others for experiments);
// counting sort (histogram, scan, atomic scatter).  Only the processing order changes.
// ---------------------------------------------------------------------------
#ifndef SOGK_BIN_CELL
#define SOGK_BIN_CELL 3 // log2 entry-cell bins per axis
#endif
#ifndef SOGK_BIN_DIR
#define SOGK_BIN_DIR 4 // log2 direction bins per axis
#endif
#ifndef SOGK_BIN_DIR_MAJOR
#define SOGK_BIN_DIR_MAJOR 0 // key order: entry cell major (0) or direction major (1)
#endif
constexpr int kBinCell = SOGK_BIN_CELL, kBinDir = SOGK_BIN_DIR;
constexpr int kBinBits = 3 * (kBinCell + kBinDir);

__device__ __forceinline__ uint32_t bin_key(const Ray& r, const GridDev& g) {
    double lo[3], hi[3], te, tx;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = g.wmin[a];
        hi[a] = g.wmin[a] + (double)g.res[a] * g.voxel;
    }
    constexpr double nc = double(1 << kBinCell), nd = double(1 << kBinDir);
    uint32_t c[3] = {0, 0, 0};
    if (clip_to_box(r, lo, hi, te, tx)) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double u = (r.o[a] + r.d[a] * te - lo[a]) / (hi[a] - lo[a]) * nc;
            c[a] = (uint32_t)(u < 0.0 ? 0.0 : (u > nc - 1.0 ? nc - 1.0 : u));
        }
    }
    uint32_t d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double u = (r.d[a] + 1.0) * (0.5 * nd);
        d[a] = (uint32_t)(u < 0.0 ? 0.0 : (u > nd - 1.0 ? nd - 1.0 : u));
    }
    const uint32_t ck = (((c[0] << kBinCell) | c[1]) << kBinCell) | c[2];
    const uint32_t dk = (((d[0] << kBinDir) | d[1]) << kBinDir) | d[2];
    return SOGK_BIN_DIR_MAJOR ? (dk << (3 * kBinCell)) | ck : (ck << (3 * kBinDir)) | dk;
}

__global__ void bin_count_kernel(const SamplerDev s, const double* rays, int64_t n, uint32_t* keys,
                                 unsigned long long* hist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = bin_key(RaysFromBuffer{rays}.load(i), s.lv[s.n_levels - 1]);
    keys[i] = k;
    atomicAdd(hist + 2 * k + 1, 1ull);
}

__global__ void bin_scatter_kernel(int64_t n, const uint32_t* keys, unsigned long long* hist,
                                   uint32_t* perm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    perm[atomicAdd(hist + 2 * keys[i], 1ull)] = (uint32_t)i;
}

size_t bin_scratch_bytes(int64_t n) {
    const int64_t bins = int64_t(1) << kBinBits;
    return size_t(n) * 8 + size_t(bins) * 16 + size_t(scan_tiles(bins)) * 8 + 256;
}

cudaError_t launch_ray_binning(const SamplerDev& s, const double* rays, int64_t n, void* scratch,
                               uint32_t** perm_out, cudaStream_t st) {
    const int64_t bins = int64_t(1) << kBinBits;
    char* p = static_cast<char*>(scratch);
    uint32_t* keys = reinterpret_cast<uint32_t*>(p);
    uint32_t* perm = keys + n;
    int64_t* hist = reinterpret_cast<int64_t*>(p + size_t(n) * 8);
    uint64_t* tiles = reinterpret_cast<uint64_t*>(hist + 2 * bins);
    int64_t* stats = reinterpret_cast<int64_t*>(tiles + scan_tiles(bins) + 1);
    cudaError_t e = cudaMemsetAsync(hist, 0, size_t(bins) * 16 + size_t(scan_tiles(bins)) * 8 + 256, st);
    if (e != cudaSuccess) return e;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    bin_count_kernel<<<blocks, 256, 0, st>>>(s, rays, n, keys, reinterpret_cast<unsigned long long*>(hist));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    e = launch_scan(bins, hist, stats, tiles, reinterpret_cast<unsigned int*>(tiles + scan_tiles(bins)), st);
    if (e != cudaSuccess) return e;
    bin_scatter_kernel<<<blocks, 256, 0, st>>>(n, keys, reinterpret_cast<unsigned long long*>(hist), perm);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *perm_out = perm;
    return cudaSuccess;
}

__global__ void add_offset_kernel(int64_t* packed, int64_t n, int64_t base) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) packed[2 * i] += base;
}

cudaError_t launch_add_offset(int64_t* packed, int64_t n, int64_t base, cudaStream_t st) {
    if (n <= 0 || base == 0) return cudaSuccess;
    add_offset_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(packed, n, base);
    return cudaGetLastError();
}

cudaError_t launch_raygen(const CameraDev& cam, int64_t first, int64_t n, double* rays,
                          cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    raygen_kernel<<<(unsigned)blocks, 256, 0, st>>>(cam, first, n, rays);
    return cudaGetLastError();
}

} // namespace sogk
