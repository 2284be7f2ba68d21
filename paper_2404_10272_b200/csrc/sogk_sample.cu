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
#include <cuda_runtime.h>

#include <climits>

#include "sogk_device.cuh"
#include "sogk_internal.h"
#include "sogk_sources.cuh"

namespace sogk {

constexpr int kBlock = 128;
constexpr int kWriteBlock = 128;
#ifndef SOGK_CASC_MINB
#define SOGK_CASC_MINB 1 // the same for the cascade variants
#endif
#ifndef SOGK_COUNT_MINB
#define SOGK_COUNT_MINB 1 // pass-1 min resident blocks per SM (register cap), A/B-tunable
#endif

// ---------------------------------------------------------------------------
// warp / block scans
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long warp_incl_scan(long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

__device__ __forceinline__ int warp_incl_scan_i(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// exclusive prefix of v within the block; *total = block sum
template <int Threads>
__device__ __forceinline__ long long block_excl_scan(long long v, long long* total) {
    __shared__ long long warp_tot[Threads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long incl = warp_incl_scan(v);
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long w = lane < Threads / 32 ? warp_tot[lane] : 0;
        w = warp_incl_scan(w);
        if (lane < Threads / 32) warp_tot[lane] = w;
    }
    __syncthreads();
    const long long before = wid > 0 ? warp_tot[wid - 1] : 0;
    *total = warp_tot[Threads / 32 - 1];
    __syncthreads();
    return before + incl - v;
}

template <int Threads>
__device__ __forceinline__ long long block_sum(long long v) {
    long long t;
    block_excl_scan<Threads>(v, &t);
    return t;
}

// resume state at `run`; tag bits 8.. carry the number of samples already in the slab
__device__ __forceinline__ void store_resume(Resume* dst, const Run& run, int filled) {
    Resume r;
    r.ijk[0] = run.ijk[0];
    r.ijk[1] = run.ijk[1];
    r.ijk[2] = run.ijk[2];
    r.tag = run.tag | (filled << 8);
    r.t_cur = run.t0;
    r.t_last = run.t_last0;
    *dst = r;
}

// ---------------------------------------------------------------------------
// pass 1: per-ray counts, status, counters, resume state
// ---------------------------------------------------------------------------
struct Stats5 {
    long long inv = 0, und = 0, lk = 0, sp = 0, klk = 0, ovf = 0, smp = 0;
    __device__ __forceinline__ void flush(int64_t* stats) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            inv += __shfl_xor_sync(0xffffffffu, inv, o);
            und += __shfl_xor_sync(0xffffffffu, und, o);
            lk += __shfl_xor_sync(0xffffffffu, lk, o);
            sp += __shfl_xor_sync(0xffffffffu, sp, o);
            klk += __shfl_xor_sync(0xffffffffu, klk, o);
            ovf += __shfl_xor_sync(0xffffffffu, ovf, o);
            smp += __shfl_xor_sync(0xffffffffu, smp, o);
        }
        if ((threadIdx.x & 31) == 0) {
            unsigned long long* S = reinterpret_cast<unsigned long long*>(stats);
            if (inv) atomicAdd(S + SOGK_STAT_INVALID_RAYS, (unsigned long long)inv);
            if (und) atomicAdd(S + SOGK_STAT_UNDEFINED_RAYS, (unsigned long long)und);
            if (lk) atomicAdd(S + SOGK_STAT_ANALYZER_LOOKUPS, (unsigned long long)lk);
            if (sp) atomicAdd(S + SOGK_STAT_ANALYZER_STEPS, (unsigned long long)sp);
            if (klk) atomicAdd(S + SOGK_STAT_KERNEL_LOOKUPS, (unsigned long long)klk);
            if (ovf) atomicAdd(S + SOGK_STAT_SLAB_OVERFLOW_RAYS, (unsigned long long)ovf);
            // the scan (when it runs) overwrites the total with the same value
            if (smp) atomicAdd(S + SOGK_STAT_TOTAL_SAMPLES, (unsigned long long)smp);
        }
    }
};

// finish one ray of pass 1: status, counters, count (offset filled by the scan)
template <class Gen>
__device__ __forceinline__ void count_finish(const Gen& gen, long long r, long long cnt,
                                             int64_t* packed, uint8_t* status, int32_t* counters,
                                             Stats5& acc) {
    int sta = SOGK_RAY_OK, lk = 0, sp = 0, klk = 0;
    if (gen.undefined()) {
        sta = SOGK_RAY_UNDEFINED;
        cnt = 0;
        ++acc.und;
    } else {
        lk = gen.an.lookups();
        sp = gen.an.steps();
        klk = gen.kernel_lookups;
    }
    if (status) status[r] = (uint8_t)sta;
    if (counters) {
        counters[3 * r] = lk;
        counters[3 * r + 1] = sp;
        counters[3 * r + 2] = klk;
    }
    reinterpret_cast<longlong2*>(packed)[r] = make_longlong2(0, cnt);
    acc.smp += cnt;
    acc.lk += lk;
    acc.sp += sp;
    acc.klk += klk;
}

__device__ __forceinline__ void count_invalid(long long r, int64_t* packed, uint8_t* status,
                                              int32_t* counters, Stats5& acc) {
    ++acc.inv; // sog::Ray would throw (ray.hpp:98-106)
    if (status) status[r] = SOGK_RAY_INVALID;
    if (counters) {
        counters[3 * r] = 0;
        counters[3 * r + 1] = 0;
        counters[3 * r + 2] = 0;
    }
    reinterpret_cast<longlong2*>(packed)[r] = make_longlong2(0, 0);
}


// ---------------------------------------------------------------------------
// pass 1: per-ray counts, status, counters, slab samples, resume state
// ---------------------------------------------------------------------------
// Pass-1 slab staging: a lane puts its samples in a 4-slot shared-memory group (SoA,
// conflict-free) and writes each group of 4 slab entries as one 256-bit (t) and one 128-bit
// (cell) store; slab rows are 32-byte aligned (C is a multiple of 4).
__device__ __forceinline__ void stage_flush(const SlabDev& S, int64_t idx, const double* st,
                                            const uint32_t* sc) {
    static_cast<double4*>(__builtin_assume_aligned(S.t + idx, 32))[0] =
        make_double4(st[0], st[kBlock], st[2 * kBlock], st[3 * kBlock]);
    static_cast<uint4*>(__builtin_assume_aligned(S.cell + idx, 16))[0] =
        make_uint4(sc[0], sc[kBlock], sc[2 * kBlock], sc[3 * kBlock]);
}

template <int AN, bool CASC, bool BR, int SCH, class Src>
__global__ void __launch_bounds__(kBlock, CASC ? SOGK_CASC_MINB : SOGK_COUNT_MINB)
    count_kernel(const __grid_constant__ SamplerDev s, const Src src, int64_t n, int64_t* __restrict__ packed,
                 int64_t* __restrict__ stats, uint8_t* __restrict__ status,
                 int32_t* __restrict__ counters, const SlabDev S) {
    __shared__ double stage_t[4 * kBlock];
    __shared__ uint32_t stage_c[4 * kBlock];
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    Stats5 acc;
    if (r < n) {
        const Ray ray = src.load(r);
        if (!ray_valid(ray)) {
            count_invalid(r, packed, status, counters, acc);
        } else {
            RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
            gen.init(ray, s);
            const int64_t row = r * S.C;
            long long c = 0;
            int filled = 0;     // samples in the slab
            bool ovf = false;   // slab full: the rest of the ray comes from its resume state
            bool stored = false;
            bool tail_flushed = false; // the group holding the slab's last sample is written
            double* const st_t = stage_t + threadIdx.x;
            uint32_t* const st_c = stage_c + threadIdx.x;
            for (;;) { // one flat loop: one analyzer step per iteration
                Event ev;
                double t_last0;
                const int st = gen.step_event(s, ev, t_last0);
                if (st == 0) break;
                if (st == 1) continue;
                int k = 0; // points of this event
                if (!ovf) { // the reference loop itself: while (t <= t1) { push(t); t += step(t); }
                    // single grids: the 2-bit Level rides in the cell word's spare top bits
                    // (cells pack 3 x 10 bits); cascades also need grid_level, in S.lvl
                    const uint32_t cw = CASC ? pack_cell(ev.ijk)
                                             : pack_cell(ev.ijk) | ((uint32_t)ev.level << 30);
                    const uint8_t lvl = (uint8_t)(ev.level | (ev.grid_level << 2));
                    double t = gen.t_last;
                    const int room = (int)S.C - filled;
                    while (t <= ev.t1 && k < room) {
                        const int p = filled + k;
                        st_t[(p & 3) * kBlock] = t;
                        st_c[(p & 3) * kBlock] = cw;
                        if (CASC) S.lvl[row + p] = lvl;
                        if ((p & 3) == 3) stage_flush(S, row + p - 3, st_t, st_c);
                        t = t + ladder_step<SCH>(t, s.dt0, s.growth);
                        ++k;
                    }
                    gen.t_last = t;
                    if (t <= ev.t1) { // slab full inside this event: it restarts in tail_kernel
                        ovf = true;
                        // this event's samples may have recycled the staging slots of the
                        // group holding position filled - 1; that group was written whole first
                        tail_flushed = filled + k >= (filled & ~3) + 4;
                        Run run;
                        run.ijk[0] = ev.ijk[0];
                        run.ijk[1] = ev.ijk[1];
                        run.ijk[2] = ev.ijk[2];
                        run.tag = gen.an.resume_tag();
                        run.t0 = ev.t0;
                        run.t_last0 = t_last0;
                        store_resume(S.resume + r, run, filled);
                        stored = true;
                    } else {
                        filled += k;
                    }
                }
                if (ovf) k += gen.seek_to(s, ev.t1); // counted, not stored
                if (BR) gen.kernel_lookups += k;
                c += k;
            }
            // the partial last group (a slab row is private to its ray: written whole)
            if ((filled & 3) && !tail_flushed) stage_flush(S, row + (filled & ~3), st_t, st_c);
            count_finish(gen, r, c, packed, status, counters, acc);
            if (stored && c > 0 && !gen.undefined()) {
                S.ovf_list[atomicAdd(S.ovf_ctr, 1u)] = (uint32_t)r;
                ++acc.ovf;
            }
        }
    }
    acc.flush(stats); // warp-level: no block barrier, finished warps leave at once
}

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

// ---------------------------------------------------------------------------
// pass 2: rays with samples restart from their resume state and regenerate the
// runs with the pass-1 loop.  Each lane streams its own contiguous output
// range through a 4-sample register buffer: aligned groups of four go out as
// one 256-bit store per array (a full 32-byte sector per lane), the unaligned
// head and tail as scalars.
// ---------------------------------------------------------------------------
struct Out {
    double* t_starts;
    double* t_ends;
    int32_t* ray_indices;
    uint32_t* cells;
    uint8_t* levels;
};

template <int SCH>
__device__ __forceinline__ void store1(const Out& o, const SamplerDev& s, long long k, double t,
                                       int32_t ri, uint32_t cell, uint8_t lvl) {
    o.t_starts[k] = t;
    if (o.t_ends) o.t_ends[k] = t + ladder_step<SCH>(t, s.dt0, s.growth);
    if (o.ray_indices) o.ray_indices[k] = ri;
    if (o.cells) o.cells[k] = cell;
    if (o.levels) o.levels[k] = lvl;
}

// Per-lane writer state of pass 2: the pending run and a 4-sample shift register.
template <int SCH, bool VEC>
struct LaneWriter {
    int32_t ri;
    long long out, end;
    double pt;
    int prem;
    uint32_t pcell;
    uint8_t plvl;
    double b0, b1, b2, b3; // pending samples (b3 newest)
    uint32_t c0, c1, c2, c3;
    uint32_t lv;
    int nb;

    __device__ __forceinline__ void start(int32_t ray_index, long long off, long long cnt) {
        ri = ray_index;
        out = off;
        end = off + cnt;
        prem = 0;
        nb = 0;
        b0 = b1 = b2 = b3 = 0.0;
        c0 = c1 = c2 = c3 = 0;
        lv = 0;
    }
    __device__ __forceinline__ bool done() const { return out + nb >= end; }
    __device__ __forceinline__ void take(const Run& run) {
        pt = run.first;
        prem = run.n;
        const long long left = end - out - nb;
        if (prem > left) prem = (int)left;
        pcell = run.cell;
        plvl = run.level;
    }
    // emit up to 4 samples of the pending run
    __device__ __forceinline__ void emit4(const Out& o, const SamplerDev& s) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (prem > 0) {
                if (VEC && (nb > 0 || (out & 3) == 0)) {
                    b0 = b1; b1 = b2; b2 = b3; b3 = pt;
                    c0 = c1; c1 = c2; c2 = c3; c3 = pcell;
                    lv = (lv >> 8) | ((uint32_t)plvl << 24);
                    if (++nb == 4) {
                        static_cast<double4*>(__builtin_assume_aligned(o.t_starts + out, 32))[0] =
                            make_double4(b0, b1, b2, b3);
                        if (o.t_ends)
                            static_cast<double4*>(__builtin_assume_aligned(o.t_ends + out, 32))[0] =
                                make_double4(b0 + ladder_step<SCH>(b0, s.dt0, s.growth),
                                             b1 + ladder_step<SCH>(b1, s.dt0, s.growth),
                                             b2 + ladder_step<SCH>(b2, s.dt0, s.growth),
                                             b3 + ladder_step<SCH>(b3, s.dt0, s.growth));
                        if (o.ray_indices)
                            static_cast<int4*>(__builtin_assume_aligned(o.ray_indices + out, 16))[0] =
                                make_int4(ri, ri, ri, ri);
                        if (o.cells)
                            static_cast<uint4*>(__builtin_assume_aligned(o.cells + out, 16))[0] =
                                make_uint4(c0, c1, c2, c3);
                        if (o.levels)
                            static_cast<uint32_t*>(__builtin_assume_aligned(o.levels + out, 4))[0] = lv;
                        out += 4;
                        nb = 0;
                    }
                } else {
                    store1<SCH>(o, s, out, pt, ri, pcell, plvl);
                    ++out;
                }
                pt = pt + ladder_step<SCH>(pt, s.dt0, s.growth);
                --prem;
            }
        }
    }
    // the nb newest samples sit in b[4-nb..3]
    __device__ __forceinline__ void flush(const Out& o, const SamplerDev& s) {
        if (nb >= 3) store1<SCH>(o, s, out++, b1, ri, c1, (uint8_t)(lv >> 8));
        if (nb >= 2) store1<SCH>(o, s, out++, b2, ri, c2, (uint8_t)(lv >> 16));
        if (nb >= 1) store1<SCH>(o, s, out++, b3, ri, c3, (uint8_t)(lv >> 24));
        nb = 0;
    }
};


// cold path: no pass-1 slabs for these rays, traverse from the start
template <int AN, bool CASC, bool BR, int SCH, bool VEC, class Src>
__global__ void __launch_bounds__(kWriteBlock)
    write_kernel(const __grid_constant__ SamplerDev s, const Src src, int64_t n, const int64_t* __restrict__ packed,
                 int64_t ray_index_base, const Out o) {
    const int64_t r = (int64_t)blockIdx.x * kWriteBlock + threadIdx.x;
    if (r >= n) return;
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
    if (pi.y == 0) return;
    RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
    gen.init(src.load(r), s);
    LaneWriter<SCH, VEC> w;
    w.start((int32_t)(ray_index_base + r), pi.x, pi.y);
    Run run;
    while (!w.done()) { // flat loop: one analyzer step or up to 4 samples per iteration
        if (w.prem == 0) {
            const int st = gen.step(s, run);
            if (st == 0) break; // unreachable when pass 1 and 2 agree
            if (st == 2) w.take(run);
        }
        w.emit4(o, s);
    }
    w.flush(o, s);
}

// pass 2: slabs -> packed arrays.  A block owns kGather consecutive rays, whose samples
// form one contiguous output range; thread i handles output samples i, i + kGather, ...
// (consecutive threads on consecutive samples: every store is coalesced and every output
// sector is written whole by one warp).  The owning ray of a sample is a binary search
// over the block's offsets in shared memory.  Samples past a ray's slab are tail_kernel's.
constexpr int kGather = 256;

template <int SCH, bool CASC>
__global__ void __launch_bounds__(kGather)
    gather_kernel(const __grid_constant__ SamplerDev s, int64_t n, const int64_t* __restrict__ packed,
                  const SlabDev S, int64_t ray_index_base, const Out o) {
    __shared__ long long s_base[2];
    __shared__ int s_off[kGather]; // ray offsets relative to the block's first sample
    __shared__ int s_fill[kGather];
    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * kGather;
    const int nr = (int)(n - r0 < kGather ? n - r0 : kGather);
    const int64_t r = r0 + tid;
    longlong2 pi = make_longlong2(0, 0);
    if (tid < nr) pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
    if (tid == 0) s_base[0] = pi.x;
    if (tid == nr - 1) s_base[1] = pi.x + pi.y;
    __syncthreads();
    const long long O0 = s_base[0], O1 = s_base[1];
    // a block's samples (<= kGather * max per-ray count) fit 31 bits
    s_off[tid] = tid < nr ? (int)(pi.x - O0) : INT_MAX;
    int fill = (int)(pi.y < S.C ? pi.y : S.C);
    if (tid < nr && pi.y > S.C) fill = S.resume[r].tag >> 8; // overflowed: what pass 1 put in the slab
    s_fill[tid] = fill;
    __syncthreads();
    const int m = (int)(O1 - O0);
    // kUnroll independent samples per thread and iteration (stride kGather: stores stay
    // coalesced), so each thread keeps several slab loads in flight
    constexpr int kUnroll = 4;
    for (int e0 = tid; e0 < m; e0 += kUnroll * kGather) {
        int j[kUnroll], k[kUnroll];
        bool ok[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int e = e0 + u * kGather;
            int jj = 0; // largest jj with s_off[jj] <= e: branch-free binary search
#pragma unroll
            for (int step = kGather / 2; step > 0; step >>= 1)
                jj += (s_off[jj + step] <= e) ? step : 0;
            j[u] = jj;
            k[u] = e - s_off[jj];
            ok[u] = e < m && k[u] < s_fill[jj];
        }
        double t[kUnroll];
        uint32_t cw[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            t[u] = 0.0;
            cw[u] = 0;
            if (ok[u]) {
                const int64_t i = (r0 + j[u]) * S.C + k[u];
                t[u] = __ldcs(S.t + i);
                cw[u] = __ldcs(reinterpret_cast<const unsigned int*>(S.cell) + i);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (!ok[u]) continue;
            const long long g = O0 + e0 + u * kGather;
            __stcs(o.t_starts + g, t[u]);
            if (o.t_ends) __stcs(o.t_ends + g, t[u] + ladder_step<SCH>(t[u], s.dt0, s.growth));
            if (o.ray_indices) __stcs(o.ray_indices + g, (int32_t)(ray_index_base + r0 + j[u]));
            if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + g, CASC ? cw[u] : cw[u] & 0x3fffffffu);
            if (o.levels) {
                const int64_t i = (r0 + j[u]) * S.C + k[u];
                o.levels[g] = CASC ? S.lvl[i] : (uint8_t)(cw[u] >> 30);
            }
        }
    }
}

// pass 2 for the rays whose slab overflowed: resume the traversal at the first run that
// did not fit and write the rest of the ray directly
template <int AN, bool CASC, bool BR, int SCH, bool VEC, class Src>
__global__ void __launch_bounds__(kWriteBlock)
    tail_kernel(const __grid_constant__ SamplerDev s, const Src src, const int64_t* __restrict__ packed,
                const SlabDev S, int64_t ray_index_base, const Out o) {
    const unsigned cnt = *S.ovf_ctr;
    for (unsigned i = blockIdx.x * kWriteBlock + threadIdx.x; i < cnt; i += gridDim.x * kWriteBlock) {
        const int64_t r = S.ovf_list[i];
        const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
        Resume res = S.resume[r];
        const long long skip = res.tag >> 8;
        res.tag &= 255;
        RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
        gen.init(src.load(r), s);
        gen.resume(s, res);
        LaneWriter<SCH, VEC> w;
        w.start((int32_t)(ray_index_base + r), pi.x + skip, pi.y - skip);
        Run run;
        while (!w.done()) {
            if (w.prem == 0) {
                const int st = gen.step(s, run);
                if (st == 0) break;
                if (st == 2) w.take(run);
            }
            w.emit4(o, s);
        }
        w.flush(o, s);
    }
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
static bool vec_ok(const Out& o) { // 256-bit stores need 32-byte aligned bases (16 for 4-byte arrays)
    return (reinterpret_cast<uintptr_t>(o.t_starts) & 31) == 0 &&
           (reinterpret_cast<uintptr_t>(o.t_ends) & 31) == 0 &&
           (reinterpret_cast<uintptr_t>(o.ray_indices) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(o.cells) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(o.levels) & 3) == 0;
}

static unsigned tail_grid(int64_t n) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const int64_t want = (n + kWriteBlock - 1) / kWriteBlock;
    const int64_t cap = (int64_t)sms * 8;
    return (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
}

template <class Src>
struct Launch {
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t count(const SamplerDev& s, const Src& src, int64_t n, int64_t* packed,
                             int64_t* stats, uint8_t* status, int32_t* counters, const SlabDev& S,
                             cudaStream_t st) {
        const int64_t blocks = (n + kBlock - 1) / kBlock;
        count_kernel<AN, CASC, BR, SCH, Src>
            <<<(unsigned)blocks, kBlock, 0, st>>>(s, src, n, packed, stats, status, counters, S);
        return cudaGetLastError();
    }
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t write(const SamplerDev& s, const Src& src, int64_t n, const int64_t* packed,
                             const SlabDev* S, int64_t base, const Out& o, cudaStream_t st) {
        const unsigned blocks = (unsigned)((n + kWriteBlock - 1) / kWriteBlock);
        const bool vec = vec_ok(o);
        if (!S) {
            if (vec)
                write_kernel<AN, CASC, BR, SCH, true, Src><<<blocks, kWriteBlock, 0, st>>>(s, src, n, packed, base, o);
            else
                write_kernel<AN, CASC, BR, SCH, false, Src><<<blocks, kWriteBlock, 0, st>>>(s, src, n, packed, base, o);
            return cudaGetLastError();
        }
        const unsigned gb = (unsigned)((n + kGather - 1) / kGather);
        gather_kernel<SCH, CASC><<<gb, kGather, 0, st>>>(s, n, packed, *S, base, o);
        const unsigned tg = tail_grid(n);
        if (vec)
            tail_kernel<AN, CASC, BR, SCH, true, Src><<<tg, kWriteBlock, 0, st>>>(s, src, packed, *S, base, o);
        else
            tail_kernel<AN, CASC, BR, SCH, false, Src><<<tg, kWriteBlock, 0, st>>>(s, src, packed, *S, base, o);
        return cudaGetLastError();
    }
};

// Variant key: analyzer (0 dda / 1 hdda), cascade, kernel == branch, schedule == linear.
cudaError_t launch_count(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, int64_t* packed,
                         int64_t* stats, uint8_t* status, int32_t* counters, const SlabDev& slab,
                         cudaStream_t st) {
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        SOGK_DISPATCH(count, s, src, n, packed, stats, status, counters, slab, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays};
        SOGK_DISPATCH(count, s, src, n, packed, stats, status, counters, slab, st);
    }
}

cudaError_t launch_scan(int64_t n, int64_t* packed, int64_t* stats, uint64_t* tiles,
                        unsigned int* ctr, cudaStream_t st) {
    const int64_t tiles_n = (n + kScanTile - 1) / kScanTile;
    scan_kernel<<<(unsigned)tiles_n, kScanThreads, 0, st>>>(n, packed, stats, tiles, ctr);
    return cudaGetLastError();
}

int64_t scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }
size_t resume_bytes(int64_t n) { return size_t(n) * sizeof(Resume); }

cudaError_t launch_write(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, const int64_t* packed,
                         const SlabDev* slab, int64_t base, double* ts, double* te, int32_t* ri,
                         uint32_t* ce, uint8_t* lv, cudaStream_t st) {
    const Out o{ts, te, ri, ce, lv};
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        SOGK_DISPATCH(write, s, src, n, packed, slab, base, o, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays};
        SOGK_DISPATCH(write, s, src, n, packed, slab, base, o, st);
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
