// sogk_sample_kernels.cuh — K2/K3/K5 pass-1 / pass-2 kernels and their per-variant launchers
// (included by the per-analyzer translation units sogk_sample_{dda,hdda,cd}.cu, so that the
// 24 variants compile in parallel).  See sogk_sample.cu for the pipeline.
#pragma once
#include <cuda_runtime.h>

#include <climits>

#include "sogk_device.cuh"
#include "sogk_internal.h"
#include "sogk_sources.cuh"

namespace sogk {

constexpr int kBlock = kGeomBlock;
constexpr int kWriteBlock = kGeomBlock;
#ifndef SOGK_GATHER_SHORT
#define SOGK_GATHER_SHORT 8
#endif
#ifndef SOGK_CASC_MINB
#define SOGK_CASC_MINB 5 // cascade variants: <= 96 registers (A/B cfg3: HDDA step -4 %, DDA -24 % vs 126)
#endif
#ifndef SOGK_ONE_TEMPLATE
#define SOGK_ONE_TEMPLATE 1 // pass 1 compiled per HDDA query mode (single-region / root read), not branched
#endif
#ifndef SOGK_REC_V4
#define SOGK_REC_V4 1 // pass 1 writes each run record with one 128-bit store
#endif
#ifndef SOGK_COUNT_MINB
#define SOGK_COUNT_MINB 7 // DDA pass-1 min resident blocks per SM: <= 72 registers (A/B: -7 % vs 76-88; 8: +4-10 %)
#endif
#ifndef SOGK_COUNT_MINB_NODE
#define SOGK_COUNT_MINB_NODE 8 // HDDA / CD pass 1: <= 64 registers, 24 B stack (A/B vs 7: HDDA cfg2 -1.7 %, cfg4 -2.5 %)
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

// resume state at `run`; tag bits 8..31 carry the number of samples already in the slab
// (filled <= kRunStartMax = 2^24 - 1: packed and unpacked as unsigned, never sign-extended)
__device__ __forceinline__ void store_resume(Resume* dst, const Run& run, uint32_t filled) {
    Resume r;
    r.ijk[0] = run.ijk[0];
    r.ijk[1] = run.ijk[1];
    r.ijk[2] = run.ijk[2];
    r.tag = (int)(((uint32_t)run.tag & 255u) | (filled << 8));
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
// one ray of pass 1 (the ray the j-th processing slot names: src.id(j))
template <int AN, bool CASC, bool BR, int SCH, class Src, int ONE>
__device__ __forceinline__ void count_one(const SamplerDev& s, const Src& src, int64_t j, int64_t* __restrict__ packed,
                                          uint8_t* __restrict__ status, int32_t* __restrict__ counters,
                                          const SlabDev& S, Stats5& acc) {
        const int64_t r = src.id(j);
        const Ray ray = src.load(r);
        if (!ray_valid(ray)) {
            count_invalid(r, packed, status, counters, acc);
            if (S.nruns) S.nruns[r] = 0;
        } else {
            RunGen<BR, SCH, typename PickAn<AN, CASC, ONE>::type> gen;
            gen.init(ray, s);
            RunRec* const row = S.runs + r * S.C;
            long long c = 0;
            int nr = 0;       // run records in the slab
            long long filled = 0; // samples they cover
            bool ovf = false; // slab full: the rest of the ray comes from its resume state
            for (;;) { // one flat loop: one analyzer step per iteration
                Event ev;
                double t_last0;
                const int st = gen.step_event(s, ev, t_last0);
                if (st == 0) break;
                if (st == 1) continue;
                const double first = gen.t_last;
                // the event's ladder points (t0, t1], counted in closed form
                const int k = gen.seek_to(s, ev.t1);
                if (BR) gen.kernel_lookups += k;
                c += k;
                if (k == 0 || ovf) continue;
                if (nr < S.C && filled + k <= (long long)kRunStartMax) {
                    RunRec rec;
                    rec.first = first;
                    rec.cell = pack_cell(ev.ijk);
                    rec.sl = (uint32_t)filled | ((uint32_t)(ev.level | (ev.grid_level << 2)) << 24);
#if SOGK_REC_V4
                    { // one 128-bit store per run (the struct copy compiles to two 64-bit stores)
                        const long long fb = __double_as_longlong(rec.first);
                        *reinterpret_cast<int4*>(row + nr) =
                            make_int4((int)(unsigned)fb, (int)(unsigned)(fb >> 32), (int)rec.cell, (int)rec.sl);
                        ++nr;
                    }
#else
                    row[nr++] = rec;
#endif
                    filled += k;
                } else { // the run that does not fit restarts in tail_kernel
                    ovf = true;
                    Run run;
                    run.ijk[0] = ev.ijk[0];
                    run.ijk[1] = ev.ijk[1];
                    run.ijk[2] = ev.ijk[2];
                    run.tag = gen.an.resume_tag();
                    run.t0 = ev.t0;
                    run.t_last0 = t_last0;
                    store_resume(S.resume + r, run, (uint32_t)filled);
                }
            }
            // run count; bit 31 marks a ray whose runs overflowed the slab
            if (S.nruns) S.nruns[r] = gen.undefined() ? 0 : (nr | (ovf ? (int)0x80000000 : 0));
            count_finish(gen, r, c, packed, status, counters, acc);
            if (ovf && c > 0 && !gen.undefined()) {
                S.ovf_list[atomicAdd(S.ovf_ctr, 1u)] = (uint32_t)r;
                ++acc.ovf;
            }
        }
}

// ONE (HDDA): 1 = every level is a single-region VDB (its root entry is GridDev::node0), 0 = not
template <int AN, bool CASC, bool BR, int SCH, class Src, int ONE>
__global__ void __launch_bounds__(kBlock, CASC ? SOGK_CASC_MINB
                                               : (AN == SOGK_DDA ? SOGK_COUNT_MINB : SOGK_COUNT_MINB_NODE))
    count_kernel(const __grid_constant__ SamplerDev s, const Src src, int64_t n, int64_t* __restrict__ packed,
                 int64_t* __restrict__ stats, uint8_t* __restrict__ status,
                 int32_t* __restrict__ counters, const SlabDev S) {
    if (SOGK_SMEM_TABLE && s.lv[0].smem_tab) { // stage the single-region child table (16 KB) in shared memory
        const int32_t node0 = __ldg(s.lv[0].root);
        const int4* tsrc = reinterpret_cast<const int4*>(s.lv[0].table + (int64_t)(node0 < 0 ? 0 : node0) * 4096);
        int4* tdst = reinterpret_cast<int4*>(sogk_dyn_smem);
        for (int i = threadIdx.x; i < 1024; i += kBlock) tdst[i] = __ldg(tsrc + i);
        __syncthreads();
    }
    Stats5 acc;
    const int64_t j = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (j < n) count_one<AN, CASC, BR, SCH, Src, ONE>(s, src, j, packed, status, counters, S, acc);
    acc.flush(stats); // warp-level: no block barrier, finished warps leave at once
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

// pass 2: run slabs -> packed arrays.  A block owns kGather consecutive rays: their samples
// form one contiguous output range and their runs one local run index space (block scan of
// the per-ray run counts in shared memory).  Thread i expands runs i, i + kGather, ...: it
// finds the owning ray by a branch-free binary search over the block's run offsets, reads
// the run record (and the next one's start for its length) and writes the run's samples
// with the reference recurrence t <- t + step(t).  Consecutive threads take consecutive
// runs, whose samples are adjacent in the output.  Samples past a ray's slab are
// tail_kernel's.
constexpr int kGather = 256;
#ifndef SOGK_GATHER_STAGED
#define SOGK_GATHER_STAGED 1 // pass-2 output staged in shared memory, stored coalesced
#endif
#ifndef SOGK_STAGE_W
#define SOGK_STAGE_W 2048 // samples per staging window (17 B each in shared memory)
#endif
constexpr int kStageW = SOGK_STAGE_W;
#ifndef SOGK_GATHER_VEC
#define SOGK_GATHER_VEC 0 // 1: 128-bit stores of four samples per thread (A/B: pass 2 +11 % time, off)
#endif

// Output-parallel expansion of one pass-2 batch (constant schedule).  Per-run expansion
// (gather_kernel's staged path) gives each long run to one lane, or one warp, while the rest
// of the block waits at the window barrier; a batch with many long tile runs is expanded by
// OUTPUT position instead.  Thread i decodes run i into the shared run table -- output start,
// length, cell, level, ray index and the closed-form ladder constants of its first point
// (t1 = f + dt0, then bits(t2) + (k - 2) * inc while in f's binade, sogk_ladder.cuh) -- and
// then writes positions P0 + i, P0 + i + kGather, ... of the batch span: a branch-free binary
// search over the run starts finds the owning run and point k comes from the closed form
// (exact: the points of the reference recurrence t <- t + dt0, sampling.hpp:115-118).
// Consecutive threads store consecutive samples of every array.  Positions no run covers
// (the tails of slab-overflow rays) are skipped; tail_kernel writes them.
#ifndef SOGK_GATHER_MP
#define SOGK_GATHER_MP 32 // output-parallel when >= 1/32 of a batch's runs are long; 0: never
#endif
#ifndef SOGK_MP_NARROW
#define SOGK_MP_NARROW 1 // search 32-bit span-relative run starts when the span allows
#endif
#ifndef SOGK_MP_PAIRS
#define SOGK_MP_PAIRS 1 // narrow spans: two adjacent positions per thread, one search, 2-wide stores
#endif
struct MpTab {
    long long g0[kGather]; // output start (LLONG_MAX past the batch)
    int rel[kGather + 1];  // g0 - P0 for spans below 2^31 (INT_MAX past the batch)
    double f[kGather], t1[kGather];
    long long b2[kGather], inc[kGather];
    int n[kGather], kf[kGather];
    uint32_t ce[kGather];
    int32_t ri[kGather];
    uint8_t lv[kGather];
};

__device__ __forceinline__ void gather_mp_batch(const SamplerDev& s, const Out& o, MpTab& T, bool have,
                                                double f, long long g0, int nn, uint32_t cell, uint8_t lv,
                                                int32_t ri, long long P0, long long P1) {
    const int tid = threadIdx.x;
    const double dt0 = s.dt0;
    const bool narrow = SOGK_MP_NARROW && P1 - P0 < (long long)INT_MAX; // block-uniform
    if (have) {
        T.g0[tid] = g0;
        T.rel[tid] = narrow ? (int)(g0 - P0) : 0;
        T.n[tid] = nn;
        T.f[tid] = f;
        T.ce[tid] = cell;
        T.lv[tid] = lv;
        T.ri[tid] = ri;
        const double t1 = f + dt0;
        T.t1[tid] = t1;
        int kf = 1;
        if (nn > 2) { // closed form after two explicit in-binade steps
            const double t2 = t1 + dt0;
            const int64_t b0 = dbits(f), b1 = dbits(t1), b2 = dbits(t2);
            const int64_t inc = b2 - b1;
            const int64_t e0 = b0 >> 52;
            if (e0 == (b2 >> 52) && e0 != 0 && inc > 0) {
                const int64_t endb = (e0 + 1) << 52;
                const int64_t kq = 2 + fix_quotient(endb - 1 - b2, inc, (dfrom(endb) - t2) * s.inv_dt0);
                kf = kq < nn ? (int)kq : nn;
            }
            T.b2[tid] = b2;
            T.inc[tid] = inc;
        }
        T.kf[tid] = kf;
    } else {
        T.g0[tid] = LLONG_MAX;
        T.rel[tid] = INT_MAX;
    }
    if (tid == 0) T.rel[kGather] = INT_MAX;
    __syncthreads();
    // point k of run j: the closed form of the reference recurrence
    auto point = [&](int j, long long k) -> double {
        if (k == 0) return T.f[j];
        if (k == 1) return T.t1[j];
        if (k <= T.kf[j]) return dfrom(T.b2[j] + (k - 2) * T.inc[j]);
        return advance_const(T.f[j], k, dt0, s.inv_dt0);
    };
    const bool pair_ok = SOGK_MP_PAIRS && narrow &&
                         (((uintptr_t)o.t_starts | (uintptr_t)o.t_ends) & 15) == 0 &&
                         (((uintptr_t)o.ray_indices | (uintptr_t)o.cells) & 7) == 0 &&
                         ((uintptr_t)o.levels & 1) == 0;
    if (pair_ok) {
        // thread i takes the aligned pair (A, A + 1), A = (P0 & ~1) + 2 i + 2 kGather m: one
        // search for the first position inside the span, the second position is the same
        // run's next point (t + dt0, the recurrence itself) or the next run's first
        const long long A0 = P0 & ~1ll;
        const long long npairs = (P1 - A0 + 1) >> 1;
        for (long long i = tid; i < npairs; i += kGather) {
            const long long A = A0 + 2 * i;
            const int r0 = (int)(A - P0); // -1 for a pair that starts before the span
            const int re = r0 < 0 ? 0 : r0;
            int j = 0;
#pragma unroll
            for (int step = kGather / 2; step > 0; step >>= 1)
                j += (T.rel[j + step] <= re) ? step : 0;
            const int k0 = re - T.rel[j];
            const bool v0 = r0 >= 0 && k0 < T.n[j];
            int j1 = j, k1 = k0;
            if (r0 >= 0) {
                if (T.rel[j + 1] <= r0 + 1) { // the next run starts at A + 1
                    j1 = j + 1;
                    k1 = 0;
                } else {
                    k1 = k0 + 1;
                }
            }
            const bool v1 = A + 1 < P1 && k1 < T.n[j1];
            const double t0 = v0 ? point(j, k0) : 0.0;
            const double t1 = v1 ? ((v0 && j1 == j) ? t0 + dt0 : point(j1, k1)) : 0.0;
            if (v0 && v1) {
                __stcs(reinterpret_cast<double2*>(o.t_starts + A), make_double2(t0, t1));
                if (o.t_ends) __stcs(reinterpret_cast<double2*>(o.t_ends + A), make_double2(t0 + dt0, t1 + dt0));
                if (o.ray_indices) __stcs(reinterpret_cast<int2*>(o.ray_indices + A), make_int2(T.ri[j], T.ri[j1]));
                if (o.cells) __stcs(reinterpret_cast<uint2*>(o.cells + A), make_uint2(T.ce[j], T.ce[j1]));
                if (o.levels)
                    *reinterpret_cast<uint16_t*>(o.levels + A) = (uint16_t)(T.lv[j] | ((uint32_t)T.lv[j1] << 8));
            } else {
                if (v0) {
                    __stcs(o.t_starts + A, t0);
                    if (o.t_ends) __stcs(o.t_ends + A, t0 + dt0);
                    if (o.ray_indices) __stcs(o.ray_indices + A, T.ri[j]);
                    if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + A, T.ce[j]);
                    if (o.levels) o.levels[A] = T.lv[j];
                }
                if (v1) {
                    __stcs(o.t_starts + A + 1, t1);
                    if (o.t_ends) __stcs(o.t_ends + A + 1, t1 + dt0);
                    if (o.ray_indices) __stcs(o.ray_indices + A + 1, T.ri[j1]);
                    if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + A + 1, T.ce[j1]);
                    if (o.levels) o.levels[A + 1] = T.lv[j1];
                }
            }
        }
        __syncthreads();
        return;
    }
    for (long long p = P0 + tid; p < P1; p += kGather) {
        int j = 0; // the last run starting at or before p
        if (narrow) {
            const int rp = (int)(p - P0);
#pragma unroll
            for (int step = kGather / 2; step > 0; step >>= 1)
                j += (T.rel[j + step] <= rp) ? step : 0;
        } else {
#pragma unroll
            for (int step = kGather / 2; step > 0; step >>= 1)
                j += (T.g0[j + step] <= p) ? step : 0;
        }
        const long long k = p - T.g0[j];
        if (k < T.n[j]) {
            const double t = point(j, k);
            __stcs(o.t_starts + p, t);
            if (o.t_ends) __stcs(o.t_ends + p, t + dt0);
            if (o.ray_indices) __stcs(o.ray_indices + p, T.ri[j]);
            if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + p, T.ce[j]);
            if (o.levels) o.levels[p] = T.lv[j];
        }
    }
    __syncthreads();
}

#ifndef SOGK_GATHER_MINB
#define SOGK_GATHER_MINB 4 // <= 64 registers: 4 blocks of 256 per SM
#endif
template <int SCH, bool VEC, bool MP>
__global__ void __launch_bounds__(kGather, SOGK_GATHER_MINB)
    gather_kernel(const __grid_constant__ SamplerDev s, int64_t n, const int64_t* __restrict__ packed,
                  const SlabDev S, int64_t ray_index_base, const Out o) {
    __shared__ int s_roff[kGather + 1]; // local run offsets (exclusive), INT_MAX past the rays
    __shared__ long long s_off[kGather]; // output offset of each ray
    __shared__ int s_fill[kGather];      // samples of each ray covered by its slab
    __shared__ int s_nr[kGather];
    __shared__ int s_wsum[kGather / 32];
    constexpr int kShort = SOGK_GATHER_SHORT; // runs up to this long: expanded by their own lane
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * kGather;
    const int nrays = (int)(n - r0 < kGather ? n - r0 : kGather);
    const int64_t r = r0 + tid;
    int nr = 0;
    if (tid < nrays) {
        const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
        const int raw = pi.y > 0 ? __ldg(S.nruns + r) : 0;
        nr = raw & 0x7fffffff;
        s_off[tid] = pi.x;
        // every sample of the ray is in its runs, unless they overflowed the slab: then the
        // slab covers the samples before the resume point (Resume::tag >> 8)
        s_fill[tid] = raw < 0 ? (int)((uint32_t)S.resume[r].tag >> 8) : (int)pi.y;
    }
    s_nr[tid] = nr;
    // block exclusive scan of the run counts
    int v = nr;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += y;
    }
    if (lane == 31) s_wsum[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int w = lane < kGather / 32 ? s_wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += y;
        }
        if (lane < kGather / 32) s_wsum[lane] = w;
    }
    __syncthreads();
    const int incl = v + (wid > 0 ? s_wsum[wid - 1] : 0);
    s_roff[tid] = tid < nrays ? incl - nr : INT_MAX;
    const int total = s_wsum[kGather / 32 - 1];
    __syncthreads();
#if SOGK_GATHER_STAGED
    // Output staging: each batch of kGather runs covers one contiguous output span [P0, P1)
    // (runs are in output order); it is produced window by window into shared memory --
    // short runs by their own lane, long runs by the whole warp, both clipped to the window --
    // and every window goes out with fully coalesced stores (a warp writes 32 consecutive
    // samples of each array).  Positions no run covers (the tails of slab-overflow rays) carry
    // stale values; tail_kernel, next on the stream, overwrites them.
    // (the same bytes hold an output-parallel batch's run table, MpTab, when that path runs)
    __shared__ __align__(16) unsigned char s_raw[kStageW * 17];
    double* const s_t = reinterpret_cast<double*>(s_raw);
    int32_t* const s_ri = reinterpret_cast<int32_t*>(s_raw + 8 * kStageW);
    uint32_t* const s_ce = reinterpret_cast<uint32_t*>(s_raw + 12 * kStageW);
    uint8_t* const s_lv = s_raw + 16 * kStageW;
    __shared__ long long s_span[2];
    static_assert(sizeof(MpTab) <= sizeof(s_raw), "run table must fit the staging window");
#endif
    // run records of the next batch are loaded while the current one is expanded (software
    // pipelining: the scattered 16-byte record loads are the kernel's long-scoreboard stall)
    auto locate = [&](int q, int& j) -> const RunRec* {
        j = 0; // largest j with s_roff[j] <= q: branch-free binary search
#pragma unroll
        for (int step = kGather / 2; step > 0; step >>= 1)
            j += (s_roff[j + step] <= q) ? step : 0;
        return S.runs + (r0 + j) * S.C + (q - s_roff[j]);
    };
    RunRec pa{};
    uint32_t pnsl = 0xffffffffu; // next record's start | level, or ~0: the ray's fill ends the run
    int pj = 0;
    if (tid < total) {
        const RunRec* rec = locate(tid, pj);
        pa = *rec;
        if (tid - s_roff[pj] + 1 < s_nr[pj]) pnsl = rec[1].sl;
    }
    for (int base = 0; base < total; base += kGather) { // block-uniform trip count
        const int q = base + tid;
        const bool have = q < total;
        double first = 0.0;
        long long g0 = 0;
        int n = 0;
        uint32_t cell = 0;
        uint8_t lv = 0;
        int32_t ri = 0;
        if (have) {
            const int start = (int)(pa.sl & kRunStartMax);
            const int end = pnsl != 0xffffffffu ? (int)(pnsl & kRunStartMax) : s_fill[pj];
            first = pa.first;
            g0 = s_off[pj] + start;
            n = end - start;
            cell = pa.cell;
            lv = (uint8_t)(pa.sl >> 24);
            ri = (int32_t)(ray_index_base + r0 + pj);
        }
        if (q + kGather < total) { // prefetch the next batch's record
            const RunRec* rec = locate(q + kGather, pj);
            pa = *rec;
            pnsl = (q + kGather - s_roff[pj] + 1 < s_nr[pj]) ? rec[1].sl : 0xffffffffu;
        }
#if SOGK_GATHER_STAGED
        if (tid == 0) s_span[0] = g0; // the batch's first run starts its span
        if (have && (q + 1 == total || tid + 1 == kGather)) s_span[1] = g0 + n;
        if constexpr (MP) {
            // batches with many long (tile) runs go output-parallel (the count rides on the
            // span barrier)
            const int nlong = __syncthreads_count(have && n > kShort);
            const int nb = total - base < kGather ? total - base : kGather;
            if (nlong * SOGK_GATHER_MP >= nb) { // block-uniform
                gather_mp_batch(s, o, *reinterpret_cast<MpTab*>(s_raw), have, first, g0, n, cell, lv, ri,
                                s_span[0], s_span[1]);
                continue;
            }
        } else {
            __syncthreads();
        }
        const long long P0 = s_span[0], P1 = s_span[1];
        for (long long w = P0; w < P1; w += kStageW) { // block-uniform
            const long long we = (P1 - w < kStageW) ? P1 : w + kStageW;
            if (n > 0 && n <= kShort && g0 < we && g0 + n > w) {
                double t = first;
                for (int k = 0; k < n; ++k) {
                    const long long g = g0 + k;
                    if (g >= we) break;
                    if (g >= w) {
                        const int p = (int)(g - w);
                        s_t[p] = t;
                        s_ri[p] = ri;
                        s_ce[p] = cell;
                        s_lv[p] = lv;
                    }
                    t = t + ladder_step<SCH>(t, s.dt0, s.growth);
                }
            }
            unsigned lm = __ballot_sync(0xffffffffu, n > kShort && g0 < we && g0 + n > w);
            while (lm) {
                const int src = __ffs(lm) - 1;
                lm &= lm - 1;
                const double f = __shfl_sync(0xffffffffu, first, src);
                const long long gb = __shfl_sync(0xffffffffu, g0, src);
                const int nn = __shfl_sync(0xffffffffu, n, src);
                const uint32_t ce = __shfl_sync(0xffffffffu, cell, src);
                const int lvl = __shfl_sync(0xffffffffu, (int)lv, src);
                const int32_t rr = __shfl_sync(0xffffffffu, ri, src);
                double t1 = 0.0;
                int64_t b2 = 0, inc = 0, kfast = 1;
                if (SCH == 0) { // closed form after two explicit in-binade steps (sogk_ladder.cuh)
                    t1 = f + s.dt0;
                    const double t2 = t1 + s.dt0;
                    const int64_t b0 = dbits(f), b1 = dbits(t1);
                    b2 = dbits(t2);
                    inc = b2 - b1;
                    const int64_t e0 = b0 >> 52;
                    if (e0 == (b2 >> 52) && e0 != 0 && inc > 0) {
                        const int64_t end = (e0 + 1) << 52;
                        kfast = 2 + fix_quotient(end - 1 - b2, inc, (dfrom(end) - t2) * s.inv_dt0);
                    }
                }
                const int ka = (int)(w > gb ? w - gb : 0);
                const int kb = (int)(gb + nn < we ? nn : we - gb);
                for (int k = ka + lane; k < kb; k += 32) {
                    double t;
                    if (SCH == 0 && k <= kfast)
                        t = k == 0 ? f : (k == 1 ? t1 : dfrom(b2 + (int64_t)(k - 2) * inc));
                    else
                        t = ladder_advance<SCH>(f, k, s.dt0, s.inv_dt0, s.growth, s.t_switch);
                    const int p = (int)(gb + k - w);
                    s_t[p] = t;
                    s_ri[p] = rr;
                    s_ce[p] = ce;
                    s_lv[p] = (uint8_t)lvl;
                }
            }
            __syncthreads();
            const int m = (int)(we - w);
            // coalesced stores; with aligned outputs the body goes out as 128-bit stores of four
            // consecutive samples per thread (the scalar head / tail align it to 4 samples)
            const int h = VEC ? (int)((-w) & 3) < m ? (int)((-w) & 3) : m : m;
            for (int p = tid; p < h; p += kGather) {
                const long long g = w + p;
                const double t = s_t[p];
                __stcs(o.t_starts + g, t);
                if (o.t_ends) __stcs(o.t_ends + g, t + ladder_step<SCH>(t, s.dt0, s.growth));
                if (o.ray_indices) __stcs(o.ray_indices + g, s_ri[p]);
                if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + g, s_ce[p]);
                if (o.levels) o.levels[g] = s_lv[p];
            }
            if (VEC) {
                const int nq = (m - h) >> 2;
                for (int qd = tid; qd < nq; qd += kGather) {
                    const int p = h + 4 * qd;
                    const long long g = w + p; // multiple of 4
                    const double a0 = s_t[p], a1 = s_t[p + 1], a2 = s_t[p + 2], a3 = s_t[p + 3];
                    double2* ts = reinterpret_cast<double2*>(o.t_starts + g);
                    __stcs(ts, make_double2(a0, a1));
                    __stcs(ts + 1, make_double2(a2, a3));
                    if (o.t_ends) {
                        double2* te = reinterpret_cast<double2*>(o.t_ends + g);
                        __stcs(te, make_double2(a0 + ladder_step<SCH>(a0, s.dt0, s.growth),
                                                a1 + ladder_step<SCH>(a1, s.dt0, s.growth)));
                        __stcs(te + 1, make_double2(a2 + ladder_step<SCH>(a2, s.dt0, s.growth),
                                                    a3 + ladder_step<SCH>(a3, s.dt0, s.growth)));
                    }
                    if (o.ray_indices)
                        __stcs(reinterpret_cast<int4*>(o.ray_indices + g),
                               make_int4(s_ri[p], s_ri[p + 1], s_ri[p + 2], s_ri[p + 3]));
                    if (o.cells)
                        __stcs(reinterpret_cast<uint4*>(o.cells + g),
                               make_uint4(s_ce[p], s_ce[p + 1], s_ce[p + 2], s_ce[p + 3]));
                    if (o.levels)
                        *reinterpret_cast<uint32_t*>(o.levels + g) =
                            (uint32_t)s_lv[p] | ((uint32_t)s_lv[p + 1] << 8) | ((uint32_t)s_lv[p + 2] << 16) |
                            ((uint32_t)s_lv[p + 3] << 24);
                }
                for (int p = h + 4 * nq + tid; p < m; p += kGather) {
                    const long long g = w + p;
                    const double t = s_t[p];
                    __stcs(o.t_starts + g, t);
                    if (o.t_ends) __stcs(o.t_ends + g, t + ladder_step<SCH>(t, s.dt0, s.growth));
                    if (o.ray_indices) __stcs(o.ray_indices + g, s_ri[p]);
                    if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + g, s_ce[p]);
                    if (o.levels) o.levels[g] = s_lv[p];
                }
            }
            __syncthreads();
        }
#else
        if (n <= kShort) { // the common case: a voxel's few points, by its own lane
            double t = first;
            for (int k = 0; k < n; ++k) {
                const double tn = t + ladder_step<SCH>(t, s.dt0, s.growth);
                const long long g = g0 + k;
                __stcs(o.t_starts + g, t);
                if (o.t_ends) __stcs(o.t_ends + g, tn);
                if (o.ray_indices) __stcs(o.ray_indices + g, ri);
                if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + g, cell);
                if (o.levels) o.levels[g] = lv;
                t = tn;
            }
        }
        // long runs (tiles): the whole warp writes each one, point k from the run's first
        // point by the closed-form ladder advance (exact), consecutive lanes on consecutive
        // points
        unsigned lm = __ballot_sync(0xffffffffu, n > kShort);
        while (lm) {
            const int src = __ffs(lm) - 1;
            lm &= lm - 1;
            const double f = __shfl_sync(0xffffffffu, first, src);
            const long long gb = __shfl_sync(0xffffffffu, g0, src);
            const int nn = __shfl_sync(0xffffffffu, n, src);
            const uint32_t ce = __shfl_sync(0xffffffffu, cell, src);
            const int lvl = __shfl_sync(0xffffffffu, (int)lv, src);
            const int32_t rr = __shfl_sync(0xffffffffu, ri, src);
            // constant schedule: after two explicit in-binade steps every further in-binade
            // step adds the same bit increment (sogk_ladder.cuh), so point k >= 2 is
            // bits(t2) + (k - 2) * inc while it stays in t0's binade
            double t1 = 0.0;
            int64_t b2 = 0, inc = 0, kfast = 1;
            if (SCH == 0) {
                t1 = f + s.dt0;
                const double t2 = t1 + s.dt0;
                const int64_t b0 = dbits(f), b1 = dbits(t1);
                b2 = dbits(t2);
                inc = b2 - b1;
                const int64_t e0 = b0 >> 52;
                if (e0 == (b2 >> 52) && e0 != 0 && inc > 0) {
                    const int64_t end = (e0 + 1) << 52;
                    kfast = 2 + fix_quotient(end - 1 - b2, inc, (dfrom(end) - t2) * s.inv_dt0);
                }
            }
            for (int k = lane; k < nn; k += 32) {
                double t;
                if (SCH == 0 && k <= kfast)
                    t = k == 0 ? f : (k == 1 ? t1 : dfrom(b2 + (int64_t)(k - 2) * inc));
                else
                    t = ladder_advance<SCH>(f, k, s.dt0, s.inv_dt0, s.growth, s.t_switch);
                const long long g = gb + k;
                __stcs(o.t_starts + g, t);
                if (o.t_ends) __stcs(o.t_ends + g, t + ladder_step<SCH>(t, s.dt0, s.growth));
                if (o.ray_indices) __stcs(o.ray_indices + g, rr);
                if (o.cells) __stcs(reinterpret_cast<unsigned int*>(o.cells) + g, ce);
                if (o.levels) o.levels[g] = (uint8_t)lvl;
            }
        }
#endif
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
        const long long skip = (long long)((uint32_t)res.tag >> 8);
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

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
static inline bool vec_ok(const Out& o) { // 256-bit stores need 32-byte aligned bases (16 for 4-byte arrays)
    return (reinterpret_cast<uintptr_t>(o.t_starts) & 31) == 0 &&
           (reinterpret_cast<uintptr_t>(o.t_ends) & 31) == 0 &&
           (reinterpret_cast<uintptr_t>(o.ray_indices) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(o.cells) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(o.levels) & 3) == 0;
}

static inline unsigned tail_grid(int64_t n) {
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
        // upper VDB level in shared memory: the child table of a single-region grid (128^3 and
        // below) is staged per block; larger grids read it through L1 / L2
        SamplerDev s2 = s;
        size_t dyn = 0;
        if (SOGK_SMEM_TABLE && AN == SOGK_HDDA && !CASC && s.lv[0].R[0] * s.lv[0].R[1] * s.lv[0].R[2] == 1) {
            s2.lv[0].smem_tab = 1;
            dyn = 4096 * sizeof(int32_t);
        }
        const unsigned grid = (unsigned)blocks;
        if constexpr (AN == SOGK_HDDA && SOGK_ONE_TEMPLATE) { // single-region levels: no root read
            bool one = SOGK_NODE0 != 0;
            for (int b = 0; b < s.n_levels; ++b) one = one && s.lv[b].node0 != kNodeMulti;
            if (one) {
                count_kernel<AN, CASC, BR, SCH, Src, 1>
                    <<<grid, kBlock, dyn, st>>>(s2, src, n, packed, stats, status, counters, S);
                return cudaGetLastError();
            }
        }
        count_kernel<AN, CASC, BR, SCH, Src, SOGK_ONE_TEMPLATE ? 0 : -1>
            <<<grid, kBlock, dyn, st>>>(s2, src, n, packed, stats, status, counters, S);
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
        // output-parallel batches for the HDDA (tile runs, constant schedule); DDA and CD runs
        // are single voxels (a few points), for which per-run expansion is cheaper
        constexpr bool kMp = AN == SOGK_HDDA && SCH == 0 && SOGK_GATHER_MP > 0;
        if (vec && SOGK_GATHER_VEC)
            gather_kernel<SCH, true, kMp><<<gb, kGather, 0, st>>>(s, n, packed, *S, base, o);
        else
            gather_kernel<SCH, false, kMp><<<gb, kGather, 0, st>>>(s, n, packed, *S, base, o);
        const unsigned tg = tail_grid(n);
        if (vec)
            tail_kernel<AN, CASC, BR, SCH, true, Src><<<tg, kWriteBlock, 0, st>>>(s, src, packed, *S, base, o);
        else
            tail_kernel<AN, CASC, BR, SCH, false, Src><<<tg, kWriteBlock, 0, st>>>(s, src, packed, *S, base, o);
        return cudaGetLastError();
    }
};

// per-analyzer entry points (sogk_sample_{dda,hdda,cd}.cu): variant key within the analyzer =
// cascade << 2 | branch << 1 | linear
#define SOGK_DISPATCH_AN(AN, FN, ...)                                                            \
    do {                                                                                          \
        switch ((v.cascade << 2) | (v.branch << 1) | v.linear) {                                  \
            case 0: return L::template FN<AN, false, false, 0>(__VA_ARGS__);                      \
            case 1: return L::template FN<AN, false, false, 1>(__VA_ARGS__);                      \
            case 2: return L::template FN<AN, false, true, 0>(__VA_ARGS__);                       \
            case 3: return L::template FN<AN, false, true, 1>(__VA_ARGS__);                       \
            case 4: return L::template FN<AN, true, false, 0>(__VA_ARGS__);                       \
            case 5: return L::template FN<AN, true, false, 1>(__VA_ARGS__);                       \
            case 6: return L::template FN<AN, true, true, 0>(__VA_ARGS__);                        \
            default: return L::template FN<AN, true, true, 1>(__VA_ARGS__);                       \
        }                                                                                         \
    } while (0)

template <int AN>
cudaError_t launch_count_an(const Variant& v, const SamplerDev& s, const double* rays, const CameraDev* cam,
                            int64_t first, int64_t n, int64_t* packed, int64_t* stats, uint8_t* status,
                            int32_t* counters, const SlabDev& slab, cudaStream_t st, const uint32_t* perm) {
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        SOGK_DISPATCH_AN(AN, count, s, src, n, packed, stats, status, counters, slab, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays, perm};
        SOGK_DISPATCH_AN(AN, count, s, src, n, packed, stats, status, counters, slab, st);
    }
}

template <int AN>
cudaError_t launch_write_an(const Variant& v, const SamplerDev& s, const double* rays, const CameraDev* cam,
                            int64_t first, int64_t n, const int64_t* packed, const SlabDev* slab, int64_t base,
                            double* ts, double* te, int32_t* ri, uint32_t* ce, uint8_t* lv, cudaStream_t st) {
    const Out o{ts, te, ri, ce, lv};
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        SOGK_DISPATCH_AN(AN, write, s, src, n, packed, slab, base, o, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays};
        SOGK_DISPATCH_AN(AN, write, s, src, n, packed, slab, base, o, st);
    }
}

} // namespace sogk
