// sogk_sample.cu — K2/K3/K5 sampling kernels and K6 raygen.
//
// Pass 1 (count_kernel): one thread per ray runs the analyzer with the
// reference kernel's control flow (sample_skip / sample_branch over
// Dda/Hdda/CascadeTraversal, sampling.hpp:87-122, 166-196, 305-455), advancing
// the ladder per event in closed form; it writes the per-ray count, status,
// counters and the resume state at the ray's first sample run.
// Scan (scan_kernel): packed_info offsets = exclusive scan of the counts.
// Pass 2 (write_kernel): rays with samples restart from their resume state,
// regenerate the runs and stage samples in shared memory; each warp flushes
// its staged samples with consecutive threads on consecutive output indices.
#include <cuda_runtime.h>

#include "sogk_device.cuh"
#include "sogk_internal.h"

namespace sogk {

constexpr int kBlock = 128;
constexpr int kWriteBlock = 128;

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

template <int AN, bool CASC>
struct PickAn {
    using Sub = typename std::conditional<AN == SOGK_HDDA, HddaAn, DdaAn>::type;
    using type = AnyAn<Sub, CASC>;
};

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

__device__ __forceinline__ void store_resume(Resume* dst, const Run& run) {
    Resume r;
    r.ijk[0] = run.ijk[0];
    r.ijk[1] = run.ijk[1];
    r.ijk[2] = run.ijk[2];
    r.tag = run.tag;
    r.t_cur = run.t0;
    r.t_last = run.t_last0;
    *dst = r;
}

// ---------------------------------------------------------------------------
// pass 1: per-ray counts, status, counters, resume state
// ---------------------------------------------------------------------------
struct Stats5 {
    long long inv = 0, und = 0, lk = 0, sp = 0, klk = 0;
    __device__ __forceinline__ void flush(int64_t* stats) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            inv += __shfl_xor_sync(0xffffffffu, inv, o);
            und += __shfl_xor_sync(0xffffffffu, und, o);
            lk += __shfl_xor_sync(0xffffffffu, lk, o);
            sp += __shfl_xor_sync(0xffffffffu, sp, o);
            klk += __shfl_xor_sync(0xffffffffu, klk, o);
        }
        if ((threadIdx.x & 31) == 0) {
            unsigned long long* S = reinterpret_cast<unsigned long long*>(stats);
            if (inv) atomicAdd(S + SOGK_STAT_INVALID_RAYS, (unsigned long long)inv);
            if (und) atomicAdd(S + SOGK_STAT_UNDEFINED_RAYS, (unsigned long long)und);
            if (lk) atomicAdd(S + SOGK_STAT_ANALYZER_LOOKUPS, (unsigned long long)lk);
            if (sp) atomicAdd(S + SOGK_STAT_ANALYZER_STEPS, (unsigned long long)sp);
            if (klk) atomicAdd(S + SOGK_STAT_KERNEL_LOOKUPS, (unsigned long long)klk);
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

template <int AN, bool CASC, bool BR, int SCH, class Src>
__global__ void __launch_bounds__(kBlock)
    count_kernel(const SamplerDev s, const Src src, int64_t n, int64_t* __restrict__ packed,
                 int64_t* __restrict__ stats, uint8_t* __restrict__ status,
                 int32_t* __restrict__ counters, Resume* __restrict__ resume) {
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    Stats5 acc;
    if (r < n) {
        const Ray ray = src.load(r);
        if (!ray_valid(ray)) {
            count_invalid(r, packed, status, counters, acc);
        } else {
            RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
            gen.init(ray, s);
            long long c = 0;
            Run run;
            for (;;) { // one flat loop: one analyzer step per iteration
                const int st = gen.step(s, run);
                if (st == 0) break;
                if (st == 2) {
                    if (c == 0 && resume) store_resume(resume + r, run);
                    c += run.n;
                }
            }
            count_finish(gen, r, c, packed, status, counters, acc);
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

template <int AN, bool CASC, bool BR, int SCH, bool VEC, class Src>
__global__ void __launch_bounds__(kWriteBlock)
    write_kernel(const SamplerDev s, const Src src, int64_t n, const int64_t* __restrict__ packed,
                 const Resume* __restrict__ resume, int64_t ray_index_base, const Out o) {
    const int64_t r = (int64_t)blockIdx.x * kWriteBlock + threadIdx.x;
    if (r >= n) return;
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + r);
    if (pi.y == 0) return;
    RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
    gen.init(src.load(r), s);
    if (resume) gen.resume(s, resume[r]);
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

// ---------------------------------------------------------------------------
// Persistent-thread variants (the default launch path).  One analyzer event
// per loop iteration and per lane; a lane that finishes its ray immediately
// takes the next ray id from its warp's batch, so warps stay full no matter
// how unevenly the work is spread over rays (0..200 samples, 10..300 events).
// Batches of 32 consecutive ray ids keep neighbouring (coherent) rays in one
// warp; the next batch is prefetched with one atomic so that the refill never
// waits on it.
// ---------------------------------------------------------------------------
constexpr int kPBlock = 128;

struct RayDispenser {
    unsigned long long* ctr;
    long long cur_base;
    int cur_used;
    unsigned long long pf; // lane 0: prefetched next batch base

    __device__ __forceinline__ void init(unsigned long long* c, int lane) {
        ctr = c;
        unsigned long long b = 0;
        if (lane == 0) {
            b = atomicAdd(ctr, 32ull);
            pf = atomicAdd(ctr, 32ull);
        }
        cur_base = (long long)__shfl_sync(0xffffffffu, b, 0);
        cur_used = 0;
    }
    // ray id for this lane if it is in `need` (warp-uniform call)
    __device__ __forceinline__ long long take(unsigned need, int lane) {
        const int k = __popc(need);
        const int rank = __popc(need & ((1u << lane) - 1u));
        const int avail = 32 - cur_used;
        long long id;
        if (k <= avail) {
            id = cur_base + cur_used + rank;
            cur_used += k;
        } else {
            const long long nb = (long long)__shfl_sync(0xffffffffu, pf, 0);
            id = rank < avail ? cur_base + cur_used + rank : nb + (rank - avail);
            cur_base = nb;
            cur_used = k - avail;
            if (lane == 0) pf = atomicAdd(ctr, 32ull);
        }
        return id;
    }
};

template <int AN, bool CASC, bool BR, int SCH, class Src>
__global__ void __launch_bounds__(kPBlock)
    count_persistent(const SamplerDev s, const Src src, int64_t n, int64_t* __restrict__ packed,
                     int64_t* __restrict__ stats, uint8_t* __restrict__ status,
                     int32_t* __restrict__ counters, Resume* __restrict__ resume,
                     unsigned long long* __restrict__ ray_ctr) {
    const int lane = threadIdx.x & 31;
    RayDispenser disp;
    disp.init(ray_ctr, lane);
    RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
    bool have = false, exhausted = false;
    long long r = 0, cnt = 0;
    Stats5 acc;
    for (;;) {
        const unsigned need = __ballot_sync(0xffffffffu, !have);
        bool got = false;
        // refill idle lanes once enough are idle (or the warp has nothing to do)
        if (!exhausted && need && (__popc(need) >= s.refill_min || need == 0xffffffffu)) {
            const long long id = disp.take(need, lane);
            if (!have && id < n) {
                got = true;
                r = id;
                const Ray ray = src.load(r);
                if (!ray_valid(ray)) {
                    count_invalid(r, packed, status, counters, acc);
                } else {
                    gen.init(ray, s);
                    have = true;
                    cnt = 0;
                }
            }
            exhausted = __any_sync(0xffffffffu, !have && !got && ((need >> lane) & 1u));
        }
        if (!__any_sync(0xffffffffu, have)) {
            if (!exhausted) continue;
            break;
        }
        if (have) {
            Run run;
            const int st = gen.step(s, run);
            if (st == 2) {
                if (cnt == 0 && resume) store_resume(resume + r, run);
                cnt += run.n;
            } else if (st == 0) {
                count_finish(gen, r, cnt, packed, status, counters, acc);
                have = false;
            }
        }
    }
    acc.flush(stats);
}

template <int AN, bool CASC, bool BR, int SCH, bool VEC, class Src>
__global__ void __launch_bounds__(kPBlock)
    write_persistent(const SamplerDev s, const Src src, int64_t n, const int64_t* __restrict__ packed,
                     const Resume* __restrict__ resume, int64_t ray_index_base, const Out o,
                     unsigned long long* __restrict__ ray_ctr) {
    const int lane = threadIdx.x & 31;
    RayDispenser disp;
    disp.init(ray_ctr, lane);
    RunGen<BR, SCH, typename PickAn<AN, CASC>::type> gen;
    LaneWriter<SCH, VEC> w;
    bool have = false, exhausted = false;
    for (;;) {
        const unsigned need = __ballot_sync(0xffffffffu, !have);
        bool got = false;
        if (!exhausted && need && (__popc(need) >= s.refill_min || need == 0xffffffffu)) {
            const long long id = disp.take(need, lane);
            if (!have && id < n) {
                got = true;
                const longlong2 pi = __ldg(reinterpret_cast<const longlong2*>(packed) + id);
                if (pi.y > 0) {
                    gen.init(src.load(id), s);
                    if (resume) gen.resume(s, resume[id]);
                    w.start((int32_t)(ray_index_base + id), pi.x, pi.y);
                    have = true;
                }
            }
            exhausted = __any_sync(0xffffffffu, !have && !got && ((need >> lane) & 1u));
        }
        if (!__any_sync(0xffffffffu, have)) {
            if (!exhausted) continue;
            break;
        }
        if (have) {
            if (w.prem == 0) {
                Run run;
                const int st = gen.step(s, run);
                if (st == 2) w.take(run);
                else if (st == 0) w.end = w.out + w.nb; // unreachable when passes agree
            }
            w.emit4(o, s);
            if (w.done()) {
                w.flush(o, s);
                have = false;
            }
        }
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
// resident blocks per SM x SMs (cached per kernel), capped by the work available
static unsigned persistent_grid(const void* kernel, int64_t n) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kPBlock, 0) != cudaSuccess || per_sm <= 0)
        per_sm = 4;
    const int64_t want = (n + 31) / 32 / (kPBlock / 32) + 1;
    int64_t g = (int64_t)sms * per_sm;
    if (g > want) g = want;
    return (unsigned)(g < 1 ? 1 : g);
}

template <class Src>
struct Launch {
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t count(const SamplerDev& s, const Src& src, int64_t n, int64_t* packed,
                             int64_t* stats, uint8_t* status, int32_t* counters, Resume* resume,
                             cudaStream_t st) {
        const int64_t blocks = (n + kBlock - 1) / kBlock;
        count_kernel<AN, CASC, BR, SCH, Src>
            <<<(unsigned)blocks, kBlock, 0, st>>>(s, src, n, packed, stats, status, counters, resume);
        return cudaGetLastError();
    }
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t count_p(const SamplerDev& s, const Src& src, int64_t n, int64_t* packed,
                               int64_t* stats, uint8_t* status, int32_t* counters, Resume* resume,
                               unsigned long long* ctr, cudaStream_t st) {
        auto k = count_persistent<AN, CASC, BR, SCH, Src>;
        const unsigned grid = persistent_grid(reinterpret_cast<const void*>(k), n);
        k<<<grid, kPBlock, 0, st>>>(s, src, n, packed, stats, status, counters, resume, ctr);
        return cudaGetLastError();
    }
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t write_p(const SamplerDev& s, const Src& src, int64_t n, const int64_t* packed,
                               const Resume* resume, int64_t base, double* ts, double* te, int32_t* ri,
                               uint32_t* ce, uint8_t* lv, unsigned long long* ctr, cudaStream_t st) {
        const Out o{ts, te, ri, ce, lv};
        const bool vec = (reinterpret_cast<uintptr_t>(ts) & 31) == 0 &&
                         (reinterpret_cast<uintptr_t>(te) & 31) == 0 &&
                         (reinterpret_cast<uintptr_t>(ri) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(ce) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(lv) & 3) == 0;
        if (vec) {
            auto k = write_persistent<AN, CASC, BR, SCH, true, Src>;
            k<<<persistent_grid(reinterpret_cast<const void*>(k), n), kPBlock, 0, st>>>(s, src, n, packed, resume, base, o, ctr);
        } else {
            auto k = write_persistent<AN, CASC, BR, SCH, false, Src>;
            k<<<persistent_grid(reinterpret_cast<const void*>(k), n), kPBlock, 0, st>>>(s, src, n, packed, resume, base, o, ctr);
        }
        return cudaGetLastError();
    }
    template <int AN, bool CASC, bool BR, int SCH>
    static cudaError_t write(const SamplerDev& s, const Src& src, int64_t n, const int64_t* packed,
                             const Resume* resume, int64_t base, double* ts, double* te, int32_t* ri,
                             uint32_t* ce, uint8_t* lv, cudaStream_t st) {
        const int64_t blocks = (n + kWriteBlock - 1) / kWriteBlock;
        const Out o{ts, te, ri, ce, lv};
        // 256-bit stores need 32-byte aligned bases (16 for the 4-byte arrays)
        const bool vec = (reinterpret_cast<uintptr_t>(ts) & 31) == 0 &&
                         (reinterpret_cast<uintptr_t>(te) & 31) == 0 &&
                         (reinterpret_cast<uintptr_t>(ri) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(ce) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(lv) & 3) == 0;
        if (vec)
            write_kernel<AN, CASC, BR, SCH, true, Src>
                <<<(unsigned)blocks, kWriteBlock, 0, st>>>(s, src, n, packed, resume, base, o);
        else
            write_kernel<AN, CASC, BR, SCH, false, Src>
                <<<(unsigned)blocks, kWriteBlock, 0, st>>>(s, src, n, packed, resume, base, o);
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
                         int64_t* stats, uint8_t* status, int32_t* counters, void* resume,
                         unsigned long long* ctr, cudaStream_t st) {
    Resume* res = static_cast<Resume*>(resume);
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        if (ctr) SOGK_DISPATCH(count_p, s, src, n, packed, stats, status, counters, res, ctr, st);
        SOGK_DISPATCH(count, s, src, n, packed, stats, status, counters, res, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays};
        if (ctr) SOGK_DISPATCH(count_p, s, src, n, packed, stats, status, counters, res, ctr, st);
        SOGK_DISPATCH(count, s, src, n, packed, stats, status, counters, res, st);
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
                         const void* resume, int64_t base, double* ts, double* te, int32_t* ri,
                         uint32_t* ce, uint8_t* lv, unsigned long long* ctr, cudaStream_t st) {
    const Resume* res = static_cast<const Resume*>(resume);
    if (cam) {
        using L = Launch<RaysFromCamera>;
        const RaysFromCamera src{*cam, first};
        if (ctr) SOGK_DISPATCH(write_p, s, src, n, packed, res, base, ts, te, ri, ce, lv, ctr, st);
        SOGK_DISPATCH(write, s, src, n, packed, res, base, ts, te, ri, ce, lv, st);
    } else {
        using L = Launch<RaysFromBuffer>;
        const RaysFromBuffer src{rays};
        if (ctr) SOGK_DISPATCH(write_p, s, src, n, packed, res, base, ts, te, ri, ce, lv, ctr, st);
        SOGK_DISPATCH(write, s, src, n, packed, res, base, ts, te, ri, ce, lv, st);
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
