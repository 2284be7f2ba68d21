// sogk_device.cuh — device-side ray geometry, analyzers and sampling loop.
//
// Bit-exactness contract: every FP64 expression below reproduces the
// reference's operation order (cited per function) and the whole library is
// compiled with -fmad=false, so no a*b+c is contracted into a DFMA.  CUDA's
// double '/', sqrt and floor are IEEE round-to-nearest / exact, matching
// libstdc++ on the host.  Ties, clamps and the degenerate-corner handling
// follow traversal.hpp line by line.
#pragma once

#include <cfloat>
#include <cstdint>

#include "sogk_layout.h"

namespace sogk {

constexpr double kInf = DBL_MAX / 4; // traversal.hpp:19 kInfiniteStep

enum : int { LV_VOXEL = 0, LV_LEAF_TILE = 1, LV_INTERNAL_TILE = 2, LV_ROOT_TILE = 3 };

__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }

struct Ray {
    double o[3], d[3], tmin, tmax;
};

// sog::Ray constructor checks (ray.hpp:98-106); Vec3::length = sqrt(dot) (vec.hpp:23-24)
__device__ __forceinline__ bool ray_valid(const Ray& r) {
    const double len = sqrt(r.d[0] * r.d[0] + r.d[1] * r.d[1] + r.d[2] * r.d[2]);
    if (fabs(len - 1.0) > 1e-9) return false;
    if (!(r.tmin >= 0.0)) return false;
    if (!(r.tmin < r.tmax)) return false;
    return true;
}

// clip_to_box, ray.hpp:121-141 (half-open box)
__device__ __forceinline__ bool clip_to_box(const Ray& r, const double lo[3], const double hi[3],
                                            double& te, double& tx) {
    double t_enter = r.tmin, t_exit = r.tmax;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double d = r.d[a], o = r.o[a];
        if (d == 0.0) {
            if (o < lo[a] || o >= hi[a]) return false;
            continue;
        }
        double ta = (lo[a] - o) / d;
        double tb = (hi[a] - o) / d;
        if (ta > tb) {
            const double t = ta;
            ta = tb;
            tb = t;
        }
        t_enter = std_max(t_enter, ta);
        t_exit = std_min(t_exit, tb);
    }
    if (!(t_enter < t_exit)) return false;
    te = t_enter;
    tx = t_exit;
    return true;
}

// RayGridGeometry, traversal.hpp:27-113
struct Geom {
    double entry[3], dir[3], inv[3];
    int step[3];
    double t_enter, t_exit;
    bool valid;

    __device__ __forceinline__ double plane_t(int a, double plane) const { // :66-68
        return t_enter + (plane - entry[a]) * inv[a];
    }
    __device__ __forceinline__ double grid_coord(int a, double t) const { // :70-72
        return entry[a] + (t - t_enter) * dir[a];
    }

    __device__ __forceinline__ void init(const Ray& r, const GridDev& g) { // :38-64
        valid = false;
        t_enter = 0.0;
        t_exit = 0.0;
        double lo[3], hi[3], te, tx;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = g.wmin[a];
            hi[a] = g.wmin[a] + (double)g.res[a] * g.voxel; // world_max, grid.hpp:36-38
        }
        if (!clip_to_box(r, lo, hi, te, tx)) { // clip_ray, grid.hpp:202-205
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                step[a] = 0;
                entry[a] = dir[a] = inv[a] = 0.0;
            }
            return;
        }
        t_enter = te;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            dir[a] = r.d[a] / g.voxel;
            entry[a] = (r.o[a] + r.d[a] * te - g.wmin[a]) / g.voxel;
            if (dir[a] > 0.0) {
                step[a] = 1;
                inv[a] = 1.0 / dir[a];
            } else if (dir[a] < 0.0) {
                step[a] = -1;
                inv[a] = 1.0 / dir[a];
            } else {
                step[a] = 0;
                inv[a] = kInf;
            }
        }
        t_exit = r.tmax;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (step[a] == 0) continue;
            const double far_plane = step[a] > 0 ? (double)g.res[a] : 0.0;
            t_exit = std_min(t_exit, plane_t(a, far_plane));
        }
        valid = t_enter < t_exit;
    }

    // entry_cell, traversal.hpp:77-85
    __device__ __forceinline__ void entry_cell(const int res[3], int ijk[3]) const {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            double c = floor(entry[a]);
            if (step[a] < 0 && c == entry[a]) c -= 1.0;
            ijk[a] = (int)std_max(0.0, std_min(c, (double)(res[a] - 1)));
        }
    }

    // cell_after_crossing, traversal.hpp:91-104
    __device__ __forceinline__ void cell_after_crossing(double t, int axis, int stepped,
                                                        int ijk[3]) const {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (a == axis) {
                ijk[a] = stepped;
            } else if (step[a] != 0) {
                const double gc = grid_coord(a, t);
                double c = floor(gc);
                if (step[a] < 0 && c == gc) c -= 1.0;
                ijk[a] = (int)c;
            }
        }
    }
};

__device__ __forceinline__ int argmin_axis(double t0, double t1, double t2) { // :107-112
    int axis = 0;
    double m = t0;
    if (t1 < m) {
        axis = 1;
        m = t1;
    }
    if (t2 < m) axis = 2;
    return axis;
}

struct Event {
    int ijk[3];
    int level;
    double t0, t1;
    bool occ;
    int grid_level;
};

__device__ __forceinline__ bool in_bounds(const GridDev& g, const int ijk[3]) {
    return ijk[0] >= 0 && ijk[1] >= 0 && ijk[2] >= 0 && ijk[0] < g.res[0] && ijk[1] < g.res[1] &&
           ijk[2] < g.res[2];
}

// DenseGrid::voxel_at, grid.hpp:129-133
__device__ __forceinline__ bool dense_voxel(const GridDev& g, const int ijk[3]) {
    if (!in_bounds(g, ijk)) return false;
    const uint64_t idx = ((uint64_t)ijk[2] * (uint64_t)g.res[1] + (uint64_t)ijk[1]) *
                             (uint64_t)g.res[0] +
                         (uint64_t)ijk[0];
    return (__ldg(g.bits + (idx >> 3)) >> (idx & 7)) & 1u;
}

// ---------------------------------------------------------------------------
// VDB query: SparseGrid::query / Accessor::query (sparse.hpp:163-214, 228-259)
// over the GPU layout of sogk_layout.h.  The per-thread leaf cache plays the
// role of the reference Accessor's cached leaf; answers are identical.
// ---------------------------------------------------------------------------
struct Query {
    int origin[3];
    int extent;
    int level;
    bool occ;
};

struct VdbCursor {
    int leaf_origin[3];
    int64_t leaf; // cached leaf index, -1 = none

    __device__ __forceinline__ void reset() { leaf = -1; }

    __device__ __forceinline__ Query query(const GridDev& g, const int ijk[3]) {
        Query q;
        if (leaf >= 0 && ijk[0] >= leaf_origin[0] && ijk[1] >= leaf_origin[1] &&
            ijk[2] >= leaf_origin[2] && ijk[0] < leaf_origin[0] + 8 &&
            ijk[1] < leaf_origin[1] + 8 && ijk[2] < leaf_origin[2] + 8) {
            const uint64_t w = __ldg(g.leaves + leaf * 8 + (ijk[2] & 7));
            q.occ = (w >> (((ijk[1] & 7) << 3) | (ijk[0] & 7))) & 1ull;
            q.level = LV_VOXEL;
            q.extent = 1;
            q.origin[0] = ijk[0];
            q.origin[1] = ijk[1];
            q.origin[2] = ijk[2];
            return q;
        }
        if (!in_bounds(g, ijk)) { // background root tile of the 128-aligned region
            q.occ = false;
            q.level = LV_ROOT_TILE;
            q.extent = 128;
            q.origin[0] = (ijk[0] >> 7) << 7; // floor_div (vec.hpp:68-76) * 128
            q.origin[1] = (ijk[1] >> 7) << 7;
            q.origin[2] = (ijk[2] >> 7) << 7;
            return q;
        }
        const int rx = ijk[0] >> 7, ry = ijk[1] >> 7, rz = ijk[2] >> 7;
        const int region = (rz * g.R[1] + ry) * g.R[0] + rx;
        const int32_t node = __ldg(g.root + region);
        if (node < 0) { // root tile (collapsed region)
            q.occ = node == kRootOccupied;
            q.level = LV_INTERNAL_TILE;
            q.extent = 128;
            q.origin[0] = rx << 7;
            q.origin[1] = ry << 7;
            q.origin[2] = rz << 7;
            return q;
        }
        const int cx = (ijk[0] >> 3) & 15, cy = (ijk[1] >> 3) & 15, cz = (ijk[2] >> 3) & 15;
        const int ci = (cz * 16 + cy) * 16 + cx;
        const int64_t wi = (int64_t)node * 64 + (ci >> 6);
        const uint64_t cm = __ldg(g.child_mask + wi);
        const int b = ci & 63;
        if (!((cm >> b) & 1ull)) { // tile child
            q.occ = (__ldg(g.value_mask + wi) >> b) & 1ull;
            q.level = LV_LEAF_TILE;
            q.extent = 8;
            q.origin[0] = ijk[0] & ~7;
            q.origin[1] = ijk[1] & ~7;
            q.origin[2] = ijk[2] & ~7;
            return q;
        }
        leaf = (int64_t)__ldg(g.prefix + wi) + __popcll(cm & ((1ull << b) - 1ull));
        leaf_origin[0] = ijk[0] & ~7;
        leaf_origin[1] = ijk[1] & ~7;
        leaf_origin[2] = ijk[2] & ~7;
        const uint64_t w = __ldg(g.leaves + leaf * 8 + (ijk[2] & 7));
        q.occ = (w >> (((ijk[1] & 7) << 3) | (ijk[0] & 7))) & 1ull;
        q.level = LV_VOXEL;
        q.extent = 1;
        q.origin[0] = ijk[0];
        q.origin[1] = ijk[1];
        q.origin[2] = ijk[2];
        return q;
    }
};

// ---------------------------------------------------------------------------
// Analyzers.  next() returns 1 with an event, 0 at end of stream, and sets
// `undefined` when the HDDA spin guard fires.
// ---------------------------------------------------------------------------
struct DdaAn { // DdaTraversal, traversal.hpp:120-193
    static constexpr bool kHdda = false;
    Geom geom;
    int ijk[3];
    int np[3];
    double tn[3];
    double t_cur;
    int lookups, steps;
    bool done;
    bool undefined;

    __device__ __forceinline__ void init(const Ray& r, const GridDev& g, int /*spin_cap*/) {
        lookups = steps = 0;
        undefined = false;
        geom.init(r, g);
        done = !geom.valid;
        if (done) return;
        geom.entry_cell(g.res, ijk);
        t_cur = geom.t_enter;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (geom.step[a] == 0) {
                np[a] = 0;
                tn[a] = kInf;
            } else {
                np[a] = ijk[a] + (geom.step[a] > 0 ? 1 : 0);
                tn[a] = geom.plane_t(a, (double)np[a]);
            }
        }
    }

    __device__ __forceinline__ void emit(const GridDev& g, double t1, Event& ev) { // :171-175
        ++steps;
        ++lookups;
        ev.ijk[0] = ijk[0];
        ev.ijk[1] = ijk[1];
        ev.ijk[2] = ijk[2];
        ev.level = LV_VOXEL;
        ev.t0 = t_cur;
        ev.t1 = t1;
        ev.occ = dense_voxel(g, ijk);
    }

    __device__ __forceinline__ void advance(const GridDev& g, int axis) { // :177-182
        // select-based updates keep the per-axis arrays in registers
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (a != axis) continue;
            ijk[a] += geom.step[a];
            np[a] += geom.step[a];
            tn[a] = geom.plane_t(a, (double)np[a]);
            if (ijk[a] < 0 || ijk[a] >= g.res[a]) done = true;
        }
    }

    __device__ __forceinline__ int next(const GridDev& g, Event& ev) { // :143-162
        if (done) return 0;
        for (;;) {
            const int axis = argmin_axis(tn[0], tn[1], tn[2]);
            const double t1 = axis == 0 ? tn[0] : (axis == 1 ? tn[1] : tn[2]);
            if (t1 >= geom.t_exit) {
                done = true;
                emit(g, geom.t_exit, ev);
                return 1;
            }
            if (t1 <= t_cur) { // degenerate corner crossing, advance silently
                advance(g, axis);
                if (done) return 0;
                continue;
            }
            emit(g, t1, ev);
            t_cur = t1;
            advance(g, axis);
            return 1;
        }
    }

    __device__ __forceinline__ bool probe(const GridDev& g, const Event& ev) const { // DenseProbe
        return dense_voxel(g, ev.ijk);
    }
};

struct HddaAn { // HddaTraversal, traversal.hpp:199-264
    static constexpr bool kHdda = true;
    Geom geom;
    int ijk[3];
    double t_cur;
    int lookups, steps;
    int spin_cap;
    bool done;
    bool undefined;
    VdbCursor cur;

    __device__ __forceinline__ void init(const Ray& r, const GridDev& g, int cap) {
        lookups = steps = 0;
        undefined = false;
        spin_cap = cap;
        cur.reset();
        geom.init(r, g);
        done = !geom.valid;
        if (done) return;
        geom.entry_cell(g.res, ijk);
        t_cur = geom.t_enter;
    }

    __device__ __forceinline__ int next(const GridDev& g, Event& ev) { // :213-248
        if (done) return 0;
        int degenerate = 0;
        for (;;) {
            const Query q = cur.query(g, ijk);
            ++lookups;
            double tc[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (geom.step[a] == 0) {
                    tc[a] = kInf;
                } else {
                    const double plane = geom.step[a] > 0 ? (double)(q.origin[a] + q.extent)
                                                          : (double)q.origin[a];
                    tc[a] = geom.plane_t(a, plane);
                }
            }
            const int axis = argmin_axis(tc[0], tc[1], tc[2]);
            const double t1 = axis == 0 ? tc[0] : (axis == 1 ? tc[1] : tc[2]);
            ev.ijk[0] = q.origin[0];
            ev.ijk[1] = q.origin[1];
            ev.ijk[2] = q.origin[2];
            ev.level = q.level;
            ev.occ = q.occ;
            if (t1 >= geom.t_exit) {
                ++steps;
                done = true;
                ev.t0 = t_cur;
                ev.t1 = geom.t_exit;
                return 1;
            }
            const int o_ax = axis == 0 ? q.origin[0] : (axis == 1 ? q.origin[1] : q.origin[2]);
            const int s_ax = axis == 0 ? geom.step[0] : (axis == 1 ? geom.step[1] : geom.step[2]);
            const int stepped = s_ax > 0 ? o_ax + q.extent : o_ax - 1;
            if (t1 <= t_cur) { // degenerate corner crossing (:238-241)
                geom.cell_after_crossing(t_cur, axis, stepped, ijk);
                // the reference spins forever at exact edge crossings
                if (++degenerate > spin_cap) {
                    undefined = true;
                    done = true;
                    return 0;
                }
                continue;
            }
            ev.t0 = t_cur;
            ev.t1 = t1;
            ++steps;
            geom.cell_after_crossing(t1, axis, stepped, ijk);
            t_cur = t1;
            return 1;
        }
    }

    __device__ __forceinline__ bool probe(const GridDev& g, const Event& ev) { // SparseProbe
        return cur.query(g, ev.ijk).occ;
    }
};

// CascadeTraversal<GridT>, sampling.hpp:305-415, over SOGK_MAX_LEVELS levels
template <class Sub>
struct CascadeAn {
    static constexpr int kMaxSeg = 2 * SOGK_MAX_LEVELS;
    Ray ray;
    double cut[kMaxSeg + 2];
    signed char seg_level[kMaxSeg + 1];
    int n_seg, seg;
    bool has_sub;
    Sub sub;
    int fin_lookups, fin_steps;
    bool valid;
    bool undefined;
    double t_enter, t_exit;

    __device__ __forceinline__ void init(const Ray& r, const SamplerDev& s) { // :312-355
        ray = r;
        n_seg = 0;
        seg = 0;
        has_sub = false;
        fin_lookups = fin_steps = 0;
        valid = false;
        undefined = false;
        t_enter = t_exit = 0.0;
        const int n = s.n_levels;
        double rf[SOGK_MAX_LEVELS], rs[SOGK_MAX_LEVELS];
        bool hit[SOGK_MAX_LEVELS];
        for (int b = 0; b < n; ++b) hit[b] = clip_to_box(r, s.lv[b].clo, s.lv[b].chi, rf[b], rs[b]);
        if (!hit[n - 1]) return;
        const double te = rf[n - 1], tx = rs[n - 1];
        double cuts[kMaxSeg + 2];
        int nc = 0;
        cuts[nc++] = te;
        cuts[nc++] = tx;
        for (int b = 0; b + 1 < n; ++b) {
            if (!hit[b]) continue;
            if (rf[b] > te && rf[b] < tx) cuts[nc++] = rf[b];
            if (rs[b] > te && rs[b] < tx) cuts[nc++] = rs[b];
        }
        for (int i = 1; i < nc; ++i) { // std::sort
            const double v = cuts[i];
            int j = i - 1;
            while (j >= 0 && cuts[j] > v) {
                cuts[j + 1] = cuts[j];
                --j;
            }
            cuts[j + 1] = v;
        }
        int m = 0; // std::unique
        for (int i = 0; i < nc; ++i)
            if (m == 0 || !(cuts[m - 1] == cuts[i])) cuts[m++] = cuts[i];
        // segments: [cut[k], cut[k+1]) for the kept k; store pairs explicitly
        for (int i = 0; i + 1 < m; ++i) {
            if (!(cuts[i] < cuts[i + 1])) continue;
            const double mid = 0.5 * (cuts[i] + cuts[i + 1]);
            int level = -1;
            for (int b = 0; b < n; ++b)
                if (hit[b] && mid >= rf[b] && mid < rs[b]) {
                    level = b;
                    break;
                }
            cut[n_seg] = cuts[i];
            cut[n_seg + 1] = cuts[i + 1]; // consecutive kept segments share this boundary
            seg_level[n_seg] = (signed char)level;
            ++n_seg;
        }
        valid = n_seg > 0;
        t_enter = te;
        t_exit = tx;
    }

    __device__ __forceinline__ int next(const SamplerDev& s, Event& ev) { // :361-392
        for (;;) {
            if (has_sub) {
                const int gl = seg_level[seg];
                if (sub.next(s.lv[gl], ev)) {
                    ev.grid_level = gl;
                    return 1;
                }
                if (sub.undefined) {
                    undefined = true;
                    return 0;
                }
                fin_lookups += sub.lookups;
                fin_steps += sub.steps;
                has_sub = false;
                ++seg;
            }
            if (seg >= n_seg) return 0;
            const int gl = seg_level[seg];
            if (gl < 0) { // outside every level: one empty event
                ev.ijk[0] = ev.ijk[1] = ev.ijk[2] = 0;
                ev.level = LV_ROOT_TILE;
                ev.t0 = cut[seg];
                ev.t1 = cut[seg + 1];
                ev.occ = false;
                ev.grid_level = -1;
                ++seg;
                ++fin_steps;
                return 1;
            }
            Ray sr = ray;
            sr.tmin = cut[seg];
            sr.tmax = cut[seg + 1];
            sub.init(sr, s.lv[gl], s.spin_cap);
            has_sub = true;
        }
    }

    __device__ __forceinline__ int lookup_count() const {
        return fin_lookups + (has_sub ? sub.lookups : 0);
    }
    __device__ __forceinline__ int step_count() const {
        return fin_steps + (has_sub ? sub.steps : 0);
    }

    __device__ __forceinline__ bool probe(const SamplerDev& s, const Event& ev) { // CascadeProbe
        if (ev.grid_level < 0) return false;
        if constexpr (Sub::kHdda) {
            VdbCursor c;
            c.reset();
            return c.query(s.lv[ev.grid_level], ev.ijk).occ;
        } else {
            return dense_voxel(s.lv[ev.grid_level], ev.ijk);
        }
    }
};

// Uniform facade over single-grid and cascade analyzers.
template <class Sub, bool Cascade>
struct AnyAn;

template <class Sub>
struct AnyAn<Sub, false> {
    Sub an;
    __device__ __forceinline__ void init(const Ray& r, const SamplerDev& s) {
        an.init(r, s.lv[0], s.spin_cap);
    }
    __device__ __forceinline__ bool valid() const { return an.geom.valid; }
    __device__ __forceinline__ double t_enter() const { return an.geom.t_enter; }
    __device__ __forceinline__ double t_exit() const { return an.geom.t_exit; }
    __device__ __forceinline__ int next(const SamplerDev& s, Event& ev) {
        const int r = an.next(s.lv[0], ev);
        ev.grid_level = 0;
        return r;
    }
    __device__ __forceinline__ bool undefined() const { return an.undefined; }
    __device__ __forceinline__ int lookups() const { return an.lookups; }
    __device__ __forceinline__ int steps() const { return an.steps; }
    __device__ __forceinline__ bool probe(const SamplerDev& s, const Event& ev) {
        return an.probe(s.lv[0], ev);
    }
};

template <class Sub>
struct AnyAn<Sub, true> {
    CascadeAn<Sub> an;
    __device__ __forceinline__ void init(const Ray& r, const SamplerDev& s) { an.init(r, s); }
    __device__ __forceinline__ bool valid() const { return an.valid; }
    __device__ __forceinline__ double t_enter() const { return an.t_enter; }
    __device__ __forceinline__ double t_exit() const { return an.t_exit; }
    __device__ __forceinline__ int next(const SamplerDev& s, Event& ev) { return an.next(s, ev); }
    __device__ __forceinline__ bool undefined() const { return an.undefined; }
    __device__ __forceinline__ int lookups() const { return an.lookup_count(); }
    __device__ __forceinline__ int steps() const { return an.step_count(); }
    __device__ __forceinline__ bool probe(const SamplerDev& s, const Event& ev) {
        return an.probe(s, ev);
    }
};

// StepSchedule::step, sampling.hpp:36-38
template <int Sched>
__device__ __forceinline__ double sched_step(const SamplerDev& s, double t) {
    if constexpr (Sched == SOGK_CONSTANT_SCHED)
        return s.dt0;
    else
        return std_max(s.dt0, s.growth * t);
}

__device__ __forceinline__ uint32_t pack_cell(const int ijk[3]) {
    return (uint32_t)(ijk[0] & 1023) | ((uint32_t)(ijk[1] & 1023) << 10) |
           ((uint32_t)(ijk[2] & 1023) << 20);
}

// sample_branch / sample_skip, sampling.hpp:87-122.  Sink::emit(t, t_next, ev)
// returns false to stop early (the write pass stops once the ray's count is
// written).  kernel_lookups counts probe calls like the reference probes.
template <bool Branch, int Sched, class An, class Sink>
__device__ __forceinline__ void run_kernel(An& an, const SamplerDev& s, Sink& sink,
                                           int& kernel_lookups) {
    if (!an.valid()) return;
    const double t_end = an.t_exit();
    double t_last = an.t_enter();
    Event ev;
    while (t_last <= t_end) {
        if (!an.next(s, ev)) break;
        if (!Branch && !ev.occ) continue;
        while (t_last <= ev.t0) t_last += sched_step<Sched>(s, t_last);
        while (t_last <= ev.t1) {
            const double nx = t_last + sched_step<Sched>(s, t_last);
            bool emit = true;
            if (Branch) {
                ++kernel_lookups;
                emit = an.probe(s, ev);
            }
            if (emit && !sink.emit(t_last, nx, ev)) return;
            t_last = nx;
        }
    }
}

} // namespace sogk
