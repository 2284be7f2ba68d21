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
#include <type_traits>

#include "sogk_ladder.cuh"
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
            // x / voxel; for a power-of-two voxel this equals x * (1/voxel) exactly
            dir[a] = g.voxel_pow2 ? r.d[a] * g.inv_voxel : r.d[a] / g.voxel;
            const double num = r.o[a] + r.d[a] * te - g.wmin[a];
            entry[a] = g.voxel_pow2 ? num * g.inv_voxel : num / g.voxel;
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

struct Event {
    int ijk[3];
    int level;
    double t0, t1;
    bool occ;
    int grid_level;
};

__device__ __forceinline__ bool in_bounds(const GridDev& g, const int ijk[3]) {
    return (unsigned)ijk[0] < (unsigned)g.res[0] && (unsigned)ijk[1] < (unsigned)g.res[1] &&
           (unsigned)ijk[2] < (unsigned)g.res[2];
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
// A query answer.  Every node the reference returns is aligned to its extent
// (region_origin = floor_div(ijk, 128) * 128, tile/leaf origins ijk & ~7, voxels ijk),
// so the origin is always ijk & -extent and is not carried.
struct Query {
    int ext;   // 1, 8 or 128
    int level;
    bool occ;
};

constexpr int kNoLeaf = -(1 << 29); // leaf-cache origin that no coordinate can hit

// dynamic shared memory of the launching kernel (the staged child table when GridDev::smem_tab)
extern __shared__ int32_t sogk_dyn_smem[];

#ifndef SOGK_QUERY_CACHE
#define SOGK_QUERY_CACHE 0 // 1: per-thread cached leaf (divergent miss path); 0: uniform walk
#endif

#ifndef SOGK_SMEM_TABLE
#define SOGK_SMEM_TABLE 0 // 1: pass 1 stages a single-region VDB's child table in shared memory
#endif

// child table entry ci of `node` (the root entry of an in-grid region, >= 0)
__device__ __forceinline__ int32_t table_at(const GridDev& g, int32_t node, int ci) {
#if SOGK_SMEM_TABLE
    if (g.smem_tab) return sogk_dyn_smem[ci];
#endif
    return __ldg(g.table + (int64_t)node * 4096 + ci);
}

struct VdbCursor {
    int lo[3];       // cached leaf origin (kNoLeaf: none)
    int64_t leaf;    // cached leaf index

    __device__ __forceinline__ void reset() { lo[0] = lo[1] = lo[2] = kNoLeaf; leaf = 0; }

    // ONE: 1 = single-region grid (the root entry is the kernel parameter g.node0), 0 = read the
    // root, -1 = decide at run time from g.node0 (a warp-uniform branch)
    template <int ONE = -1>
    __device__ __forceinline__ Query query(const GridDev& g, const int ijk[3]) {
        Query q;
#if SOGK_QUERY_CACHE
        const unsigned lx = (unsigned)(ijk[0] - lo[0]), ly = (unsigned)(ijk[1] - lo[1]),
                       lz = (unsigned)(ijk[2] - lo[2]);
        if ((lx | ly | lz) >= 8u) { // not the cached leaf (Accessor fast path, sparse.hpp:229-233)
            q.occ = false;
            q.level = LV_ROOT_TILE;
            q.ext = 128;
            if (!in_bounds(g, ijk)) return q; // background root tile at region_origin (:164-165)
            const int region = ((ijk[2] >> 7) * g.R[1] + (ijk[1] >> 7)) * g.R[0] + (ijk[0] >> 7);
            const int32_t node = __ldg(g.root + region);
            q.level = LV_INTERNAL_TILE;
            if (node < 0) { // collapsed region (root tile)
                q.occ = node == kRootOccupied;
                return q;
            }
            const int ci = ((((ijk[2] >> 3) & 15) * 16 + ((ijk[1] >> 3) & 15)) * 16) + ((ijk[0] >> 3) & 15);
            const int32_t code = table_at(g, node, ci); // child table
            if (code < 0) { // tile child (:205-208)
                q.occ = code == kTileOccupied;
                q.level = LV_LEAF_TILE;
                q.ext = 8;
                return q;
            }
            leaf = code;
            lo[0] = ijk[0] & ~7;
            lo[1] = ijk[1] & ~7;
            lo[2] = ijk[2] & ~7;
        }
        // the leaf word of ijk (cached leaf or just found)
        const uint64_t w = __ldg(g.leaves + leaf * 8 + (ijk[2] & 7));
        q.occ = (w >> (((ijk[1] & 7) << 3) | (ijk[0] & 7))) & 1ull;
        q.level = LV_VOXEL;
        q.ext = 1;
        return q;
#else
        // Uniform walk, no per-lane cache: root -> child table -> leaf word for every lane and
        // every query, the loads made unconditional by clamping to valid entries and the answer
        // picked with selects.  A per-lane leaf cache makes the miss path divergent: neighbouring
        // rays leave their leaves on different iterations, so most warp iterations ran the
        // ~45-instruction miss path for a handful of lanes (ncu: 3-10 of 32 active).
        const bool inb = in_bounds(g, ijk);
        int32_t node;
        if (ONE == 1 || (ONE < 0 && SOGK_NODE0 && g.node0 != kNodeMulti)) { // single region
            node = g.node0;
        } else {
            const int region = inb ? ((ijk[2] >> 7) * g.R[1] + (ijk[1] >> 7)) * g.R[0] + (ijk[0] >> 7) : 0;
            node = __ldg(g.root + region);
        }
        const int ci = ((((ijk[2] >> 3) & 15) * 16 + ((ijk[1] >> 3) & 15)) * 16) + ((ijk[0] >> 3) & 15);
        const int32_t code = table_at(g, node < 0 ? 0 : node, ci);
        const uint64_t w = __ldg(g.leaves + (int64_t)(code < 0 ? 0 : code) * 8 + (ijk[2] & 7));
        const bool bit = (w >> (((ijk[1] & 7) << 3) | (ijk[0] & 7))) & 1ull;
        const bool leafv = inb && node >= 0 && code >= 0;
        const bool tile = inb && node >= 0 && code < 0;
        q.ext = leafv ? 1 : (tile ? 8 : 128);
        q.level = !inb ? LV_ROOT_TILE : (node < 0 ? LV_INTERNAL_TILE : (code < 0 ? LV_LEAF_TILE : LV_VOXEL));
        // root tile: empty; collapsed region: its value; tile child: its value; leaf: the bit
        q.occ = inb && (node < 0 ? node == kRootOccupied : (code < 0 ? code == kTileOccupied : bit));
        return q;
#endif
    }
};

// argmin with ties toward the lowest axis (argmin_axis, traversal.hpp:107-112),
// written as compare-and-select so that no branch is emitted
__device__ __forceinline__ int argmin3(double a, double b, double c, double& m) {
    int axis = 0;
    m = a;
    if (b < m) {
        m = b;
        axis = 1;
    }
    if (c < m) {
        m = c;
        axis = 2;
    }
    return axis;
}

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
    int64_t lin;        // linear voxel index of ijk (x-fastest), kept incrementally
    int64_t stride[3];  // signed linear-index step per axis
    int lookups, steps;
    bool done;
    bool undefined;

    __device__ __forceinline__ void set_lin(const GridDev& g) {
        lin = ((int64_t)ijk[2] * g.res[1] + ijk[1]) * g.res[0] + ijk[0];
        stride[0] = geom.step[0];
        stride[1] = (int64_t)geom.step[1] * g.res[0];
        stride[2] = (int64_t)geom.step[2] * g.res[0] * g.res[1];
    }

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
            np[a] = ijk[a] + (geom.step[a] > 0 ? 1 : 0);
            tn[a] = geom.step[a] == 0 ? kInf : geom.plane_t(a, (double)np[a]);
        }
        set_lin(g);
    }

    // ijk is always inside the grid while the stream is live (entry_cell clamps,
    // advance() ends the stream on leaving), so the lookup needs no bounds test
    __device__ __forceinline__ void emit(const GridDev& g, double t1, Event& ev) { // :171-175
        ++steps;
        ++lookups;
        ev.ijk[0] = ijk[0];
        ev.ijk[1] = ijk[1];
        ev.ijk[2] = ijk[2];
        ev.level = LV_VOXEL;
        ev.t0 = t_cur;
        ev.t1 = t1;
        ev.occ = (__ldg(g.bits + (lin >> 3)) >> (lin & 7)) & 1u;
    }

    __device__ __forceinline__ void advance(const GridDev& g, int axis) { // :177-182
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (a == axis) {
                ijk[a] += geom.step[a];
                np[a] += geom.step[a];
                tn[a] = geom.plane_t(a, (double)np[a]);
                lin += stride[a];
                if ((unsigned)ijk[a] >= (unsigned)g.res[a]) done = true;
            }
        }
    }

    // One iteration of DdaTraversal::next's loop (:143-162): 1 = event, 0 = end of
    // stream, -1 = degenerate corner crossing consumed (call again).  Callers
    // loop; keeping the retry out of here keeps kernels to one flat loop.
    __device__ __forceinline__ int next(const GridDev& g, Event& ev) {
        if (done) return 0;
        double t1;
        const int axis = argmin3(tn[0], tn[1], tn[2], t1);
        if (t1 >= geom.t_exit) {
            done = true;
            emit(g, geom.t_exit, ev);
            return 1;
        }
        if (t1 <= t_cur) { // degenerate corner crossing, advance silently
            advance(g, axis);
            return done ? 0 : -1;
        }
        emit(g, t1, ev);
        t_cur = t1;
        advance(g, axis);
        return 1;
    }

    __device__ __forceinline__ bool probe(const GridDev& g, const Event& ev) const { // DenseProbe
        return dense_voxel(g, ev.ijk);
    }

    __device__ __forceinline__ bool is_valid() const { return geom.valid; }
    __device__ __forceinline__ double enter_t() const { return geom.t_enter; }
    __device__ __forceinline__ double exit_t() const { return geom.t_exit; }

    // Resume at an emitted event: (ijk, t_cur) = (ev.ijk, ev.t0) reproduces it.
    __device__ __forceinline__ void restore(const GridDev& g, const int in_ijk[3], double in_t) {
        done = false;
        t_cur = in_t;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            ijk[a] = in_ijk[a];
            np[a] = ijk[a] + (geom.step[a] > 0 ? 1 : 0);
            tn[a] = geom.step[a] == 0 ? kInf : geom.plane_t(a, (double)np[a]);
        }
        set_lin(g);
    }
};

// HddaTraversal, traversal.hpp:199-264.
//
// The loop runs in per-axis mirrored coordinates: an axis the ray walks down is
// negated (entry' = -entry, dir' = -dir, inv' = -inv, plane' = -plane), so every
// moving axis walks up.  Negation is exact and round-to-nearest is symmetric, so
//   plane_t:    t_enter + (plane' - entry') * inv'  ==  t_enter + (plane - entry) * inv
//   grid_coord: entry' + dt * dir'                  == -(entry + dt * dir)
// bit for bit, and cell_after_crossing's "floor, minus one on an exact plane
// when walking down" (traversal.hpp:96-100) becomes ~floor(grid_coord') there:
//   ceil(x) - 1 == -floor(-x) - 1 == ~floor(-x).
// A static axis (dir == 0) gets entry' = cell + 0.5, dir' = 0, inv' = +inf: its
// exit time is +inf (the reference's kInfiniteStep: only ever compared, never the
// minimum of a valid ray) and its re-derived cell is its constant cell.
#ifndef SOGK_HDDA_SMEM
#define SOGK_HDDA_SMEM 1
#endif
// Kernels using the node analyzers or the cascade launch 1-D blocks of at most kGeomBlock
// threads (per-thread shared-memory columns).
#ifndef SOGK_BLOCK
#define SOGK_BLOCK 128 // threads per block of the traversal kernels (pass 1, tail, cold write, traverse)
#endif
constexpr int kGeomBlock = SOGK_BLOCK;
#if SOGK_HDDA_SMEM
// The per-ray geometry lives in shared memory (one column per thread, SoA: conflict-free),
// which keeps ~22 registers out of the traversal loop.
struct HddaGeomSmem {
    double e[3][kGeomBlock], dv[3][kGeomBlock], iv[3][kGeomBlock];
    double te[kGeomBlock], tx[kGeomBlock];
    int m[3][kGeomBlock];
};
__device__ __forceinline__ HddaGeomSmem& hdda_geom() {
    __shared__ HddaGeomSmem g;
    return g;
}
#endif

// The same loop serves CdTraversal (traversal.hpp:270-337, CD = true): its "node" is the
// cube of half-width d-1 around the voxel (d = chessboard distance, proven empty), with
// low corner ijk - (d-1) instead of an extent-aligned VDB node; everything else -- exit
// planes, argmin, clamp to t_exit, degenerate re-derivation, spin guard -- is identical.
template <bool CD, int ONE = -1> // ONE: VdbCursor::query's single-region mode
struct NodeAn {
    static constexpr bool kHdda = !CD;
#if SOGK_HDDA_SMEM
    __device__ __forceinline__ double& E(int a) { return hdda_geom().e[a][threadIdx.x]; }
    __device__ __forceinline__ double& DV(int a) { return hdda_geom().dv[a][threadIdx.x]; }
    __device__ __forceinline__ double& IV(int a) { return hdda_geom().iv[a][threadIdx.x]; }
    __device__ __forceinline__ int& M(int a) { return hdda_geom().m[a][threadIdx.x]; }
    __device__ __forceinline__ double& TE() { return hdda_geom().te[threadIdx.x]; }
    __device__ __forceinline__ double& TX() { return hdda_geom().tx[threadIdx.x]; }
    __device__ __forceinline__ double TE() const { return hdda_geom().te[threadIdx.x]; }
    __device__ __forceinline__ double TX() const { return hdda_geom().tx[threadIdx.x]; }
#else
    double e[3], dv[3], iv[3]; // mirrored entry, |dir|, 1/|dir|
    int m[3];                  // -1 on mirrored axes, else 0
    double t_enter, t_exit;
    __device__ __forceinline__ double& E(int a) { return e[a]; }
    __device__ __forceinline__ double& DV(int a) { return dv[a]; }
    __device__ __forceinline__ double& IV(int a) { return iv[a]; }
    __device__ __forceinline__ int& M(int a) { return m[a]; }
    __device__ __forceinline__ double& TE() { return t_enter; }
    __device__ __forceinline__ double& TX() { return t_exit; }
    __device__ __forceinline__ double TE() const { return t_enter; }
    __device__ __forceinline__ double TX() const { return t_exit; }
#endif
    bool valid;
    int ijk[3];
    double t_cur;
    int lookups, steps;
    int spin_cap;
    int degenerate; // consecutive degenerate iterations
    bool done;
    bool undefined;
    VdbCursor cur;

    __device__ __forceinline__ void init(const Ray& r, const GridDev& g, int cap) {
        lookups = steps = 0;
        undefined = false;
        spin_cap = cap;
        degenerate = 0;
        cur.reset();
        Geom geom;
        geom.init(r, g);
        valid = geom.valid;
        TE() = geom.t_enter;
        TX() = geom.t_exit;
        done = !valid;
        if (done) return;
        geom.entry_cell(g.res, ijk);
        t_cur = geom.t_enter;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (geom.step[a] > 0) {
                E(a) = geom.entry[a];
                DV(a) = geom.dir[a];
                IV(a) = geom.inv[a];
                M(a) = 0;
            } else if (geom.step[a] < 0) {
                E(a) = -geom.entry[a];
                DV(a) = -geom.dir[a];
                IV(a) = -geom.inv[a];
                M(a) = -1;
            } else {
                E(a) = (double)ijk[a] + 0.5;
                DV(a) = 0.0;
                IV(a) = __longlong_as_double(0x7ff0000000000000ll); // +inf
                M(a) = 0;
            }
        }
    }

    // One iteration of HddaTraversal::next's loop (:213-248): 1 = event, 0 = end,
    // -1 = degenerate iteration consumed (call again).
    __device__ __forceinline__ int next(const GridDev& g, Event& ev) {
        if (done) return 0;
        Query q;
        int half = 0;
        if constexpr (CD) { // DistanceGrid::at: out of bounds reads 1 (distance.hpp:27-30)
            const int32_t d = in_bounds(g, ijk)
                                  ? __ldg(g.dist + ((int64_t)ijk[2] * g.res[1] + ijk[1]) * g.res[0] + ijk[0])
                                  : 1;
            half = d > 1 ? d - 1 : 0;
            q.ext = 2 * half + 1;
            q.level = LV_VOXEL;
            q.occ = d == 0;
        } else {
            q = cur.template query<ONE>(g, ijk);
        }
        ++lookups;
        // exit plane of the node on each axis (:218-228), mirrored: lo + ext walking up,
        // -lo walking down; the cell just past it (`stepped`, :236-237) is plane' ^ m
        const double te = TE();
        double tc[3];
        int pl[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int lo = CD ? ijk[a] - half : (ijk[a] & -q.ext);
            ev.ijk[a] = lo;
            pl[a] = (lo ^ M(a)) + (M(a) ? 1 : q.ext);
            tc[a] = te + ((double)pl[a] - E(a)) * IV(a);
        }
        double t1;
        const int axis = argmin3(tc[0], tc[1], tc[2], t1);
        ev.level = q.level;
        ev.occ = q.occ;
        const double tx = TX();
        if (t1 >= tx) {
            ++steps;
            done = true;
            ev.t0 = t_cur;
            ev.t1 = tx;
            return 1;
        }
        const bool degen = t1 <= t_cur; // degenerate corner crossing (:238-241)
        // cell_after_crossing (:91-104) at t_cur (degenerate) or t1, all axes
        // evaluated and the stepped one overridden
        const double dt = (degen ? t_cur : t1) - te;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int c = __double2int_rd(E(a) + dt * DV(a)) ^ M(a);
            ijk[a] = (a == axis) ? (pl[a] ^ M(a)) : c;
        }
        if (degen) {
            // the reference spins forever at exact edge crossings
            if (++degenerate > spin_cap) {
                undefined = true;
                done = true;
                return 0;
            }
            return -1;
        }
        degenerate = 0;
        ev.t0 = t_cur;
        ev.t1 = t1;
        ++steps;
        t_cur = t1;
        return 1;
    }

    __device__ __forceinline__ bool probe(const GridDev& g, const Event& ev) { // SparseProbe
        if constexpr (CD) return ev.occ; // DenseProbe at the cube's low corner == (d == 0)
        else return cur.query(g, ev.ijk).occ;
    }

    // Resume at an emitted event: the node origin queries the same node, so
    // (ijk, t_cur) = (ev.ijk, ev.t0) reproduces it.
    __device__ __forceinline__ void restore(const GridDev&, const int in_ijk[3], double in_t) {
        done = false;
        degenerate = 0;
        t_cur = in_t;
        ijk[0] = in_ijk[0];
        ijk[1] = in_ijk[1];
        ijk[2] = in_ijk[2];
        cur.reset(); // the accessor cache is semantically transparent
    }

    __device__ __forceinline__ bool is_valid() const { return valid; }
    __device__ __forceinline__ double enter_t() const { return TE(); }
    __device__ __forceinline__ double exit_t() const { return TX(); }
};

using HddaAn = NodeAn<false>;
using CdAn = NodeAn<true>;

// CascadeTraversal<GridT>, sampling.hpp:305-415, over SOGK_MAX_LEVELS levels.
// Every loop over levels and cuts has a fixed trip count (unrolled, guarded by n_levels)
// and the cut list is sorted by a sorting network, so nothing here is dynamically indexed
// in registers: the sorted cut list and the ray live in per-thread shared-memory columns,
// the segment levels in one packed register.  (Dynamic indexing sent the whole analyzer,
// sub-analyzer included, to local memory.)
constexpr int kCascadeCuts = 2 * SOGK_MAX_LEVELS; // te, tx + 2 per inner level

struct CascadeSmem {
    double cut[kCascadeCuts][kGeomBlock];
    double od[6][kGeomBlock]; // ray origin, direction
};
__device__ __forceinline__ CascadeSmem& cascade_smem() {
    __shared__ CascadeSmem c;
    return c;
}

__device__ __forceinline__ void cmp_swap(double& a, double& b) {
    const double lo = (b < a) ? b : a, hi = (b < a) ? a : b;
    a = lo;
    b = hi;
}

template <class Sub>
struct CascadeAn {
    unsigned seg_lv;       // 3 bits per segment: grid level + 1 (0: outside every level)
    int n_seg, seg;
    bool has_sub;
    int cur_gl;            // grid level of the open segment
    const GridDev* cur_g;  // &s.lv[cur_gl] (a __grid_constant__ parameter)
    Sub sub;
    int fin_lookups, fin_steps;
    bool valid;
    bool undefined;
    double t_enter, t_exit;

    __device__ __forceinline__ double& CUT(int i) { return cascade_smem().cut[i][threadIdx.x]; }

    __device__ __forceinline__ void init(const Ray& r, const SamplerDev& s) { // :312-355
        n_seg = 0;
        seg = 0;
        seg_lv = 0;
        has_sub = false;
        fin_lookups = fin_steps = 0;
        valid = false;
        undefined = false;
        t_enter = t_exit = 0.0;
        const int n = s.n_levels;
        double rf[SOGK_MAX_LEVELS], rs[SOGK_MAX_LEVELS];
        bool hit[SOGK_MAX_LEVELS];
        double te = 0.0, tx = 0.0;
        bool hit_last = false;
#pragma unroll
        for (int b = 0; b < SOGK_MAX_LEVELS; ++b) {
            rf[b] = rs[b] = 0.0;
            hit[b] = b < n && clip_to_box(r, s.lv[b].clo, s.lv[b].chi, rf[b], rs[b]);
            if (b == n - 1) {
                hit_last = hit[b];
                te = rf[b];
                tx = rs[b];
            }
        }
        if (!hit_last) return;
        // cuts: te, tx and every inner boundary strictly inside (te, tx); +inf = absent
        const double inf = __longlong_as_double(0x7ff0000000000000ll);
        double c[kCascadeCuts];
        c[0] = te;
        c[1] = tx;
#pragma unroll
        for (int b = 0; b + 1 < SOGK_MAX_LEVELS; ++b) {
            const bool use = b + 1 < n && hit[b];
            c[2 + 2 * b] = (use && rf[b] > te && rf[b] < tx) ? rf[b] : inf;
            c[3 + 2 * b] = (use && rs[b] > te && rs[b] < tx) ? rs[b] : inf;
        }
        // std::sort: odd-even transposition network (fixed size, all indices constant)
#pragma unroll
        for (int pass = 0; pass < kCascadeCuts; ++pass) {
#pragma unroll
            for (int i = pass & 1; i + 1 < kCascadeCuts; i += 2) cmp_swap(c[i], c[i + 1]);
        }
        // std::unique, then one segment per consecutive pair; level = the finest level whose
        // voxel-centre box holds the segment midpoint (:340-351)
        int m = 0;
        double prev = 0.0;
#pragma unroll
        for (int i = 0; i < kCascadeCuts; ++i) {
            const double v = c[i];
            if (v == inf) continue;
            if (m > 0 && v == prev) continue;
            if (m > 0) {
                const double mid = 0.5 * (prev + v);
                int level = -1;
#pragma unroll
                for (int b = SOGK_MAX_LEVELS - 1; b >= 0; --b)
                    if (b < n && hit[b] && mid >= rf[b] && mid < rs[b]) level = b;
                seg_lv |= (unsigned)(level + 1) << (3 * (m - 1));
            }
            CUT(m) = v;
            prev = v;
            ++m;
        }
        n_seg = m - 1;
        CascadeSmem& cs = cascade_smem();
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            cs.od[a][threadIdx.x] = r.o[a];
            cs.od[3 + a][threadIdx.x] = r.d[a];
        }
        valid = n_seg > 0;
        t_enter = te;
        t_exit = tx;
    }

    __device__ __forceinline__ int seg_level(int i) const { return (int)((seg_lv >> (3 * i)) & 7u) - 1; }

    __device__ __forceinline__ void open_sub(const SamplerDev& s) {
        Ray sr; // Ray(origin, dir, seg.t0, seg.t1) (:389-390)
        const CascadeSmem& cs = cascade_smem();
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            sr.o[a] = cs.od[a][threadIdx.x];
            sr.d[a] = cs.od[3 + a][threadIdx.x];
        }
        sr.tmin = CUT(seg);
        sr.tmax = CUT(seg + 1);
        cur_gl = seg_level(seg);
        cur_g = &s.lv[cur_gl];
        sub.init(sr, *cur_g, s.spin_cap);
        has_sub = true;
    }

    // One action of CascadeTraversal::next (:361-392): 1 = event, 0 = end,
    // -1 = internal transition (sub-analyzer step, segment change) — call again.
    __device__ __forceinline__ int next(const SamplerDev& s, Event& ev) {
        if (has_sub) {
            const int r = sub.next(*cur_g, ev);
            if (r != 0) {
                ev.grid_level = cur_gl;
                return r;
            }
            if (sub.undefined) {
                undefined = true;
                return 0;
            }
            fin_lookups += sub.lookups;
            fin_steps += sub.steps;
            has_sub = false;
            ++seg;
            return -1;
        }
        if (seg >= n_seg) return 0;
        const int gl = seg_level(seg);
        if (gl < 0) { // outside every level: one empty event
            ev.ijk[0] = ev.ijk[1] = ev.ijk[2] = 0;
            ev.level = LV_ROOT_TILE;
            ev.t0 = CUT(seg);
            ev.t1 = CUT(seg + 1);
            ev.occ = false;
            ev.grid_level = -1;
            ++seg;
            ++fin_steps;
            return 1;
        }
        open_sub(s);
        return -1;
    }

    // resume inside the sub-analyzer of the current segment
    __device__ __forceinline__ int resume_tag() const { return seg; }
    __device__ __forceinline__ void restore(const SamplerDev& s, int tag, const int in_ijk[3],
                                            double in_t) {
        seg = tag;
        open_sub(s);
        sub.restore(*cur_g, in_ijk, in_t);
    }

    __device__ __forceinline__ int lookup_count() const {
        return fin_lookups + (has_sub ? sub.lookups : 0);
    }
    __device__ __forceinline__ int step_count() const {
        return fin_steps + (has_sub ? sub.steps : 0);
    }

    __device__ __forceinline__ bool probe(const SamplerDev& s, const Event& ev) { // CascadeProbe
        if (ev.grid_level < 0) return false;
        if constexpr (std::is_same<Sub, CdAn>::value) {
            return ev.occ;
        } else if constexpr (Sub::kHdda) {
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
    __device__ __forceinline__ bool valid() const { return an.is_valid(); }
    __device__ __forceinline__ double t_enter() const { return an.enter_t(); }
    __device__ __forceinline__ double t_exit() const { return an.exit_t(); }
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
    __device__ __forceinline__ int resume_tag() const { return 0; }
    __device__ __forceinline__ void restore(const SamplerDev& s, int, const int ijk[3], double t) {
        an.restore(s.lv[0], ijk, t);
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
    __device__ __forceinline__ int resume_tag() const { return an.resume_tag(); }
    __device__ __forceinline__ void restore(const SamplerDev& s, int tag, const int ijk[3], double t) {
        an.restore(s, tag, ijk, t);
    }
};

__device__ __forceinline__ uint32_t pack_cell(const int ijk[3]) {
    return (uint32_t)(ijk[0] & 1023) | ((uint32_t)(ijk[1] & 1023) << 10) |
           ((uint32_t)(ijk[2] & 1023) << 20);
}

// A run: the ladder points one event contributes, S[first .. first + n).
struct Run {
    double first;  // first ladder point > ev.t0
    int n;         // ladder points in (ev.t0, ev.t1]
    uint32_t cell;
    uint8_t level; // Level | grid_level << 2
    // resume point of the event (written by pass 1 for the ray's first run)
    int ijk[3];
    int tag;
    double t0, t_last0;
};


// sample_branch / sample_skip (sampling.hpp:87-122) as a generator of runs.
// Identical control flow to the reference kernels -- the outer loop pulls an
// event while t_last <= t_exit, the skip kernel ignores unoccupied events, the
// branch kernel walks all of them -- but the ladder is advanced per event in
// closed form (sogk_ladder.cuh) instead of point by point.  The branch
// kernel's per-point probe returns the same answer for every point of an
// event (same ijk), so it is evaluated once per event and counted n times
// (kernel_lookups), exactly as many probes as the reference makes.
template <bool Branch, int Sched, class An>
struct RunGen {
    An an;
    double t_last, t_end;
    int kernel_lookups;
    bool alive;
    bool stalled;

    __device__ __forceinline__ void init(const Ray& r, const SamplerDev& s) {
        an.init(r, s);
        kernel_lookups = 0;
        stalled = false;
        alive = an.valid();
        t_last = an.t_enter();
        t_end = an.t_exit();
    }

    // One analyzer call (one event) for callers that emit the samples themselves:
    // 0 = ray finished, 1 = nothing to emit, 2 = occupied event `ev`: the ladder has been
    // advanced past ev.t0 (t_last0 = where it stood before) and the caller takes the
    // points t_last <= ev.t1 (sampling.hpp:96-99, 115-118), e.g. with seek_to().
    // The branch kernel's per-point probe (DenseProbe / SparseProbe / CascadeProbe) asks
    // the grid about ev.ijk, i.e. the event's own cell or node, so it answers ev.occ and is
    // counted, not evaluated (kernel_lookups += points of the event) -- except on HDDA
    // root-tile events, where it is evaluated once (see step_event).
    __device__ __forceinline__ int step_event(const SamplerDev& s, Event& ev, double& t_last0) {
        if (!(alive && t_last <= t_end)) {
            alive = false;
            return 0;
        }
        const int got = an.next(s, ev);
        if (got == 0) {
            alive = false;
            return 0;
        }
        if (got < 0) return 1; // analyzer-internal iteration, no event yet
        if (!Branch && !ev.occ) return 1;
        // The branch kernel's probe (SparseProbe, sampling.hpp:59-67) queries the grid at
        // ev.ijk.  That is the event's own node -- answer ev.occ -- except for an HDDA root-tile
        // event (a cell just outside the grid, e.g. the sliver before t_exit when the
        // re-derived cell has left the box): its ijk is the region origin, which can be an
        // in-bounds voxel, and the reference samples there if that voxel is occupied.
        if (Branch && ev.level == LV_ROOT_TILE && !ev.occ) ev.occ = an.probe(s, ev);
        t_last0 = t_last;
        ladder_seek<Sched>(t_last, ev.t0, s.dt0, s.inv_dt0, s.growth, s.t_switch, stalled);
        if (!ev.occ) { // branch kernel, empty event: its points are probed, not sampled
            kernel_lookups += (int)ladder_seek<Sched>(t_last, ev.t1, s.dt0, s.inv_dt0, s.growth,
                                                      s.t_switch, stalled);
            if (stalled) alive = false;
            return stalled ? 0 : 1;
        }
        if (stalled) {
            alive = false;
            return 0;
        }
        return 2;
    }

    // take the remaining points <= T in closed form; returns how many
    __device__ __forceinline__ int seek_to(const SamplerDev& s, double T) {
        const int n = (int)ladder_seek<Sched>(t_last, T, s.dt0, s.inv_dt0, s.growth, s.t_switch, stalled);
        if (stalled) alive = false;
        return n;
    }

    // One analyzer call (one event):
    // 0 = ray finished, 1 = event without samples, 2 = `run` holds the event's samples.
    __device__ __forceinline__ int step(const SamplerDev& s, Run& run) {
        Event ev;
        double t_last0;
        const int st = step_event(s, ev, t_last0);
        if (st != 2) return st;
        const double first = t_last;
        const int n = seek_to(s, ev.t1);
        if (stalled) return 0;
        if (Branch) kernel_lookups += n;
        if (n == 0) return 1;
        run.first = first;
        run.n = n;
        run.cell = pack_cell(ev.ijk);
        run.level = (uint8_t)(ev.level | (ev.grid_level << 2));
        run.ijk[0] = ev.ijk[0];
        run.ijk[1] = ev.ijk[1];
        run.ijk[2] = ev.ijk[2];
        run.tag = an.resume_tag();
        run.t0 = ev.t0;
        run.t_last0 = t_last0;
        return 2;
    }

    // next run with n >= 1 samples; false at the end of the ray
    __device__ __forceinline__ bool next(const SamplerDev& s, Run& run) {
        int st;
        while ((st = step(s, run)) == 1) {
        }
        return st == 2;
    }

    __device__ __forceinline__ void resume(const SamplerDev& s, const Resume& r) {
        if (!alive) return;
        an.restore(s, r.tag, r.ijk, r.t_cur);
        t_last = r.t_last;
    }

    __device__ __forceinline__ bool undefined() const { return an.undefined() || stalled; }
};

} // namespace sogk
