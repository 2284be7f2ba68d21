/*
 * sog_oracle.h — CPU restatement of the reference ray-sampler path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker.
 *
 * This is a plain-C restatement of the reference's header-only C++ library
 * (`/root/reference/proj/include/sog/*.hpp`); every function cites the
 * reference file:line it follows.  It is compiled FMA-free
 * (-ffp-contract=off, no -march) exactly like the reference CMake build, so
 * its FP64 results are bit-identical to the reference's.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against
 *  (1) the known-answer tests of the reference's own unit suite
 *      (proj/tests/unit/test_sampling.cpp, test_traversal.cpp,
 *       test_vdb_tree.cpp) re-expressed in Python, and
 *  (2) golden vectors produced by the unmodified reference headers
 *      (oracle/ref_shim.cpp -> oracle/_ref/libsogref.so, fixtures committed
 *      under tests/golden/ by tests/golden/make_golden.py).
 */
#ifndef SOG_ORACLE_H
#define SOG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct og_grid og_grid;

/* analyzer / kernel / schedule / status codes (same values as include/sogk.h) */
enum { OG_DDA = 0, OG_HDDA = 1, OG_CD = 2 };
enum { OG_BRANCH = 0, OG_SKIP = 1 };
enum { OG_CONSTANT = 0, OG_LINEAR = 1 };
enum { OG_RAY_OK = 0, OG_RAY_INVALID = 1, OG_RAY_UNDEFINED = 2 };

typedef struct {
    int32_t ijk[3];
    int32_t level;      /* sog::Level: 0 leaf_voxel, 1 leaf_tile, 2 internal_tile, 3 root_tile */
    double t0, t1;
    int32_t occupied;
    int32_t grid_level; /* cascade level, -1 outside every level; 0 for single grids */
} og_event;

typedef struct {
    const og_grid* levels[8];
    int32_t n_levels;
    int32_t cascade;    /* 1: CascadeTraversal (sampling.hpp:305-415) even for one level */
    int32_t analyzer;   /* OG_DDA (dense levels) / OG_HDDA (sparse levels) / OG_CD (distance levels) */
    int32_t kernel;     /* OG_BRANCH / OG_SKIP */
    int32_t sched_kind; /* OG_CONSTANT / OG_LINEAR */
    double dt0, growth;
    int32_t spin_cap;   /* consecutive degenerate HDDA iterations before REF_UNDEFINED */
} og_sampler;

/* grids ------------------------------------------------------------------ */
og_grid* og_dense_create(const int32_t res[3], const double wmin[3], double voxel,
                         const uint8_t* bits);
og_grid* og_sparse_build(const og_grid* dense);            /* sparse.hpp:333-371 */
og_grid* og_distance_build(const og_grid* dense);          /* distance.hpp:45-103 */
/* the distance payload (int32 per voxel, x fastest) and DistanceGrid::all_empty */
const int32_t* og_distance_data(const og_grid* dist, int32_t* all_empty);
void og_grid_free(og_grid* g);
int64_t og_sparse_serialize(const og_grid* sparse, uint8_t* buf, int64_t cap); /* io.hpp:161-181 */
int64_t og_sparse_leaf_count(const og_grid* sparse);
int32_t og_dense_voxel_at(const og_grid* dense, const int32_t ijk[3]);          /* grid.hpp:129-133 */
/* query -> occupied; writes level, origin[3], extent (sparse.hpp:163-214) */
int32_t og_sparse_query(const og_grid* sparse, const int32_t ijk[3], int32_t* level,
                        int32_t origin[3], int32_t* extent);

/* traversal ---------------------------------------------------------------- */
/* Drains the sampler's analyzer for one ray into `events` (up to cap); returns the
 * event count, or -1 when the HDDA spin guard fired.  counters = {lookups, steps}. */
int64_t og_collect_events(const og_sampler* s, const double ray[8], int64_t cap,
                          og_event* events, int64_t counters[2]);

/* sampling ----------------------------------------------------------------- */
/* One ray through run_sampler / run_cascade_sampler (sampling.hpp:166-196,440-455).
 * Returns the sample count (may exceed cap; only cap samples are written).
 * counters = {analyzer_lookups, analyzer_steps, kernel_lookups}. */
int64_t og_sample_ray(const og_sampler* s, const double ray[8], int64_t cap, double* t_starts,
                      double* t_ends, uint32_t* cells, uint8_t* levels, int64_t counters[3],
                      int32_t* status);

/* Batched packed output, same contract as sogk_sample_count + sogk_sample_write.
 * Returns the total sample count; when total > cap nothing past cap is written
 * (call again with a larger cap).  Any output pointer may be NULL. */
int64_t og_sample_batch(const og_sampler* s, const double* rays, int64_t n,
                        int64_t ray_index_base, int64_t cap, int64_t* packed_info,
                        double* t_starts, double* t_ends, int32_t* ray_indices, uint32_t* cells,
                        uint8_t* levels, int32_t* counters, uint8_t* status);

/* compositing (render.hpp) ------------------------------------------------ */
typedef struct { /* sog::Primitive (render.hpp:19-56); same layout as sogk_primitive */
    int32_t shape; /* 0 sphere, 1 box */
    double center[3];
    double radius;
    double lo[3], hi[3];
    double density;
    double color[3];
} og_primitive;

/* composite_detailed (render.hpp:97-118): out[5] = color rgb, weight_sum, transmittance.
 * sched_kind / dt0 / growth: the StepSchedule of the last sample's step. */
void og_composite(const double ray[8], const double* samples, int64_t n, const og_primitive* prims,
                  int32_t n_prims, const double background[3], int32_t sched_kind, double dt0,
                  double growth, double out[5]);
/* Image::set_pixel (render.hpp:133-139) of a linear color */
void og_set_pixel(const double rgb[3], uint8_t out[3]);
/* psnr (render.hpp:168-182) of two 8-bit buffers of n bytes (99 = identical) */
double og_psnr(const uint8_t* a, const uint8_t* b, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
