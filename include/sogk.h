/*
 * sogk.h — C-ABI of the B200-native ray sampler (arXiv 2404.10272 hot path).
 *
 * The reference (`/root/reference/proj/include/sog/`, namespace `sog`) is a
 * header-only C++20 CPU library with no FFI; its drop-in boundary is its own
 * C++ entry points for grid build, traverse and sample.  This header is the
 * flat C surface those entry points map onto (plain pointers and sizes, no
 * C++ or torch types); `sogk_sog.hpp` is the C++ shim that keeps the
 * reference signatures on top of it.  Each entry point cites the reference
 * interface it replaces.
 *
 * Conventions
 *  - Limits: n < 2^32 rays per call; ray_indices are int32, so ray_index_base + n - 1 <=
 *    INT32_MAX when they are written; cells pack 10 bits per axis, so cells are refused
 *    for grids above 1024 voxels on an axis (SOGK_INVALID_ARG); device rays and
 *    packed_info / event_info must be 16-byte aligned (any cudaMalloc / torch allocation is),
 *    events 8-byte (SOGK_INVALID_ARG otherwise); sample output arrays may have any alignment.
 *  - Every function returns an int status (sogk_status); no exceptions cross
 *    the boundary.  sogk_last_error() returns the thread-local message of the
 *    last failure.
 *  - Device buffers ("d_" prefix) are caller-owned CUDA device pointers;
 *    host buffers ("h_" prefix) are caller-owned host pointers (pinned memory
 *    recommended).  `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Grids are immutable after creation and may be shared by samplers, host
 *    threads and streams (mirrors the reference, README "Concurrency").  Builds are
 *    stream-ordered; every sampling launch first waits (cudaStreamWaitEvent) for the
 *    builds of its levels, so a grid built on one stream can be sampled on any other.
 *  - sogk_sample_host and the render calls lock the sampler: one sampler may be called from
 *    several host threads (the reference's render_frame does this through make_sampler).
 *    A sampler owns scratch memory: use one sampler per concurrent stream.
 *  - Rays are the reference `sog::Ray` layout (ray.hpp:92-114): 8 doubles per
 *    ray {origin.xyz, direction.xyz, t_min, t_max}, i.e. a std::vector<sog::Ray>
 *    can be passed as is.
 *
 * Output contract (the reference returns a per-ray
 * std::vector<double>, sampling.hpp:42,157-164):
 *    packed_info[r] = {offset_r, count_r}   (int64 pairs, exclusive scan of counts in ray order)
 *    t_starts[offset_r + k] = S_r[k]        (the reference sample buffer, bit-exact)
 *    t_ends  [offset_r + k] = S_r[k] + step(S_r[k])   (the next t_last, sampling.hpp:99,118)
 *    ray_indices[offset_r + k] = ray_index_base + r
 *    cells[...]  = ijk of the emitting event packed x | y<<10 | z<<20
 *                  (voxel for DDA, node origin for HDDA)
 *    levels[...] = event Level (grid.hpp:75) | cascade grid_level << 2
 */
#ifndef SOGK_H
#define SOGK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOGK_ABI_VERSION 1
#define SOGK_MAX_LEVELS 8
#define SOGK_DEFAULT_SPIN_CAP 64

typedef enum {
    SOGK_OK = 0,
    SOGK_INVALID_ARG = 1,           /* std::invalid_argument / std::out_of_range in the reference */
    SOGK_CUDA_ERROR = 2,
    SOGK_OOM = 3,
    SOGK_INSUFFICIENT_CAPACITY = 4, /* host/device output buffers too small (stats hold the total) */
    SOGK_IO_ERROR = 5,              /* sog::io_error (io.hpp:17-36); message carries the io_errc */
    SOGK_NO_DEVICE = 6
} sogk_status;

/* per-ray status (uint8) */
enum {
    SOGK_RAY_OK = 0,
    SOGK_RAY_INVALID = 1,   /* would throw in sog::Ray's constructor (ray.hpp:98-106) */
    SOGK_RAY_UNDEFINED = 2  /* reference HddaTraversal::next never returns (traversal.hpp:238-241) */
};

typedef enum { SOGK_DDA = 0, SOGK_HDDA = 1, SOGK_CD = 2 } sogk_analyzer; /* bench.hpp:27 AnalyzerKind */
typedef enum { SOGK_BRANCH = 0, SOGK_SKIP = 1 } sogk_kernel;       /* sampling.hpp:155 KernelKind */
typedef enum { SOGK_CONSTANT = 0, SOGK_LINEAR = 1 } sogk_schedule; /* sampling.hpp:18-39 */
typedef enum { SOGK_GRID_DENSE = 0, SOGK_GRID_VDB = 1, SOGK_GRID_DISTANCE = 2 } sogk_grid_kind;
typedef enum { SOGK_BLOBS = 0, SOGK_SHELL = 1, SOGK_SPONGE = 2, SOGK_RANDOM = 3 } sogk_scene_kind;

/* stats block written by sogk_sample_count (int64[SOGK_STATS_LEN], device) */
enum {
    SOGK_STAT_TOTAL_SAMPLES = 0,
    SOGK_STAT_INVALID_RAYS = 1,
    SOGK_STAT_UNDEFINED_RAYS = 2,
    SOGK_STAT_ANALYZER_LOOKUPS = 3, /* sum of SampleRun::analyzer_lookups */
    SOGK_STAT_ANALYZER_STEPS = 4,   /* sum of SampleRun::analyzer_steps */
    SOGK_STAT_KERNEL_LOOKUPS = 5,   /* sum of SampleRun::kernel_lookups */
    SOGK_STAT_SLAB_OVERFLOW_RAYS = 6, /* rays whose samples overflowed the pass-1 slab (diagnostic) */
    SOGK_STATS_LEN = 8
};

typedef struct sogk_grid sogk_grid;
typedef struct sogk_sampler sogk_sampler;

/* sog::GridTransform (grid.hpp:18-70) */
typedef struct {
    int32_t res[3];
    double world_min[3];
    double voxel_size;
} sogk_transform;

typedef struct {
    int32_t kind;           /* sogk_grid_kind */
    sogk_transform transform;
    int64_t root_entries;   /* SparseGrid::root().size() (VDB) */
    int64_t internal_nodes; /* root entries of kind internal */
    int64_t leaf_count;     /* SparseGrid::leaf_count() (sparse.hpp:173-178) */
    int64_t memory_bytes;   /* sog::memory_bytes (io.hpp:223-238) */
    int64_t device_bytes;   /* HBM footprint of this handle */
} sogk_grid_info;

typedef struct {
    int32_t analyzer;  /* sogk_analyzer; DDA needs dense levels, HDDA needs VDB levels */
    int32_t kernel;    /* sogk_kernel */
    int32_t schedule;  /* sogk_schedule */
    double dt0;        /* StepSchedule::constant(dt) / linear(dt0, growth) */
    double growth;
    int32_t cascade;   /* 1: run_cascade_sampler (sampling.hpp:440-455) even for one level;
                          n_levels > 1 always means a cascade */
    int32_t spin_cap;  /* consecutive degenerate HDDA iterations before SOGK_RAY_UNDEFINED; 0 = 64 */
} sogk_sampler_desc;

/* Pinhole camera with the host-side part of Camera::pixel_ray precomputed
 * (camera.hpp:167-173: forward/right/cam_up/tan_half/aspect; std::tan stays on the host). */
typedef struct {
    double position[3];
    double forward[3];
    double right[3];
    double cam_up[3];
    double tan_half;
    double aspect;
    double t_far;
    int32_t width, height;
} sogk_camera;

/* ---- library ----------------------------------------------------------- */
const char* sogk_version(void);
int sogk_abi_version(void);
const char* sogk_status_string(int status);
/* copies the calling thread's last error message into buf; returns its full length */
int sogk_last_error(char* buf, size_t len);
/* sets the calling thread's last error (status passthrough); for layers built on this ABI */
int sogk_last_error_set(int status, const char* msg);
/* number of visible CUDA devices (0 on a CPU-only host) */
int sogk_device_count(void);

/* ---- grids ------------------------------------------------------------- */
/* DenseGrid(transform) + payload (grid.hpp:120-124): host bit payload, ceil(N/8) bytes */
int sogk_grid_create_dense(const sogk_transform* t, const uint8_t* h_bits, size_t nbytes,
                           void* stream, sogk_grid** out);
/* same from a device payload (e.g. after an NCCL broadcast); the bytes are copied */
int sogk_grid_create_dense_device(const sogk_transform* t, const uint8_t* d_bits, size_t nbytes,
                                  void* stream, sogk_grid** out);
/* Multi-GPU setup: rank `root` broadcasts its grid -- the transform, then the
 * ceil(N/8)-byte payload -- over the caller's NCCL communicator (`nccl_comm` is an ncclComm_t;
 * NVLink / NVSwitch on one node) and every rank gets the same dense grid; rays then shard with
 * no data-path collective.  The root passes t and h_bits, other ranks may pass NULL for both.
 * Collective: every rank of the communicator calls it.  NCCL is resolved at run time
 * (libnccl.so.2; a copy the process already loaded is preferred). */
int sogk_grid_create_dense_broadcast(const sogk_transform* t, const uint8_t* h_bits, size_t nbytes,
                                     int root, void* nccl_comm, void* stream, sogk_grid** out);
/* build_sparse (sparse.hpp:333-371) on the GPU: ballot/popc masks + prefix-scan leaf slots */
int sogk_grid_build_vdb(const sogk_grid* dense, void* stream, sogk_grid** out);
/* build_distance (distance.hpp:45-103): the chessboard distance field of a dense grid
 * (int32 per voxel in HBM), the grid the CD analyzer (CdTraversal, traversal.hpp:270-337)
 * marches.  Exact, so equal to the reference's chamfer values. */
int sogk_grid_build_distance(const sogk_grid* dense, void* stream, sogk_grid** out);
/* DistanceGrid payload (int32 per voxel, x fastest) to the host; *all_empty = all_empty() */
int sogk_grid_download_distance(const sogk_grid* g, int32_t* h_dist, size_t count,
                                int32_t* all_empty);
/* deserialize_dense / deserialize_sparse (io.hpp:143-151, 183-214) straight to HBM */
int sogk_grid_load_sog0(const uint8_t* bytes, size_t len, void* stream, sogk_grid** out);
int sogk_grid_load_sog1(const uint8_t* bytes, size_t len, void* stream, sogk_grid** out);
/* serialize_dense / serialize_sparse (io.hpp:134-141, 161-181).  buf == NULL queries *len. */
int sogk_grid_export_sog0(const sogk_grid* dense, uint8_t* buf, size_t* len);
int sogk_grid_export_sog1(const sogk_grid* vdb, uint8_t* buf, size_t* len);
/* DenseGrid::payload() back to the host (to_dense for a VDB, sparse.hpp:374-383) */
int sogk_grid_download_dense(const sogk_grid* g, uint8_t* h_bits, size_t nbytes);
int sogk_grid_get_info(const sogk_grid* g, sogk_grid_info* out);
int sogk_grid_destroy(sogk_grid* g);

/* ---- samplers ---------------------------------------------------------- */
/* make_sampler (bench.hpp:382-413) for one variant: validates the schedule
 * (StepSchedule, sampling.hpp:25-34) and the cascade (validate_cascade, :253-273). */
int sogk_sampler_create(const sogk_grid* const* levels, int n_levels,
                        const sogk_sampler_desc* desc, sogk_sampler** out);
int sogk_sampler_destroy(sogk_sampler* s);
/* Processing order of pass 1 for device ray buffers: 0 (default) as given; 1 binned by the
 * cell where a ray enters the grid and its direction (counting sort on the device), for
 * incoherent batches such as probe rays.  Outputs are identical either way. */
int sogk_sampler_set_ray_order(sogk_sampler* s, int order);
/* Frees every pass-1 -> pass-2 workspace (one per device and stream, kept between calls);
 * after it, a write without a fresh count takes the exact cold path.  Synchronizes the device. */
int sogk_release_workspaces(void);

/* Pass 1 of run_sampler / run_cascade_sampler over a batch (sampling.hpp:166-196, 440-455):
 * per-ray sample counts, exclusive-scanned on the device into d_packed_info[n][2]
 * (single-pass decoupled look-back).  d_stats (int64[SOGK_STATS_LEN]) is overwritten.
 * d_status (uint8[n]) and d_counters (int32[n][3] = analyzer_lookups, analyzer_steps,
 * kernel_lookups) are optional (NULL). */
int sogk_sample_count(sogk_sampler* s, const double* d_rays, int64_t n, int64_t* d_packed_info,
                      int64_t* d_stats, uint8_t* d_status, int32_t* d_counters, void* stream);
/* Pass 2: writes the packed samples at the offsets of d_packed_info.  Buffers must hold
 * stats[SOGK_STAT_TOTAL_SAMPLES] entries; d_cells / d_levels / d_t_ends / d_ray_indices
 * may be NULL.  Pass 1 leaves each ray's sample runs in the workspace of the stream (a
 * fixed slab of run records per ray, SOGK_SLAB, default 128, reduced when 40 % of the free
 * device memory cannot hold it); a write that directly follows the count of the same rays on
 * the same sampler and stream only expands them into place, and rays whose runs did not fit
 * resume their traversal.  Any other write traverses from scratch.
 * Calls on one sampler must therefore be ordered (one stream, or synchronised). */
int sogk_sample_write(sogk_sampler* s, const double* d_rays, int64_t n,
                      const int64_t* d_packed_info, int64_t ray_index_base, double* d_t_starts,
                      double* d_t_ends, int32_t* d_ray_indices, uint32_t* d_cells,
                      uint8_t* d_levels, void* stream);
/* The same two passes with an explicit pass-1 -> pass-2 handshake: sogk_sample_count_ex
 * returns a token naming its run slabs, and sogk_sample_write_ex uses them only when it
 * presents that token on the same stream (and sampler) with no other count in between;
 * any other token (0 included) takes the exact cold path.  Use these when ray buffers are
 * rewritten in place or counts run on several streams: the token-less calls match a write
 * to its count by (sampler, stream, ray and packed_info pointers, n). */
int sogk_sample_count_ex(sogk_sampler* s, const double* d_rays, int64_t n, int64_t* d_packed_info,
                         int64_t* d_stats, uint8_t* d_status, int32_t* d_counters, void* stream,
                         uint64_t* token);
int sogk_sample_write_ex(sogk_sampler* s, const double* d_rays, int64_t n,
                         const int64_t* d_packed_info, uint64_t token, int64_t ray_index_base,
                         double* d_t_starts, double* d_t_ends, int32_t* d_ray_indices,
                         uint32_t* d_cells, uint8_t* d_levels, void* stream);
/* Camera-fused variants: the rays of pixels [first_pixel, first_pixel + n) are generated
 * in registers (Camera::pixel_ray, camera.hpp:167-179) instead of read from HBM. */
int sogk_sample_count_camera(sogk_sampler* s, const sogk_camera* cam, int64_t first_pixel,
                             int64_t n, int64_t* d_packed_info, int64_t* d_stats,
                             uint8_t* d_status, int32_t* d_counters, void* stream);
int sogk_sample_write_camera(sogk_sampler* s, const sogk_camera* cam, int64_t first_pixel,
                             int64_t n, const int64_t* d_packed_info, int64_t ray_index_base,
                             double* d_t_starts, double* d_t_ends, int32_t* d_ray_indices,
                             uint32_t* d_cells, uint8_t* d_levels, void* stream);

/* End-to-end from HOST buffers: H2D rays, count, scan, write, D2H of every output
 * (the batched form of calling run_sampler per ray).  When the total exceeds
 * `capacity` the call returns SOGK_INSUFFICIENT_CAPACITY with h_stats filled and
 * h_packed_info valid; outputs may be NULL to skip them. */
int sogk_sample_host(sogk_sampler* s, const double* h_rays, int64_t n, int64_t ray_index_base,
                     int64_t capacity, int64_t* h_packed_info, double* h_t_starts,
                     double* h_t_ends, int32_t* h_ray_indices, uint32_t* h_cells,
                     uint8_t* h_levels, uint8_t* h_status, int32_t* h_counters,
                     int64_t* h_stats, void* stream);

/* ---- traverse ----------------------------------------------------------
 * The analyzers' event streams (the reference's traverse entry points): for every ray, the
 * events DdaTraversal / HddaTraversal / CdTraversal / CascadeTraversal::next() return until
 * the stream ends, i.e. collect_events (traversal.hpp:120-264, 270-359; sampling.hpp:305-415),
 * plus lookup_count() / step_count() after the last event.  The sampler handle supplies the
 * grids, the analyzer, the cascade flag and the spin cap; its kernel and schedule are unused.
 * Rays the reference never returns on (HddaTraversal / CdTraversal edge-crossing spin) get
 * status SOGK_RAY_UNDEFINED and no events; invalid rays SOGK_RAY_INVALID. */
/* sog::TraversalEvent (grid.hpp:98-104) / sog::CascadeEvent (sampling.hpp:297-299) */
typedef struct {
    int32_t ijk[3];     /* lowest voxel of the node (voxel for DDA, node origin for HDDA / CD) */
    int32_t level;      /* sog::Level (grid.hpp:75) */
    double t0, t1;      /* [t0, t1); consecutive events share the boundary exactly */
    int32_t occupied;
    int32_t grid_level; /* cascade level, -1 outside every level; 0 for a single grid */
} sogk_event;
/* pass 1: per-ray event counts scanned into d_event_info[n][2] = {offset, count}; d_stats:
 * SOGK_STAT_TOTAL_SAMPLES holds the event total, _ANALYZER_LOOKUPS / _STEPS and
 * _INVALID_RAYS / _UNDEFINED_RAYS as for sampling.  d_status (uint8[n]) and d_counters
 * (int32[n][2] = lookup_count, step_count) are optional. */
int sogk_traverse_count(sogk_sampler* s, const double* d_rays, int64_t n, int64_t* d_event_info,
                        int64_t* d_stats, uint8_t* d_status, int32_t* d_counters, void* stream);
/* pass 2: the events of every ray at its d_event_info offset (d_events holds the total) */
int sogk_traverse_write(sogk_sampler* s, const double* d_rays, int64_t n,
                        const int64_t* d_event_info, sogk_event* d_events, void* stream);
/* both passes from host buffers (synchronous); SOGK_INSUFFICIENT_CAPACITY when the event
 * total exceeds `capacity` (h_stats and h_event_info are filled) */
int sogk_traverse_host(sogk_sampler* s, const double* h_rays, int64_t n, int64_t capacity,
                       int64_t* h_event_info, sogk_event* h_events, uint8_t* h_status,
                       int32_t* h_counters, int64_t* h_stats, void* stream);

/* sog::QueryResult (sparse.hpp:130-135) */
typedef struct {
    int32_t occupied;
    int32_t level;      /* sog::Level */
    int32_t origin[3];  /* lowest voxel of the uniform node that answered */
    int32_t extent;     /* 1, 8 or 128 */
} sogk_query;
/* SparseGrid::query (sparse.hpp:163-171) for a VDB grid (out of bounds: the empty root tile
 * of the 128-aligned region); DenseGrid::voxel_at (grid.hpp:129-133) as a leaf_voxel answer
 * for a dense grid.  d_ijk: int32[n][3]. */
int sogk_grid_query(const sogk_grid* g, const int32_t* d_ijk, int64_t n, sogk_query* d_out,
                    void* stream);
int sogk_grid_query_host(const sogk_grid* g, const int32_t* h_ijk, int64_t n, sogk_query* h_out);

/* ---- rays -------------------------------------------------------------- */
/* host: Camera::pixel_ray's per-camera terms (camera.hpp:158-173) */
int sogk_camera_setup(const double position[3], const double target[3], const double up[3],
                      double vfov_deg, int32_t width, int32_t height, double t_far,
                      sogk_camera* out);
/* device: rays of pixels [first_pixel, first_pixel + n), row-major (px fastest) */
int sogk_camera_rays(const sogk_camera* cam, int64_t first_pixel, int64_t n, double* d_rays,
                     void* stream);
/* host twin of sogk_camera_rays (bit-identical) */
int sogk_camera_rays_host(const sogk_camera* cam, int64_t first_pixel, int64_t n,
                          double* h_rays);

/* ---- compositing consumer (render.hpp) -----------------------------------
 * The emission-absorption renderer the reference composites sample buffers with. */
enum { SOGK_SPHERE = 0, SOGK_BOX = 1 };
/* sog::Primitive (render.hpp:19-56) */
typedef struct {
    int32_t shape;          /* SOGK_SPHERE / SOGK_BOX */
    double center[3];       /* sphere */
    double radius;          /* sphere */
    double lo[3], hi[3];    /* box, half-open */
    double density;         /* sigma >= 0 */
    double color[3];        /* in [0, 1] */
} sogk_primitive;
typedef struct sogk_scene sogk_scene; /* sog::AnalyticScene (render.hpp:58-92) in HBM */

/* AnalyticScene::validate (render.hpp:62-70) + upload; n may be 0 (background only) */
int sogk_scene_create(const sogk_primitive* h_prims, int32_t n, const double background[3],
                      sogk_scene** out);
int sogk_scene_destroy(sogk_scene* scene);

/* composite_detailed (render.hpp:97-118) of every ray of a packed batch (the output of
 * sogk_sample_count/write on the same rays): d_result[n][5] = color r, g, b, weight_sum,
 * transmittance; d_rgb8[n][3] (optional) = Image::set_pixel bytes (render.hpp:133-139).
 * dt of sample i is t[i+1] - t[i], of the last the schedule's step (render.hpp:106). */
int sogk_composite(const sogk_sampler* s, const sogk_scene* scene, const double* d_rays, int64_t n,
                   const int64_t* d_packed_info, const double* d_t_starts, double* d_result,
                   uint8_t* d_rgb8, void* stream);
/* render_frame's per-pixel work (bench.hpp:424-461) fused into one kernel: each pixel's ray
 * is generated, sampled and composited in registers, no sample array is written.
 * d_stats: SOGK_STAT_TOTAL_SAMPLES, _ANALYZER_LOOKUPS, _ANALYZER_STEPS, _KERNEL_LOOKUPS,
 * _UNDEFINED_RAYS of the pixels (FrameResult lookups / steps / samples). */
int sogk_render_camera(sogk_sampler* s, const sogk_scene* scene, const sogk_camera* cam,
                       int64_t first_pixel, int64_t n, double* d_result, uint8_t* d_rgb8,
                       int64_t* d_stats, void* stream);
/* The whole frame into HOST buffers: h_rgb8[height][width][3] (Image bytes, rows top to
 * bottom) and h_stats[SOGK_STATS_LEN]; synchronous. */
int sogk_render_frame_host(sogk_sampler* s, const sogk_scene* scene, const sogk_camera* cam,
                           uint8_t* h_rgb8, int64_t* h_stats, void* stream);

/* ---- host input generators (deterministic; no GPU needed) ---------------
 * Restatements of the reference generators so that identical inputs can be
 * produced where the reference is absent (tests pin them to the reference). */
/* generate_scene (scene_gen.hpp:94-192); *occupancy = occupancy_fraction() */
int sogk_scene_generate(int kind, const sogk_transform* t, uint64_t seed, double fraction,
                        int32_t count, double threshold, uint8_t* h_bits, double* occupancy);
/* build_dense_cascade (scene_gen.hpp:196-209) of generate_scene(kind, base, ...):
 * levels consecutive payloads; out_transforms[levels] */
int sogk_scene_cascade(int kind, const sogk_transform* base, uint64_t seed, double fraction,
                       int32_t count, double threshold, int32_t levels, uint8_t* h_bits,
                       sogk_transform* out_transforms);
/* generate_scene's AnalyticScene (scene_gen.hpp:94-176, background :112): the primitives the
 * occupancy is rasterized from.  h_prims == NULL: size query (*n_prims only). */
int sogk_scene_analytic(int kind, const sogk_transform* t, uint64_t seed, int32_t count,
                        sogk_primitive* h_prims, int32_t cap, int32_t* n_prims,
                        double background[3]);
/* make_probe_rays (bench.hpp:628-649) */
int sogk_probe_rays(const sogk_transform* t, int64_t count, uint64_t seed, double* h_rays);
/* testsupport::random_ray x count from one mt19937_64(seed) (tests/support/test_support.hpp:66-82) */
int sogk_random_rays(const sogk_transform* t, int64_t count, uint64_t seed, double* h_rays);
/* testsupport::random_grid / random_blocky_grid (test_support.hpp:29-62) */
int sogk_random_grid(const sogk_transform* t, uint64_t seed, double fraction, uint8_t* h_bits);
int sogk_random_blocky_grid(const sogk_transform* t, uint64_t seed, double block_fraction,
                            double noise_fraction, uint8_t* h_bits);

#ifdef __cplusplus
}
#endif
#endif /* SOGK_H */
