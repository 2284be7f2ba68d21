// sogk_internal.h — host-side declarations shared by the C-ABI and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "sogk_layout.h"

namespace sogk {

struct Variant {
    int analyzer; // 0 DDA, 1 HDDA
    int cascade;  // 1: CascadeTraversal
    int branch;   // 1: sample_branch, 0: sample_skip
    int linear;   // 1: linear schedule
};

// A sample run: the ladder points one occupied event contributes, S[start .. start + n)
// of its ray (n = the next run's start, or the ray's slab fill for its last run).
struct __align__(16) RunRec {
    double first;  // first ladder point of the run
    uint32_t cell; // x | y << 10 | z << 20 (pack_cell)
    uint32_t sl;   // start (24 bits) | (Level | grid_level << 2) << 24
};
constexpr uint32_t kRunStartMax = (1u << 24) - 1;

// Pass 1 -> pass 2 state (sampler workspace): every ray's first runs in a fixed per-ray slab
// of C run records, the number of records per ray, the resume state of rays whose runs did
// not all fit (Resume::tag bits 8.. = samples covered by the slab), and the list of those rays.
struct SlabDev {
    RunRec* runs;       // [n][C]
    int32_t* nruns;     // [n]
    int64_t C;          // run records per ray; 0 = no slab (every ray resumes in tail_kernel)
    Resume* resume;     // [n]
    uint32_t* ovf_list; // [n]
    unsigned* ovf_ctr;  // [1], zeroed before pass 1
};

cudaError_t launch_count(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, int64_t* packed,
                         int64_t* stats, uint8_t* status, int32_t* counters, const SlabDev& slab,
                         cudaStream_t st, const uint32_t* perm = nullptr); // perm: processing order
// ray binning (opt-in): a processing order grouping rays by grid entry cell and direction
size_t bin_scratch_bytes(int64_t n);
cudaError_t launch_ray_binning(const SamplerDev& s, const double* rays, int64_t n, void* scratch,
                               uint32_t** perm, cudaStream_t st);
cudaError_t launch_scan(int64_t n, int64_t* packed, int64_t* stats, uint64_t* tiles,
                        unsigned int* ctr, cudaStream_t st);
int64_t scan_tiles(int64_t n);
size_t resume_bytes(int64_t n);
// slab == nullptr: cold path (no matching pass 1), traverse every ray from its start
cudaError_t launch_write(const Variant& v, const SamplerDev& s, const double* rays,
                         const CameraDev* cam, int64_t first, int64_t n, const int64_t* packed,
                         const SlabDev* slab, int64_t base, double* ts, double* te, int32_t* ri,
                         uint32_t* ce, uint8_t* lv, cudaStream_t st);
// compositing consumer (sogk_render.cu)
struct SceneDev { // sog::AnalyticScene in HBM
    const sogk_primitive* prims;
    int n;
    double bg[3];
    // candidate grid over the primitives' bounding boxes: the primitives that may contain a
    // point of cell c are cand[cstart[c] .. cstart[c+1]) in increasing index order (every
    // box grown by one cell), so density/emission sums visit the same primitives in the
    // same order as the reference's full loop
    int gres;           // cells per axis (0: no grid, loop over all primitives)
    double glo[3];      // grid origin
    double ginv;        // 1 / cell size
    const int* cstart;  // [gres^3 + 1]
    const int* cand;
};
cudaError_t launch_composite(const Variant& v, const SamplerDev& s, const SceneDev& sc,
                             const double* rays, int64_t n, const int64_t* packed, const double* ts,
                             double* result, uint8_t* rgb8, cudaStream_t st);
// frame compositing after pass 1 + scan + gather: per-sample shading (32 B each into
// `shaded`), then the per-ray front-to-back sums
// (grid-stride over *d_total samples, read on the device; total_hint sizes the grid: the
// exact total when known on the host, else the sample capacity)
cudaError_t launch_shade_accumulate(const Variant& v, const SamplerDev& s, const SceneDev& sc,
                                    const double* rays, int64_t n, const int64_t* packed,
                                    const double* ts, const int32_t* ri, const int64_t* d_total,
                                    int64_t total_hint, int64_t ray_index_base, void* shaded,
                                    double* result, uint8_t* rgb8, cudaStream_t st);


// traverse (sogk_traverse.cu): event counts per ray -> info[r] = {0, count}, stats, status,
// counters [n][2]; then events at the scanned offsets
cudaError_t launch_traverse_count(const Variant& v, const SamplerDev& s, const double* rays, int64_t n,
                                  int64_t* info, int64_t* stats, uint8_t* status, int32_t* counters,
                                  cudaStream_t st);
cudaError_t launch_traverse_write(const Variant& v, const SamplerDev& s, const double* rays, int64_t n,
                                  const int64_t* info, sogk_event* events, cudaStream_t st);
cudaError_t launch_query(const GridDev& g, int vdb, const int32_t* ijk, int64_t n, sogk_query* out,
                         cudaStream_t st);

// packed_info[r].offset += base for r < n
cudaError_t launch_add_offset(int64_t* packed, int64_t n, int64_t base, cudaStream_t st);

cudaError_t launch_raygen(const CameraDev& cam, int64_t first, int64_t n, double* rays,
                          cudaStream_t st);

// VDB build (sogk_vdb.cu)
struct VdbBuildArgs {
    GridDev dense;       // source payload + transform
    int R[3];
    int32_t* root;       // [nreg]
    uint64_t* child_mask; // [nreg*64]
    uint64_t* value_mask; // [nreg*64]
    uint32_t* prefix;    // [nreg*64]
    uint64_t* leaves;    // [nreg*4096*8] worst case
    uint32_t* region_leaves; // [nreg] scratch
    uint32_t* total_leaves;  // [1]
    int32_t* table;          // [nreg*4096] child table (sogk_layout.h)
};
cudaError_t launch_vdb_build(const VdbBuildArgs& a, cudaStream_t st);
// the child table of a VDB whose root/masks/prefix are set (built or loaded)
cudaError_t launch_vdb_table(const VdbBuildArgs& a, cudaStream_t st);
// build_distance (sogk_distance.cu): exact chessboard distances of a dense grid into dist
// (int32 per voxel); scratch has the same size; *any_occupied = 0 means all_empty()
cudaError_t launch_distance_build(const GridDev& dense, int32_t* dist, int32_t* scratch,
                                  unsigned* any_occupied, cudaStream_t st);
// to_dense (sparse.hpp:374-383): expands a VDB into a dense payload
cudaError_t launch_vdb_to_dense(const GridDev& vdb, uint8_t* bits, int64_t nbytes,
                                cudaStream_t st);

} // namespace sogk
