// sogk_layout.h — HBM layout of grids and the by-value kernel parameter blocks.
//
// Dense grid (DenseGrid, grid.hpp:117-124): the reference bit payload as is,
// x-fastest, LSB-first, ceil(N/8) bytes.
//
// VDB (SparseGrid, sparse.hpp:141-218), one node slot per 128^3 region so the
// build needs no host round trip:
//   root[region]            int32: kRootEmpty / kRootOccupied (collapsed region,
//                           RootKind::empty_tile / occupied_tile) or the node index
//   child_mask[node][64]    u64: bit ci set <=> child ci is a resolved leaf (ChildKind::leaf)
//   value_mask[node][64]    u64: bit ci set <=> tile child ci is occupied (ChildKind::occupied_tile)
//   prefix[node][64]        u32: global index of the first leaf child of word w
//                           (leaf index = prefix[w] + popc(child_mask[w] & below(ci)))
//   leaves[leaf][8]         u64: word z holds leaf bytes (z*8 + y), bit x — byte-identical
//                           to LeafNode::bytes_ (sparse.hpp:21-25)
//   table[node][4096]       i32: child ci's leaf index, or kTileEmpty / kTileOccupied — the
//                           masks + prefix flattened into one lookup for traversal (the
//                           reference's InternalNode kinds_/slots_, sparse.hpp:101-106)
// Leaves are stored in (region, ci) order, which is also SOG1 order.
#pragma once
#include <cstdint>

#include "sogk.h"

namespace sogk {

constexpr int32_t kRootEmpty = -1;
constexpr int32_t kRootOccupied = -2;
constexpr int32_t kTileEmpty = -1;
constexpr int32_t kTileOccupied = -2;
#ifndef SOGK_NODE0
#define SOGK_NODE0 1 // 1: a single-region VDB's root entry is a sampler constant (GridDev::node0)
#endif
constexpr int32_t kNodeMulti = -2147483647 - 1; // GridDev::node0: read the root per query
constexpr int SOGK_CONSTANT_SCHED = 0;
constexpr int SOGK_LINEAR_SCHED = 1;

struct GridDev {
    int res[3];
    double wmin[3];
    double voxel;
    double inv_voxel;      // 1/voxel
    int voxel_pow2;        // voxel is a power of two: x / voxel == x * inv_voxel exactly
    double clo[3], chi[3]; // voxel-centre bounds (center_bounds, sampling.hpp:248-251)
    const uint8_t* bits;   // dense payload
    int R[3];              // regions per axis
    const int32_t* root;
    const uint64_t* child_mask;
    const uint64_t* value_mask;
    const uint32_t* prefix;
    const uint64_t* leaves;
    const int32_t* table;
    int32_t node0;         // single-region VDB: its root entry, read once by the sampler (kNodeMulti:
                           // several regions or not known, the query reads the root)
    const int32_t* dist;   // DistanceGrid (distance.hpp:15-43): chessboard distance per voxel
    int smem_tab;          // launch-local: the child table of this single-region VDB is staged
                           // in the kernel's dynamic shared memory (sogk_dyn_smem)
};

struct SamplerDev {
    GridDev lv[SOGK_MAX_LEVELS];
    int n_levels;
    int spin_cap;
    double dt0, growth;
    double inv_dt0;  // 1/dt0, jump-length estimates only
    double t_switch; // linear schedule: largest t with fl(growth * t) <= dt0 (DBL_MAX if growth == 0)
};

// Per-ray resume state of pass 2: restarting the analyzer at the event that
// produced a run, with the ladder where it stood before it.
struct Resume {
    int ijk[3];
    int tag;    // cascade segment
    double t_cur;
    double t_last;
};

struct CameraDev {
    double position[3], forward[3], right[3], cam_up[3];
    double tan_half, aspect, t_far;
    int width, height;
};

} // namespace sogk
