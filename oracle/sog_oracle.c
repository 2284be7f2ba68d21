/*
 * sog_oracle.c — plain-C restatement of the reference ray-sampler path.
 * TEST INFRASTRUCTURE ONLY (see sog_oracle.h).  Compile with
 *   gcc -O2 -std=c11 -ffp-contract=off   (no -march: the reference build is FMA-free)
 *
 * Reference files (all under /root/reference/proj/include/sog/):
 *   ray.hpp        Ray validation 98-106, clip_to_box 121-141
 *   grid.hpp       GridTransform 18-70, DenseGrid::voxel_at 129-133, clip_ray 202-205
 *   sparse.hpp     LeafNode 14-54, InternalNode 60-112, SparseGrid::query 163-214,
 *                  read_leaf_block 283-324, build_sparse 333-371
 *   traversal.hpp  RayGridGeometry 27-113, DdaTraversal 120-193, HddaTraversal 199-264
 *   sampling.hpp   StepSchedule 18-39, probes 50-67, sample_branch 87-103,
 *                  sample_skip 105-122, run_sampler 166-196, cascades 222-455
 *   io.hpp         serialize_sparse 161-181
 */
#include "sog_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define KINF (DBL_MAX / 4) /* traversal.hpp:19 kInfiniteStep */

enum { LV_VOXEL = 0, LV_LEAF_TILE = 1, LV_INTERNAL_TILE = 2, LV_ROOT_TILE = 3 };
enum { CK_EMPTY = 0, CK_OCC = 1, CK_LEAF = 2 }; /* sparse.hpp:56 ChildKind / :114 RootKind */

struct og_grid {
    int32_t sparse;
    int32_t res[3];
    double wmin[3];
    double voxel;
    /* dense */
    uint8_t* bits;
    int64_t nbytes;
    /* sparse: region table (every region has an entry, sparse.hpp:368) */
    int32_t R[3];
    uint8_t* root_kind;  /* per region */
    int32_t* root_node;  /* per region: node index or -1 */
    uint8_t* kinds;      /* [nodes][4096] */
    int32_t* slots;      /* [nodes][4096] */
    uint8_t* leaves;     /* [leaves][64] */
    int64_t n_nodes, n_leaves;
    /* distance (DistanceGrid, distance.hpp:15-43): int32 per voxel, x fastest */
    int32_t* dist;
    int32_t all_empty;
};

/* ------------------------------------------------------------------------ */
/* math helpers mirroring the exact std:: semantics used by the reference    */
/* ------------------------------------------------------------------------ */
static inline double std_max(double a, double b) { return (a < b) ? b : a; } /* std::max */
static inline double std_min(double a, double b) { return (b < a) ? b : a; } /* std::min */

static inline int floor_div(int a, int b) { /* vec.hpp:68-76 */
    int q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

static inline double world_max(const og_grid* g, int a) { /* grid.hpp:36-38 */
    return g->wmin[a] + (double)g->res[a] * g->voxel;
}

static inline int contains(const og_grid* g, const int ijk[3]) { /* grid.hpp:52-55 */
    return ijk[0] >= 0 && ijk[1] >= 0 && ijk[2] >= 0 && ijk[0] < g->res[0] &&
           ijk[1] < g->res[1] && ijk[2] < g->res[2];
}

static inline int dense_bit(const og_grid* g, const int ijk[3]) { /* grid.hpp:129-133 */
    if (!contains(g, ijk)) return 0;
    const uint64_t idx =
        ((uint64_t)ijk[2] * (uint64_t)g->res[1] + (uint64_t)ijk[1]) * (uint64_t)g->res[0] +
        (uint64_t)ijk[0];
    return (g->bits[idx >> 3] >> (idx & 7)) & 1u;
}

/* ------------------------------------------------------------------------ */
/* grids                                                                     */
/* ------------------------------------------------------------------------ */
og_grid* og_dense_create(const int32_t res[3], const double wmin[3], double voxel,
                         const uint8_t* bits) {
    if (res[0] < 1 || res[1] < 1 || res[2] < 1 || !(voxel > 0.0)) return NULL; /* grid.hpp:26-29 */
    og_grid* g = (og_grid*)calloc(1, sizeof(og_grid));
    for (int a = 0; a < 3; ++a) {
        g->res[a] = res[a];
        g->wmin[a] = wmin[a];
    }
    g->voxel = voxel;
    const uint64_t n = (uint64_t)res[0] * res[1] * res[2];
    g->nbytes = (int64_t)((n + 7) / 8);
    g->bits = (uint8_t*)malloc((size_t)g->nbytes);
    memcpy(g->bits, bits, (size_t)g->nbytes);
    return g;
}

void og_grid_free(og_grid* g) {
    if (!g) return;
    free(g->bits);
    free(g->root_kind);
    free(g->root_node);
    free(g->kinds);
    free(g->slots);
    free(g->leaves);
    free(g->dist);
    free(g);
}

/* build_distance, distance.hpp:45-103: two-pass chamfer over the 26-neighbourhood with unit
 * weights (exact for the chessboard metric), sentinel max(resolution) when nothing is occupied */
og_grid* og_distance_build(const og_grid* d) {
    if (!d || d->sparse || d->dist) return NULL;
    og_grid* g = (og_grid*)calloc(1, sizeof(og_grid));
    for (int a = 0; a < 3; ++a) {
        g->res[a] = d->res[a];
        g->wmin[a] = d->wmin[a];
    }
    g->voxel = d->voxel;
    const int rx = d->res[0], ry = d->res[1], rz = d->res[2];
    const int64_t n = (int64_t)rx * ry * rz;
    g->dist = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    const int32_t kInf = 1 << 29;
    int any = 0;
    int64_t idx = 0;
    for (int z = 0; z < rz; ++z)
        for (int y = 0; y < ry; ++y)
            for (int x = 0; x < rx; ++x, ++idx) {
                const int ijk[3] = {x, y, z};
                const int occ = dense_bit(d, ijk);
                g->dist[idx] = occ ? 0 : kInf;
                any |= occ;
            }
    if (!any) {
        int32_t sentinel = rx > ry ? rx : ry;
        if (rz > sentinel) sentinel = rz;
        for (int64_t i = 0; i < n; ++i) g->dist[i] = sentinel;
        g->all_empty = 1;
        return g;
    }
#define DAT(X, Y, Z) (((X) < 0 || (Y) < 0 || (Z) < 0 || (X) >= rx || (Y) >= ry || (Z) >= rz) \
                          ? kInf : g->dist[((int64_t)(Z) * ry + (Y)) * rx + (X)])
#define MIN1(b, v) do { const int32_t v_ = (v) + 1; if (v_ < (b)) (b) = v_; } while (0)
    for (int z = 0; z < rz; ++z) /* forward: neighbours lexicographically before (dz, dy, dx) */
        for (int y = 0; y < ry; ++y)
            for (int x = 0; x < rx; ++x) {
                int32_t best = DAT(x, y, z);
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) MIN1(best, DAT(x + dx, y + dy, z - 1));
                MIN1(best, DAT(x - 1, y - 1, z));
                MIN1(best, DAT(x, y - 1, z));
                MIN1(best, DAT(x + 1, y - 1, z));
                MIN1(best, DAT(x - 1, y, z));
                g->dist[((int64_t)z * ry + y) * rx + x] = best;
            }
    for (int z = rz - 1; z >= 0; --z) /* backward: the mirror image */
        for (int y = ry - 1; y >= 0; --y)
            for (int x = rx - 1; x >= 0; --x) {
                int32_t best = DAT(x, y, z);
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) MIN1(best, DAT(x + dx, y + dy, z + 1));
                MIN1(best, DAT(x + 1, y + 1, z));
                MIN1(best, DAT(x, y + 1, z));
                MIN1(best, DAT(x - 1, y + 1, z));
                MIN1(best, DAT(x + 1, y, z));
                g->dist[((int64_t)z * ry + y) * rx + x] = best;
            }
#undef DAT
#undef MIN1
    return g;
}

const int32_t* og_distance_data(const og_grid* g, int32_t* all_empty) {
    if (all_empty) *all_empty = g ? g->all_empty : 0;
    return g ? g->dist : NULL;
}

/* DistanceGrid::at (distance.hpp:27-30): out of bounds reads 1 */
static inline int32_t dist_at(const og_grid* g, const int ijk[3]) {
    if (!contains(g, ijk)) return 1;
    return g->dist[((int64_t)ijk[2] * g->res[1] + ijk[1]) * g->res[0] + ijk[0]];
}

/* read_leaf_block, sparse.hpp:283-324.  Both the aligned fast path and the
 * padded general path produce the same bytes; the general path is the
 * definition (out-of-bounds voxels read empty). */
static void read_leaf_block(const og_grid* d, const int bo[3], uint8_t leaf[64], int* uniform,
                            int* value) {
    int all0 = 1, all1 = 1;
    memset(leaf, 0, 64);
    for (int lz = 0; lz < 8; ++lz)
        for (int ly = 0; ly < 8; ++ly)
            for (int lx = 0; lx < 8; ++lx) {
                const int ijk[3] = {bo[0] + lx, bo[1] + ly, bo[2] + lz};
                const int bit = dense_bit(d, ijk);
                const int bi = (lz * 8 + ly) * 8 + lx; /* LeafNode::bit_index, :20-22 */
                if (bit) leaf[bi >> 3] |= (uint8_t)(1u << (bi & 7));
                all0 &= !bit;
                all1 &= bit;
            }
    *uniform = all0 || all1;
    *value = all1;
}

og_grid* og_sparse_build(const og_grid* d) { /* build_sparse, sparse.hpp:333-371 */
    if (!d || d->sparse) return NULL;
    og_grid* g = (og_grid*)calloc(1, sizeof(og_grid));
    g->sparse = 1;
    for (int a = 0; a < 3; ++a) {
        g->res[a] = d->res[a];
        g->wmin[a] = d->wmin[a];
        g->R[a] = (d->res[a] + 127) / 128;
    }
    g->voxel = d->voxel;
    const int64_t nreg = (int64_t)g->R[0] * g->R[1] * g->R[2];
    g->root_kind = (uint8_t*)calloc((size_t)nreg, 1);
    g->root_node = (int32_t*)malloc(sizeof(int32_t) * (size_t)nreg);
    g->kinds = (uint8_t*)malloc((size_t)nreg * 4096);
    g->slots = (int32_t*)malloc(sizeof(int32_t) * (size_t)nreg * 4096);
    int64_t leaf_cap = 1024;
    g->leaves = (uint8_t*)malloc((size_t)leaf_cap * 64);
    uint8_t kinds[4096];
    int32_t slots[4096];
    for (int rz = 0; rz < g->R[2]; ++rz)
        for (int ry = 0; ry < g->R[1]; ++ry)
            for (int rx = 0; rx < g->R[0]; ++rx) {
                const int64_t r = ((int64_t)rz * g->R[1] + ry) * g->R[0] + rx;
                const int64_t leaf_start = g->n_leaves;
                int any_leaf = 0;
                for (int cz = 0; cz < 16; ++cz)
                    for (int cy = 0; cy < 16; ++cy)
                        for (int cx = 0; cx < 16; ++cx) {
                            const int ci = (cz * 16 + cy) * 16 + cx; /* :70 child_index */
                            const int bo[3] = {rx * 128 + cx * 8, ry * 128 + cy * 8,
                                               rz * 128 + cz * 8};
                            uint8_t leaf[64];
                            int uniform, value;
                            read_leaf_block(d, bo, leaf, &uniform, &value);
                            if (uniform) { /* set_tile :78-82 */
                                kinds[ci] = value ? CK_OCC : CK_EMPTY;
                                slots[ci] = -1;
                            } else { /* emplace_leaf :84-88 */
                                if (g->n_leaves == leaf_cap) {
                                    leaf_cap *= 2;
                                    g->leaves = (uint8_t*)realloc(g->leaves, (size_t)leaf_cap * 64);
                                }
                                kinds[ci] = CK_LEAF;
                                slots[ci] = (int32_t)(g->n_leaves - leaf_start);
                                memcpy(g->leaves + g->n_leaves * 64, leaf, 64);
                                g->n_leaves++;
                                any_leaf = 1;
                            }
                        }
                /* uniform_tiles :92-99 */
                int uniform_tiles = kinds[0] != CK_LEAF;
                for (int ci = 1; ci < 4096 && uniform_tiles; ++ci)
                    if (kinds[ci] != kinds[0]) uniform_tiles = 0;
                if (!any_leaf && uniform_tiles) {
                    g->root_kind[r] = kinds[0] == CK_OCC ? CK_OCC : CK_EMPTY;
                    g->root_node[r] = -1;
                } else {
                    g->root_kind[r] = CK_LEAF; /* RootKind::internal == 2 */
                    g->root_node[r] = (int32_t)g->n_nodes;
                    memcpy(g->kinds + g->n_nodes * 4096, kinds, 4096);
                    for (int ci = 0; ci < 4096; ++ci)
                        g->slots[g->n_nodes * 4096 + ci] =
                            slots[ci] < 0 ? -1 : (int32_t)(slots[ci] + leaf_start);
                    g->n_nodes++;
                }
            }
    return g;
}

int64_t og_sparse_leaf_count(const og_grid* g) { return g && g->sparse ? g->n_leaves : -1; }

int32_t og_dense_voxel_at(const og_grid* d, const int32_t ijk[3]) {
    const int v[3] = {ijk[0], ijk[1], ijk[2]};
    return dense_bit(d, v);
}

/* serialize_sparse, io.hpp:161-181 (write_transform :308-316) */
static int64_t put(uint8_t* buf, int64_t cap, int64_t pos, const void* src, int64_t n) {
    if (buf && pos + n <= cap) memcpy(buf + pos, src, (size_t)n);
    return pos + n;
}
static int64_t put_u32(uint8_t* buf, int64_t cap, int64_t pos, uint32_t v) {
    uint8_t b[4];
    for (int i = 0; i < 4; ++i) b[i] = (uint8_t)(v >> (8 * i));
    return put(buf, cap, pos, b, 4);
}
static int64_t put_f64(uint8_t* buf, int64_t cap, int64_t pos, double v) {
    uint64_t bits;
    memcpy(&bits, &v, 8);
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(bits >> (8 * i));
    return put(buf, cap, pos, b, 8);
}

int64_t og_sparse_serialize(const og_grid* g, uint8_t* buf, int64_t cap) {
    if (!g || !g->sparse) return -1;
    int64_t p = 0;
    p = put(buf, cap, p, "SOG1", 4);
    p = put_u32(buf, cap, p, 1u);
    for (int a = 0; a < 3; ++a) p = put_u32(buf, cap, p, (uint32_t)g->res[a]);
    for (int a = 0; a < 3; ++a) p = put_f64(buf, cap, p, g->wmin[a]);
    p = put_f64(buf, cap, p, g->voxel);
    const int64_t nreg = (int64_t)g->R[0] * g->R[1] * g->R[2];
    p = put_u32(buf, cap, p, (uint32_t)nreg);
    /* root map order is z, then y, then x (sparse.hpp:119-125) == linear region order */
    for (int rz = 0; rz < g->R[2]; ++rz)
        for (int ry = 0; ry < g->R[1]; ++ry)
            for (int rx = 0; rx < g->R[0]; ++rx) {
                const int64_t r = ((int64_t)rz * g->R[1] + ry) * g->R[0] + rx;
                p = put_u32(buf, cap, p, (uint32_t)(rx * 128));
                p = put_u32(buf, cap, p, (uint32_t)(ry * 128));
                p = put_u32(buf, cap, p, (uint32_t)(rz * 128));
                const uint8_t k = g->root_kind[r];
                p = put(buf, cap, p, &k, 1);
                if (k != CK_LEAF) continue;
                const int64_t node = g->root_node[r];
                for (int ci = 0; ci < 4096; ++ci) {
                    const uint8_t ck = g->kinds[node * 4096 + ci];
                    p = put(buf, cap, p, &ck, 1);
                    if (ck == CK_LEAF)
                        p = put(buf, cap, p, g->leaves + (int64_t)g->slots[node * 4096 + ci] * 64,
                                64);
                }
            }
    return p;
}

/* SparseGrid::query + query_in_entry, sparse.hpp:163-171,198-214.  The
 * reference's Accessor (:224-276) returns identical answers (its cache is
 * semantically transparent), so the oracle uses the uncached lookup. */
typedef struct {
    int occupied, level, extent;
    int origin[3];
} og_q;

static og_q sparse_query(const og_grid* g, const int ijk[3]) {
    og_q q;
    int region[3];
    for (int a = 0; a < 3; ++a) region[a] = floor_div(ijk[a], 128) * 128; /* :159 */
    if (!contains(g, ijk)) {
        q.occupied = 0;
        q.level = LV_ROOT_TILE;
        q.extent = 128;
        for (int a = 0; a < 3; ++a) q.origin[a] = region[a];
        return q;
    }
    const int64_t r =
        ((int64_t)(region[2] / 128) * g->R[1] + region[1] / 128) * g->R[0] + region[0] / 128;
    if (g->root_kind[r] != CK_LEAF) {
        q.occupied = g->root_kind[r] == CK_OCC;
        q.level = LV_INTERNAL_TILE;
        q.extent = 128;
        for (int a = 0; a < 3; ++a) q.origin[a] = region[a];
        return q;
    }
    int local[3], child[3];
    for (int a = 0; a < 3; ++a) {
        local[a] = ijk[a] - region[a];
        child[a] = local[a] >> 3;
    }
    const int ci = (child[2] * 16 + child[1]) * 16 + child[0];
    const int64_t node = g->root_node[r];
    const uint8_t ck = g->kinds[node * 4096 + ci];
    if (ck != CK_LEAF) {
        q.occupied = ck == CK_OCC;
        q.level = LV_LEAF_TILE;
        q.extent = 8;
        for (int a = 0; a < 3; ++a) q.origin[a] = region[a] + child[a] * 8;
        return q;
    }
    const uint8_t* leaf = g->leaves + (int64_t)g->slots[node * 4096 + ci] * 64;
    const int bi = ((local[2] & 7) * 8 + (local[1] & 7)) * 8 + (local[0] & 7);
    q.occupied = (leaf[bi >> 3] >> (bi & 7)) & 1u;
    q.level = LV_VOXEL;
    q.extent = 1;
    for (int a = 0; a < 3; ++a) q.origin[a] = ijk[a];
    return q;
}

int32_t og_sparse_query(const og_grid* g, const int32_t ijk[3], int32_t* level,
                        int32_t origin[3], int32_t* extent) {
    const int v[3] = {ijk[0], ijk[1], ijk[2]};
    const og_q q = sparse_query(g, v);
    *level = q.level;
    *extent = q.extent;
    for (int a = 0; a < 3; ++a) origin[a] = q.origin[a];
    return q.occupied;
}

/* ------------------------------------------------------------------------ */
/* rays and geometry                                                         */
/* ------------------------------------------------------------------------ */
typedef struct {
    double o[3], d[3], tmin, tmax;
} og_ray;

/* Ray constructor validation, ray.hpp:98-106 (Vec3::length = sqrt(dot), vec.hpp:23-24) */
static int ray_valid(const og_ray* r) {
    const double len = sqrt(r->d[0] * r->d[0] + r->d[1] * r->d[1] + r->d[2] * r->d[2]);
    if (fabs(len - 1.0) > 1e-9) return 0;
    if (!(r->tmin >= 0.0)) return 0;
    if (!(r->tmin < r->tmax)) return 0;
    return 1;
}

/* clip_to_box, ray.hpp:121-141 */
static int clip_to_box(const og_ray* r, const double lo[3], const double hi[3], double* te,
                       double* tx) {
    double t_enter = r->tmin, t_exit = r->tmax;
    for (int a = 0; a < 3; ++a) {
        const double d = r->d[a], o = r->o[a];
        if (d == 0.0) {
            if (o < lo[a] || o >= hi[a]) return 0;
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
    if (!(t_enter < t_exit)) return 0;
    *te = t_enter;
    *tx = t_exit;
    return 1;
}

typedef struct {
    double entry[3], dir[3], inv[3];
    int step[3];
    double t_enter, t_exit;
    int valid;
} og_geom;

static inline double plane_t(const og_geom* g, int a, double plane) { /* traversal.hpp:66-68 */
    return g->t_enter + (plane - g->entry[a]) * g->inv[a];
}
static inline double grid_coord(const og_geom* g, int a, double t) { /* :70-72 */
    return g->entry[a] + (t - g->t_enter) * g->dir[a];
}

/* RayGridGeometry ctor, traversal.hpp:38-64 */
static void geom_init(og_geom* g, const og_ray* r, const og_grid* grid) {
    memset(g, 0, sizeof(*g));
    double lo[3], hi[3], te, tx;
    for (int a = 0; a < 3; ++a) {
        lo[a] = grid->wmin[a];
        hi[a] = world_max(grid, a);
    }
    if (!clip_to_box(r, lo, hi, &te, &tx)) return; /* clip_ray, grid.hpp:202-205 */
    g->t_enter = te;
    for (int a = 0; a < 3; ++a) {
        g->dir[a] = r->d[a] / grid->voxel;
        g->entry[a] = (r->o[a] + r->d[a] * te - grid->wmin[a]) / grid->voxel;
        if (g->dir[a] > 0.0) {
            g->step[a] = 1;
            g->inv[a] = 1.0 / g->dir[a];
        } else if (g->dir[a] < 0.0) {
            g->step[a] = -1;
            g->inv[a] = 1.0 / g->dir[a];
        } else {
            g->step[a] = 0;
            g->inv[a] = KINF;
        }
    }
    g->t_exit = r->tmax;
    for (int a = 0; a < 3; ++a) {
        if (g->step[a] == 0) continue;
        const double far_plane = g->step[a] > 0 ? (double)grid->res[a] : 0.0;
        g->t_exit = std_min(g->t_exit, plane_t(g, a, far_plane));
    }
    g->valid = g->t_enter < g->t_exit;
}

/* entry_cell, traversal.hpp:77-85 */
static void entry_cell(const og_geom* g, const int res[3], int ijk[3]) {
    for (int a = 0; a < 3; ++a) {
        double c = floor(g->entry[a]);
        if (g->step[a] < 0 && c == g->entry[a]) c -= 1.0;
        ijk[a] = (int)std_max(0.0, std_min(c, (double)(res[a] - 1)));
    }
}

/* cell_after_crossing, traversal.hpp:91-104 */
static void cell_after_crossing(const og_geom* g, double t, int axis, int stepped, int ijk[3]) {
    for (int a = 0; a < 3; ++a) {
        if (a == axis) {
            ijk[a] = stepped;
        } else if (g->step[a] != 0) {
            const double gc = grid_coord(g, a, t);
            double c = floor(gc);
            if (g->step[a] < 0 && c == gc) c -= 1.0;
            ijk[a] = (int)c;
        }
    }
}

static inline int argmin_axis(const double t[3]) { /* traversal.hpp:107-112 */
    int axis = 0;
    if (t[1] < t[0]) axis = 1;
    if (t[2] < t[axis]) axis = 2;
    return axis;
}

/* ------------------------------------------------------------------------ */
/* analyzers                                                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    const og_grid* grid;
    int hdda; /* 0 DDA, 1 HDDA, 2 CD */
    og_geom geom;
    int ijk[3];
    int next_plane[3];
    double t_next[3];
    double t_cur;
    int64_t lookups, steps;
    int done;
    int spin_cap;
    int undefined; /* HDDA spin guard fired */
} og_an;

/* DdaTraversal ctor :124-141 / HddaTraversal ctor :203-211 */
static void an_init(og_an* an, const og_grid* grid, int hdda, const og_ray* r, int spin_cap) {
    memset(an, 0, sizeof(*an));
    an->grid = grid;
    an->hdda = hdda;
    an->spin_cap = spin_cap;
    geom_init(&an->geom, r, grid);
    if (!an->geom.valid) {
        an->done = 1;
        return;
    }
    entry_cell(&an->geom, grid->res, an->ijk);
    an->t_cur = an->geom.t_enter;
    if (hdda) return; /* HDDA and CD derive their planes per step */
    for (int a = 0; a < 3; ++a) {
        if (an->geom.step[a] == 0) {
            an->next_plane[a] = 0;
            an->t_next[a] = KINF;
        } else {
            an->next_plane[a] = an->ijk[a] + (an->geom.step[a] > 0 ? 1 : 0);
            an->t_next[a] = plane_t(&an->geom, a, (double)an->next_plane[a]);
        }
    }
}

static void dda_emit(og_an* an, double t1, og_event* ev) { /* :171-175 */
    ++an->steps;
    ++an->lookups;
    for (int a = 0; a < 3; ++a) ev->ijk[a] = an->ijk[a];
    ev->level = LV_VOXEL;
    ev->t0 = an->t_cur;
    ev->t1 = t1;
    ev->occupied = dense_bit(an->grid, an->ijk);
    ev->grid_level = 0;
}

static void dda_advance(og_an* an, int axis) { /* :177-182 */
    an->ijk[axis] += an->geom.step[axis];
    an->next_plane[axis] += an->geom.step[axis];
    an->t_next[axis] = plane_t(&an->geom, axis, (double)an->next_plane[axis]);
    if (an->ijk[axis] < 0 || an->ijk[axis] >= an->grid->res[axis]) an->done = 1;
}

/* returns 1 with *ev filled, 0 at end of stream */
static int dda_next(og_an* an, og_event* ev) { /* DdaTraversal::next :143-162 */
    if (an->done) return 0;
    for (;;) {
        const int axis = argmin_axis(an->t_next);
        const double t1 = an->t_next[axis];
        if (t1 >= an->geom.t_exit) {
            an->done = 1;
            dda_emit(an, an->geom.t_exit, ev);
            return 1;
        }
        if (t1 <= an->t_cur) {
            dda_advance(an, axis);
            if (an->done) return 0;
            continue;
        }
        dda_emit(an, t1, ev);
        an->t_cur = t1;
        dda_advance(an, axis);
        return 1;
    }
}

static int hdda_next(og_an* an, og_event* ev) { /* HddaTraversal::next :213-248 */
    if (an->done) return 0;
    int degenerate = 0;
    for (;;) {
        const og_q q = sparse_query(an->grid, an->ijk);
        ++an->lookups;
        double t_cross[3];
        for (int a = 0; a < 3; ++a) {
            if (an->geom.step[a] == 0) {
                t_cross[a] = KINF;
            } else {
                const double plane = an->geom.step[a] > 0 ? (double)(q.origin[a] + q.extent)
                                                          : (double)q.origin[a];
                t_cross[a] = plane_t(&an->geom, a, plane);
            }
        }
        const int axis = argmin_axis(t_cross);
        const double t1 = t_cross[axis];
        ev->level = q.level;
        ev->occupied = q.occupied;
        ev->grid_level = 0;
        for (int a = 0; a < 3; ++a) ev->ijk[a] = q.origin[a];
        if (t1 >= an->geom.t_exit) {
            ++an->steps;
            an->done = 1;
            ev->t0 = an->t_cur;
            ev->t1 = an->geom.t_exit;
            return 1;
        }
        const int stepped =
            an->geom.step[axis] > 0 ? q.origin[axis] + q.extent : q.origin[axis] - 1;
        if (t1 <= an->t_cur) { /* degenerate corner crossing (:238-241) */
            cell_after_crossing(&an->geom, an->t_cur, axis, stepped, an->ijk);
            /* Spin guard: the reference loops forever here at exact edge
             * crossings; a ray that hits the cap has no defined
             * reference output. */
            if (++degenerate > an->spin_cap) {
                an->undefined = 1;
                an->done = 1;
                return 0;
            }
            continue;
        }
        ev->t0 = an->t_cur;
        ev->t1 = t1;
        ++an->steps;
        cell_after_crossing(&an->geom, t1, axis, stepped, an->ijk);
        an->t_cur = t1;
        return 1;
    }
}

static int cd_next(og_an* an, og_event* ev) { /* CdTraversal::next, traversal.hpp:290-327 */
    if (an->done) return 0;
    int degenerate = 0;
    for (;;) {
        const int32_t d = dist_at(an->grid, an->ijk);
        ++an->lookups;
        const int half = d > 1 ? d - 1 : 0;
        int low[3];
        for (int a = 0; a < 3; ++a) low[a] = an->ijk[a] - half;
        const int extent = 2 * half + 1;
        double t_cross[3];
        for (int a = 0; a < 3; ++a) {
            if (an->geom.step[a] == 0) {
                t_cross[a] = KINF;
            } else {
                const double plane = an->geom.step[a] > 0 ? (double)(low[a] + extent) : (double)low[a];
                t_cross[a] = plane_t(&an->geom, a, plane);
            }
        }
        const int axis = argmin_axis(t_cross);
        const double t1 = t_cross[axis];
        ev->level = LV_VOXEL;
        ev->occupied = d == 0;
        ev->grid_level = 0;
        for (int a = 0; a < 3; ++a) ev->ijk[a] = low[a];
        if (t1 >= an->geom.t_exit) {
            ++an->steps;
            an->done = 1;
            ev->t0 = an->t_cur;
            ev->t1 = an->geom.t_exit;
            return 1;
        }
        const int stepped = an->geom.step[axis] > 0 ? low[axis] + extent : low[axis] - 1;
        if (t1 <= an->t_cur) { /* degenerate corner crossing (:311-314) */
            cell_after_crossing(&an->geom, an->t_cur, axis, stepped, an->ijk);
            /* the same edge-crossing spin as HddaTraversal */
            if (++degenerate > an->spin_cap) {
                an->undefined = 1;
                an->done = 1;
                return 0;
            }
            continue;
        }
        ev->t0 = an->t_cur;
        ev->t1 = t1;
        ++an->steps;
        cell_after_crossing(&an->geom, t1, axis, stepped, an->ijk);
        an->t_cur = t1;
        return 1;
    }
}

static int an_next(og_an* an, og_event* ev) {
    return an->hdda == 2 ? cd_next(an, ev) : an->hdda ? hdda_next(an, ev) : dda_next(an, ev);
}

/* ------------------------------------------------------------------------ */
/* cascades, sampling.hpp:222-415                                            */
/* ------------------------------------------------------------------------ */
typedef struct {
    const og_sampler* s;
    og_ray ray;
    double seg_t0[16], seg_t1[16];
    int seg_level[16];
    int n_seg, seg;
    int has_sub;
    og_an sub;
    int64_t finished_lookups, finished_steps;
    int valid;
    double t_enter, t_exit;
    int undefined;
} og_cascade;

static void center_bounds(const og_grid* g, double lo[3], double hi[3]) { /* :248-251 */
    const double h = g->voxel * 0.5;
    for (int a = 0; a < 3; ++a) {
        lo[a] = g->wmin[a] + h;
        hi[a] = world_max(g, a) - h;
    }
}

static void cascade_init(og_cascade* c, const og_sampler* s, const og_ray* r) { /* :312-355 */
    memset(c, 0, sizeof(*c));
    c->s = s;
    c->ray = *r;
    const int n = s->n_levels;
    double rf[8], rs[8];
    int hit[8];
    for (int b = 0; b < n; ++b) {
        double lo[3], hi[3];
        center_bounds(s->levels[b], lo, hi);
        hit[b] = clip_to_box(r, lo, hi, &rf[b], &rs[b]);
    }
    if (!hit[n - 1]) return;
    const double t_enter = rf[n - 1], t_exit = rs[n - 1];
    double cuts[18];
    int nc = 0;
    cuts[nc++] = t_enter;
    cuts[nc++] = t_exit;
    for (int b = 0; b + 1 < n; ++b) {
        if (!hit[b]) continue;
        if (rf[b] > t_enter && rf[b] < t_exit) cuts[nc++] = rf[b];
        if (rs[b] > t_enter && rs[b] < t_exit) cuts[nc++] = rs[b];
    }
    /* std::sort + std::unique (values are finite and NaN-free) */
    for (int i = 1; i < nc; ++i) {
        const double v = cuts[i];
        int j = i - 1;
        while (j >= 0 && cuts[j] > v) {
            cuts[j + 1] = cuts[j];
            --j;
        }
        cuts[j + 1] = v;
    }
    int m = 0;
    for (int i = 0; i < nc; ++i)
        if (m == 0 || !(cuts[m - 1] == cuts[i])) cuts[m++] = cuts[i];
    for (int i = 0; i + 1 < m; ++i) {
        if (!(cuts[i] < cuts[i + 1])) continue;
        const double mid = 0.5 * (cuts[i] + cuts[i + 1]);
        int level = -1;
        for (int b = 0; b < n; ++b)
            if (hit[b] && mid >= rf[b] && mid < rs[b]) {
                level = b;
                break;
            }
        c->seg_t0[c->n_seg] = cuts[i];
        c->seg_t1[c->n_seg] = cuts[i + 1];
        c->seg_level[c->n_seg] = level;
        c->n_seg++;
    }
    c->valid = c->n_seg > 0;
    c->t_enter = t_enter;
    c->t_exit = t_exit;
}

static int cascade_next(og_cascade* c, og_event* ev) { /* :361-392 */
    for (;;) {
        if (c->has_sub) {
            if (an_next(&c->sub, ev)) {
                ev->grid_level = c->seg_level[c->seg];
                return 1;
            }
            if (c->sub.undefined) {
                c->undefined = 1;
                return 0;
            }
            c->finished_lookups += c->sub.lookups;
            c->finished_steps += c->sub.steps;
            c->has_sub = 0;
            ++c->seg;
        }
        if (c->seg >= c->n_seg) return 0;
        if (c->seg_level[c->seg] < 0) {
            ev->ijk[0] = ev->ijk[1] = ev->ijk[2] = 0;
            ev->level = LV_ROOT_TILE;
            ev->t0 = c->seg_t0[c->seg];
            ev->t1 = c->seg_t1[c->seg];
            ev->occupied = 0;
            ev->grid_level = -1;
            ++c->seg;
            ++c->finished_steps;
            return 1;
        }
        og_ray sub = c->ray;
        sub.tmin = c->seg_t0[c->seg];
        sub.tmax = c->seg_t1[c->seg];
        an_init(&c->sub, c->s->levels[c->seg_level[c->seg]], c->s->analyzer, &sub,
                c->s->spin_cap);
        c->has_sub = 1;
    }
}

/* ------------------------------------------------------------------------ */
/* generic analyzer wrapper                                                  */
/* ------------------------------------------------------------------------ */
typedef struct {
    int cascade;
    og_an an;
    og_cascade cas;
} og_any;

static void any_init(og_any* x, const og_sampler* s, const og_ray* r) {
    x->cascade = s->cascade || s->n_levels > 1;
    if (x->cascade)
        cascade_init(&x->cas, s, r);
    else
        an_init(&x->an, s->levels[0], s->analyzer, r, s->spin_cap);
}
static int any_valid(const og_any* x) { return x->cascade ? x->cas.valid : x->an.geom.valid; }
static double any_t_enter(const og_any* x) { return x->cascade ? x->cas.t_enter : x->an.geom.t_enter; }
static double any_t_exit(const og_any* x) { return x->cascade ? x->cas.t_exit : x->an.geom.t_exit; }
static int any_next(og_any* x, og_event* ev) {
    return x->cascade ? cascade_next(&x->cas, ev) : an_next(&x->an, ev);
}
static int any_undefined(const og_any* x) { return x->cascade ? x->cas.undefined : x->an.undefined; }
static void any_counts(const og_any* x, int64_t* lookups, int64_t* steps) {
    if (!x->cascade) {
        *lookups = x->an.lookups;
        *steps = x->an.steps;
        return;
    }
    /* CascadeTraversal::lookup_count / step_count :394-397 */
    *lookups = x->cas.finished_lookups + (x->cas.has_sub ? x->cas.sub.lookups : 0);
    *steps = x->cas.finished_steps + (x->cas.has_sub ? x->cas.sub.steps : 0);
}

static int load_ray(const double* p, og_ray* r) {
    for (int a = 0; a < 3; ++a) {
        r->o[a] = p[a];
        r->d[a] = p[3 + a];
    }
    r->tmin = p[6];
    r->tmax = p[7];
    return ray_valid(r);
}

int64_t og_collect_events(const og_sampler* s, const double ray[8], int64_t cap,
                          og_event* events, int64_t counters[2]) {
    og_ray r;
    if (!load_ray(ray, &r)) return -2;
    og_any x;
    any_init(&x, s, &r);
    int64_t n = 0;
    og_event ev;
    while (any_next(&x, &ev)) {
        if (n < cap) events[n] = ev;
        ++n;
    }
    if (counters) any_counts(&x, &counters[0], &counters[1]);
    if (any_undefined(&x)) return -1;
    return n;
}

/* ------------------------------------------------------------------------ */
/* sampling kernels, sampling.hpp:87-122                                     */
/* ------------------------------------------------------------------------ */
static inline double sched_step(const og_sampler* s, double t) { /* StepSchedule::step :36-38 */
    return s->sched_kind == OG_CONSTANT ? s->dt0 : std_max(s->dt0, s->growth * t);
}

/* probes :50-67 and CascadeProbe :417-438 */
static int probe(const og_sampler* s, const og_event* ev) {
    if (ev->grid_level < 0) return 0;
    const og_grid* g = s->levels[(s->cascade || s->n_levels > 1) ? ev->grid_level : 0];
    if (s->analyzer == OG_HDDA) return sparse_query(g, ev->ijk).occupied;
    /* CD: the single-grid kernel probes the dense grid (DenseProbe, sampling.hpp:200-203),
     * the cascade one the distance level (grid_occupancy, :281); both answer ev.occupied */
    if (s->analyzer == OG_CD) return dist_at(g, ev->ijk) == 0;
    return dense_bit(g, ev->ijk);
}

static inline uint32_t pack_cell(const int ijk[3]) {
    return (uint32_t)(ijk[0] & 1023) | ((uint32_t)(ijk[1] & 1023) << 10) |
           ((uint32_t)(ijk[2] & 1023) << 20);
}

int64_t og_sample_ray(const og_sampler* s, const double ray[8], int64_t cap, double* t_starts,
                      double* t_ends, uint32_t* cells, uint8_t* levels, int64_t counters[3],
                      int32_t* status) {
    og_ray r;
    int64_t n = 0, kernel_lookups = 0;
    if (counters) counters[0] = counters[1] = counters[2] = 0;
    if (!load_ray(ray, &r)) {
        if (status) *status = OG_RAY_INVALID;
        return 0;
    }
    og_any x;
    any_init(&x, s, &r);
    if (any_valid(&x)) {
        const double t_end = any_t_exit(&x);
        double t_last = any_t_enter(&x);
        og_event ev;
        while (t_last <= t_end) {
            if (!any_next(&x, &ev)) break;
            if (s->kernel == OG_SKIP && !ev.occupied) continue;
            while (t_last <= ev.t0) t_last += sched_step(s, t_last);
            while (t_last <= ev.t1) {
                int emit = 1;
                if (s->kernel == OG_BRANCH) {
                    ++kernel_lookups;
                    emit = probe(s, &ev);
                }
                const double next = t_last + sched_step(s, t_last);
                if (emit) {
                    if (n < cap) {
                        if (t_starts) t_starts[n] = t_last;
                        if (t_ends) t_ends[n] = next;
                        if (cells) cells[n] = pack_cell(ev.ijk);
                        if (levels) levels[n] = (uint8_t)(ev.level | (ev.grid_level << 2));
                    }
                    ++n;
                }
                t_last = next;
            }
        }
    }
    if (any_undefined(&x)) {
        if (status) *status = OG_RAY_UNDEFINED;
        if (counters) counters[0] = counters[1] = counters[2] = 0;
        return 0;
    }
    if (status) *status = OG_RAY_OK;
    if (counters) {
        any_counts(&x, &counters[0], &counters[1]);
        counters[2] = kernel_lookups;
    }
    return n;
}

int64_t og_sample_batch(const og_sampler* s, const double* rays, int64_t n,
                        int64_t ray_index_base, int64_t cap, int64_t* packed_info,
                        double* t_starts, double* t_ends, int32_t* ray_indices, uint32_t* cells,
                        uint8_t* levels, int32_t* counters, uint8_t* status) {
    int64_t off = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t ctr[3];
        int32_t st = 0;
        const int64_t room = off < cap ? cap - off : 0;
        const int64_t c = og_sample_ray(s, rays + 8 * i, room, t_starts ? t_starts + off : NULL,
                                        t_ends ? t_ends + off : NULL, cells ? cells + off : NULL,
                                        levels ? levels + off : NULL, ctr, &st);
        if (packed_info) {
            packed_info[2 * i] = off;
            packed_info[2 * i + 1] = c;
        }
        if (ray_indices)
            for (int64_t k = 0; k < c && off + k < cap; ++k) ray_indices[off + k] = (int32_t)(ray_index_base + i);
        if (counters)
            for (int a = 0; a < 3; ++a) counters[3 * i + a] = (int32_t)ctr[a];
        if (status) status[i] = (uint8_t)st;
        off += c;
    }
    return off;
}

/* ---------------------------------------------------------------------------
 * compositing consumer (render.hpp)
 * ------------------------------------------------------------------------- */
/* Primitive::contains (render.hpp:44-51) */
static int prim_contains(const og_primitive* q, const double p[3]) {
    if (q->shape == 0) {
        const double dx = p[0] - q->center[0], dy = p[1] - q->center[1], dz = p[2] - q->center[2];
        return dx * dx + dy * dy + dz * dz <= q->radius * q->radius; /* d.dot(d) <= r*r */
    }
    return p[0] >= q->lo[0] && p[1] >= q->lo[1] && p[2] >= q->lo[2] && p[0] < q->hi[0] &&
           p[1] < q->hi[1] && p[2] < q->hi[2];
}

void og_composite(const double ray[8], const double* samples, int64_t n, const og_primitive* prims,
                  int32_t n_prims, const double background[3], int32_t sched_kind, double dt0,
                  double growth, double out[5]) {
    double c[3] = {0.0, 0.0, 0.0}, ws = 0.0, T = 1.0; /* CompositeResult (render.hpp:91-95) */
    for (int64_t i = 0; i < n; ++i) {                  /* render.hpp:104-116 */
        const double t = samples[i];
        double dt;
        if (i + 1 < n) {
            dt = samples[i + 1] - t;
        } else if (sched_kind == OG_LINEAR) { /* StepSchedule::step (sampling.hpp:36-38) */
            const double g = growth * t;
            dt = (dt0 < g) ? g : dt0;
        } else {
            dt = dt0;
        }
        double p[3];
        for (int a = 0; a < 3; ++a) p[a] = ray[a] + ray[3 + a] * t; /* Ray::at (ray.hpp:35) */
        double sigma = 0.0; /* density_at (render.hpp:72-77) */
        for (int32_t k = 0; k < n_prims; ++k)
            if (prim_contains(&prims[k], p)) sigma += prims[k].density;
        if (sigma <= 0.0) continue;
        const double alpha = 1.0 - exp(-sigma * dt);
        const double w = T * alpha;
        double e[3] = {0.0, 0.0, 0.0}, s2 = 0.0; /* emission_at (render.hpp:80-90) */
        for (int32_t k = 0; k < n_prims; ++k)
            if (prim_contains(&prims[k], p)) {
                for (int a = 0; a < 3; ++a) e[a] += prims[k].color[a] * prims[k].density;
                s2 += prims[k].density;
            }
        for (int a = 0; a < 3; ++a) {
            const double em = s2 > 0.0 ? e[a] / s2 : e[a];
            c[a] += em * w;
        }
        ws += w;
        T *= 1.0 - alpha;
    }
    for (int a = 0; a < 3; ++a) c[a] += background[a] * T; /* render.hpp:117 */
    out[0] = c[0];
    out[1] = c[1];
    out[2] = c[2];
    out[3] = ws;
    out[4] = T;
}

void og_set_pixel(const double rgb[3], uint8_t out[3]) { /* render.hpp:133-139 */
    for (int a = 0; a < 3; ++a) {
        const double lo = (0.0 < rgb[a]) ? rgb[a] : 0.0; /* std::max(0.0, v) */
        const double v = (lo < 1.0) ? lo : 1.0;          /* std::min(1.0, .) */
        out[a] = (uint8_t)lround(v * 255.0);
    }
}

double og_psnr(const uint8_t* a, const uint8_t* b, int64_t n) { /* render.hpp:168-182 */
    double sq = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = (double)a[i] - (double)b[i];
        sq += d * d;
    }
    if (sq == 0.0) return 99.0;
    const double mse = sq / (double)n;
    const double v = 10.0 * log10(255.0 * 255.0 / mse);
    return v < 99.0 ? v : 99.0;
}
