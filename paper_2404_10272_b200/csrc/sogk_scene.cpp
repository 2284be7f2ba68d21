// sogk_scene.cpp — host input generators and camera setup (C-ABI part).
//
// Restatements of the reference's deterministic generators so the product
// can synthesize the exact inputs the reference would (the GPU box has no
// reference sources).  tests/test_host_generators.py pins every function here
// bit-for-bit against the unmodified reference (oracle/_ref).  Compiled with
// -ffp-contract=off (no FMA) like the reference build.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "sogk.h"

namespace {

constexpr double kPi = 3.14159265358979323846; // M_PI

struct V3 {
    double x, y, z;
    double operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
    double& operator[](int a) { return a == 0 ? x : (a == 1 ? y : z); }
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 mul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 dvs(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; } // vec.hpp:22
inline double length(V3 a) { return std::sqrt(dot(a, a)); }
inline V3 normalized(V3 a) { return dvs(a, length(a)); }
inline V3 cross(V3 a, V3 o) { // vec.hpp:26-28
    return {a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x};
}

struct Xform { // sog::GridTransform (grid.hpp:18-70)
    int res[3];
    V3 wmin;
    double voxel;
    explicit Xform(const sogk_transform& t) : wmin{t.world_min[0], t.world_min[1], t.world_min[2]} {
        for (int a = 0; a < 3; ++a) res[a] = t.res[a];
        voxel = t.voxel_size;
    }
    V3 wmax() const {
        return add(wmin, mul(V3{double(res[0]), double(res[1]), double(res[2])}, voxel));
    }
    V3 center_of(int x, int y, int z) const { // index_to_world_center :44-46
        return add(wmin, mul(V3{x + 0.5, y + 0.5, z + 0.5}, voxel));
    }
    void world_to_index(V3 p, int out[3]) const { // :48-52
        const V3 g = dvs(sub(p, wmin), voxel);
        out[0] = int(std::floor(g.x));
        out[1] = int(std::floor(g.y));
        out[2] = int(std::floor(g.z));
    }
    uint64_t count() const { return uint64_t(res[0]) * res[1] * res[2]; }
    uint64_t lin(int x, int y, int z) const {
        return (uint64_t(z) * res[1] + y) * res[0] + x;
    }
};

bool valid_transform(const sogk_transform* t) {
    return t && t->res[0] >= 1 && t->res[1] >= 1 && t->res[2] >= 1 && t->voxel_size > 0.0;
}

inline double uniform01(std::mt19937_64& rng) { // scene_gen.hpp:47-49
    return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}
inline double uniform(std::mt19937_64& rng, double lo, double hi) { // :50-52
    return lo + (hi - lo) * uniform01(rng);
}

struct Prim { // Primitive (render.hpp:19-55)
    bool sphere;
    V3 center;
    double radius;
    V3 lo, hi;
    double density;
    V3 color;
    bool contains(V3 p) const {
        if (sphere) {
            const V3 d = sub(p, center);
            return dot(d, d) <= radius * radius;
        }
        return p.x >= lo.x && p.y >= lo.y && p.z >= lo.z && p.x < hi.x && p.y < hi.y &&
               p.z < hi.z;
    }
};

inline void set_bit(uint8_t* bits, uint64_t idx) { bits[idx >> 3] |= uint8_t(1u << (idx & 7)); }

// rasterize_occupancy + binarize (scene_gen.hpp:59-88, grid.hpp:169-198)
void rasterize(const std::vector<Prim>& prims, const Xform& t, double threshold, uint8_t* bits) {
    std::vector<double> field(t.count(), 0.0);
    for (const Prim& p : prims) {
        V3 lo, hi;
        if (p.sphere) {
            const V3 r{p.radius, p.radius, p.radius};
            lo = sub(p.center, r);
            hi = add(p.center, r);
        } else {
            lo = p.lo;
            hi = p.hi;
        }
        int ilo[3], ihi[3];
        t.world_to_index(lo, ilo);
        t.world_to_index(hi, ihi);
        const int x0 = std::max(0, ilo[0]), x1 = std::min(t.res[0] - 1, ihi[0]);
        const int y0 = std::max(0, ilo[1]), y1 = std::min(t.res[1] - 1, ihi[1]);
        const int z0 = std::max(0, ilo[2]), z1 = std::min(t.res[2] - 1, ihi[2]);
        for (int z = z0; z <= z1; ++z)
            for (int y = y0; y <= y1; ++y)
                for (int x = x0; x <= x1; ++x)
                    if (p.contains(t.center_of(x, y, z))) field[t.lin(x, y, z)] += p.density;
    }
    std::memset(bits, 0, (t.count() + 7) / 8);
    for (uint64_t i = 0; i < t.count(); ++i)
        if (field[i] > threshold) set_bit(bits, i);
}

// generate_scene's primitive list (scene_gen.hpp:94-176); returns false for the random kind
bool make_prims(int kind, const Xform& t, int count, std::mt19937_64& rng, std::vector<Prim>& out) {
    const V3 wmin = t.wmin, wmax = t.wmax();
    const V3 extent = sub(wmax, wmin);
    const V3 center = add(wmin, mul(extent, 0.5));
    const double min_extent = std::min({extent.x, extent.y, extent.z});
    switch (kind) {
        case SOGK_BLOBS:
            for (int i = 0; i < count; ++i) {
                V3 c;
                for (int a = 0; a < 3; ++a)
                    c[a] = uniform(rng, wmin[a] + 0.15 * extent[a], wmax[a] - 0.15 * extent[a]);
                const double r = uniform(rng, 0.04, 0.10) * min_extent;
                const double sigma = uniform(rng, 4.0, 12.0) / min_extent;
                V3 rgb;
                for (int k = 0; k < 3; ++k) rgb[k] = uniform(rng, 0.1, 1.0);
                out.push_back(Prim{true, c, r, {}, {}, sigma, rgb});
            }
            return true;
        case SOGK_SHELL: {
            const int n = std::max(64, count);
            const double shell_radius = 0.35 * min_extent;
            const double bump = 1.6 * shell_radius * std::sqrt(kPi / n);
            const double golden = kPi * (3.0 - std::sqrt(5.0));
            for (int i = 0; i < n; ++i) {
                const double y = 1.0 - 2.0 * (i + 0.5) / n;
                const double r = std::sqrt(1.0 - y * y);
                const double phi = golden * i;
                const V3 dir{r * std::cos(phi), y, r * std::sin(phi)};
                const V3 c = add(center, mul(dir, shell_radius));
                const V3 rgb = add(V3{0.5, 0.5, 0.5}, mul(dir, 0.45));
                out.push_back(Prim{true, c, bump, {}, {}, 8.0 / min_extent, rgb});
            }
            return true;
        }
        case SOGK_SPONGE: {
            const int cells = 4;
            const double inset = 0.1 * min_extent;
            const V3 lo = add(wmin, V3{inset, inset, inset});
            const V3 hi = sub(wmax, V3{inset, inset, inset});
            const double w = 0.01 * min_extent;
            const double sigma = 10.0 / min_extent;
            auto plane = [&](int axis, int i) { return lo[axis] + (hi[axis] - lo[axis]) * i / cells; };
            for (int axis = 0; axis < 3; ++axis) {
                const int u = (axis + 1) % 3, v = (axis + 2) % 3;
                V3 col{0.15, 0.15, 0.15};
                col[axis] = 0.9;
                for (int i = 0; i <= cells; ++i)
                    for (int j = 0; j <= cells; ++j) {
                        V3 blo{0, 0, 0}, bhi{0, 0, 0};
                        blo[axis] = lo[axis];
                        bhi[axis] = hi[axis];
                        blo[u] = plane(u, i) - w;
                        bhi[u] = plane(u, i) + w;
                        blo[v] = plane(v, j) - w;
                        bhi[v] = plane(v, j) + w;
                        out.push_back(Prim{false, {}, 0.0, blo, bhi, sigma, col});
                    }
            }
            return true;
        }
        default:
            out.push_back(Prim{false, {}, 0.0, wmin, wmax, 3.0 / min_extent, {0.7, 0.7, 0.7}});
            return false;
    }
}

void store_ray(V3 o, V3 d, double tmin, double tmax, double* out) {
    out[0] = o.x;
    out[1] = o.y;
    out[2] = o.z;
    out[3] = d.x;
    out[4] = d.y;
    out[5] = d.z;
    out[6] = tmin;
    out[7] = tmax;
}

} // namespace

extern "C" {

int sogk_scene_generate(int kind, const sogk_transform* tr, uint64_t seed, double fraction,
                        int32_t count, double threshold, uint8_t* h_bits, double* occupancy) {
    if (!valid_transform(tr) || !h_bits || kind < 0 || kind > 3) return SOGK_INVALID_ARG;
    if (fraction < 0.0 || fraction > 1.0 || count < 1) return SOGK_INVALID_ARG; // :96-99
    const Xform t(*tr);
    std::mt19937_64 rng(seed);
    std::vector<Prim> prims;
    if (make_prims(kind, t, count, rng, prims)) {
        rasterize(prims, t, threshold, h_bits);
    } else { // random: iid Bernoulli voxels (:179-186)
        std::memset(h_bits, 0, (t.count() + 7) / 8);
        uint64_t i = 0;
        for (int z = 0; z < t.res[2]; ++z)
            for (int y = 0; y < t.res[1]; ++y)
                for (int x = 0; x < t.res[0]; ++x, ++i)
                    if (uniform01(rng) < fraction) set_bit(h_bits, i);
    }
    if (occupancy) { // occupancy_fraction (grid.hpp:150-158)
        uint64_t n = 0;
        for (uint64_t i = 0; i < t.count(); ++i) n += (h_bits[i >> 3] >> (i & 7)) & 1u;
        *occupancy = double(n) / double(t.count());
    }
    return SOGK_OK;
}

int sogk_scene_analytic(int kind, const sogk_transform* tr, uint64_t seed, int32_t count,
                        sogk_primitive* h_prims, int32_t cap, int32_t* n_prims,
                        double background[3]) {
    if (!valid_transform(tr) || !n_prims || kind < 0 || kind > 3 || count < 1)
        return SOGK_INVALID_ARG;
    const Xform t(*tr);
    std::mt19937_64 rng(seed);
    std::vector<Prim> prims;
    make_prims(kind, t, count, rng, prims);
    *n_prims = int32_t(prims.size());
    if (background) { // scene.background (scene_gen.hpp:112)
        background[0] = 0.05;
        background[1] = 0.06;
        background[2] = 0.08;
    }
    if (!h_prims) return SOGK_OK; // size query
    if (cap < int32_t(prims.size())) return SOGK_INSUFFICIENT_CAPACITY;
    for (size_t i = 0; i < prims.size(); ++i) {
        const Prim& p = prims[i];
        sogk_primitive& q = h_prims[i];
        q.shape = p.sphere ? SOGK_SPHERE : SOGK_BOX;
        for (int a = 0; a < 3; ++a) {
            q.center[a] = p.center[a];
            q.lo[a] = p.lo[a];
            q.hi[a] = p.hi[a];
            q.color[a] = p.color[a];
        }
        q.radius = p.radius;
        q.density = p.density;
    }
    return SOGK_OK;
}

int sogk_scene_cascade(int kind, const sogk_transform* base, uint64_t seed, double fraction,
                       int32_t count, double threshold, int32_t levels, uint8_t* h_bits,
                       sogk_transform* out) {
    if (!valid_transform(base) || !h_bits || !out || levels < 1 || kind < 0 || kind > 3)
        return SOGK_INVALID_ARG;
    if (fraction < 0.0 || fraction > 1.0 || count < 1) return SOGK_INVALID_ARG;
    const Xform b0(*base);
    std::mt19937_64 rng(seed);
    std::vector<Prim> prims;
    make_prims(kind, b0, count, rng, prims); // the analytic scene of generate_scene
    // build_dense_cascade (scene_gen.hpp:196-209)
    const V3 extent = sub(b0.wmax(), b0.wmin);
    const V3 center = add(b0.wmin, mul(extent, 0.5));
    const uint64_t nb = (b0.count() + 7) / 8;
    for (int b = 0; b < levels; ++b) {
        const double scale = static_cast<double>(1u << b);
        const V3 wm = sub(center, mul(extent, 0.5 * scale));
        sogk_transform t = *base;
        t.world_min[0] = wm.x;
        t.world_min[1] = wm.y;
        t.world_min[2] = wm.z;
        t.voxel_size = base->voxel_size * scale;
        out[b] = t;
        rasterize(prims, Xform(t), threshold, h_bits + nb * b);
    }
    return SOGK_OK;
}

int sogk_probe_rays(const sogk_transform* tr, int64_t count, uint64_t seed, double* h_rays) {
    if (!valid_transform(tr) || count < 0 || (count && !h_rays)) return SOGK_INVALID_ARG;
    const Xform t(*tr);
    std::mt19937_64 rng(seed); // make_probe_rays, bench.hpp:628-649
    const V3 extent = sub(t.wmax(), t.wmin);
    const V3 center = add(t.wmin, mul(extent, 0.5));
    const double radius = length(extent);
    int64_t n = 0;
    while (n < count) {
        const double z = uniform(rng, -1.0, 1.0);
        const double phi = uniform(rng, 0.0, 2.0 * kPi);
        const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
        const V3 pos = add(center, mul(V3{r * std::cos(phi), z, r * std::sin(phi)}, radius));
        V3 aim;
        for (int a = 0; a < 3; ++a)
            aim[a] = uniform(rng, t.wmin[a] + 0.1 * extent[a], t.wmax()[a] - 0.1 * extent[a]);
        const V3 dir = sub(aim, pos);
        if (length(dir) < 1e-12) continue;
        store_ray(pos, normalized(dir), 0.0, 1e9, h_rays + 8 * n); // Ray::from_dir
        ++n;
    }
    return SOGK_OK;
}

int sogk_random_rays(const sogk_transform* tr, int64_t count, uint64_t seed, double* h_rays) {
    if (!valid_transform(tr) || count < 0 || (count && !h_rays)) return SOGK_INVALID_ARG;
    const Xform t(*tr);
    std::mt19937_64 rng(seed); // testsupport::random_ray, test_support.hpp:66-82
    const V3 extent = sub(t.wmax(), t.wmin);
    const V3 center = add(t.wmin, mul(extent, 0.5));
    const double radius = length(extent);
    for (int64_t n = 0; n < count;) {
        const double z = uniform(rng, -1.0, 1.0);
        const double phi = uniform(rng, 0.0, 2.0 * kPi);
        const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
        const V3 pos = add(center, mul(V3{r * std::cos(phi), z, r * std::sin(phi)}, radius));
        V3 aim;
        for (int a = 0; a < 3; ++a)
            aim[a] = uniform(rng, t.wmin[a] + 0.05 * extent[a], t.wmax()[a] - 0.05 * extent[a]);
        const V3 dir = sub(aim, pos);
        if (length(dir) > 1e-9) {
            store_ray(pos, normalized(dir), 0.0, 1e9, h_rays + 8 * n);
            ++n;
        }
    }
    return SOGK_OK;
}

int sogk_random_grid(const sogk_transform* tr, uint64_t seed, double fraction, uint8_t* h_bits) {
    if (!valid_transform(tr) || !h_bits) return SOGK_INVALID_ARG;
    const Xform t(*tr);
    std::mt19937_64 rng(seed); // test_support.hpp:29-37
    std::memset(h_bits, 0, (t.count() + 7) / 8);
    for (int z = 0; z < t.res[2]; ++z)
        for (int y = 0; y < t.res[1]; ++y)
            for (int x = 0; x < t.res[0]; ++x)
                if (uniform01(rng) < fraction) set_bit(h_bits, t.lin(x, y, z));
    return SOGK_OK;
}

int sogk_random_blocky_grid(const sogk_transform* tr, uint64_t seed, double block_fraction,
                            double noise_fraction, uint8_t* h_bits) {
    if (!valid_transform(tr) || !h_bits) return SOGK_INVALID_ARG;
    const Xform t(*tr);
    std::mt19937_64 rng(seed); // test_support.hpp:41-62
    std::memset(h_bits, 0, (t.count() + 7) / 8);
    const int bx = (t.res[0] + 7) / 8, by = (t.res[1] + 7) / 8, bz = (t.res[2] + 7) / 8;
    for (int z = 0; z < bz; ++z)
        for (int y = 0; y < by; ++y)
            for (int x = 0; x < bx; ++x) {
                if (uniform01(rng) >= block_fraction) continue;
                for (int lz = 0; lz < 8; ++lz)
                    for (int ly = 0; ly < 8; ++ly)
                        for (int lx = 0; lx < 8; ++lx) {
                            const int i = x * 8 + lx, j = y * 8 + ly, k = z * 8 + lz;
                            if (i < t.res[0] && j < t.res[1] && k < t.res[2])
                                set_bit(h_bits, t.lin(i, j, k));
                        }
            }
    for (int z = 0; z < t.res[2]; ++z)
        for (int y = 0; y < t.res[1]; ++y)
            for (int x = 0; x < t.res[0]; ++x)
                if (uniform01(rng) < noise_fraction) set_bit(h_bits, t.lin(x, y, z));
    return SOGK_OK;
}

// Camera::pixel_ray's per-camera terms (camera.hpp:170-174)
int sogk_camera_setup(const double position[3], const double target[3], const double up[3],
                      double vfov_deg, int32_t width, int32_t height, double t_far,
                      sogk_camera* out) {
    if (!position || !target || !up || !out || width < 1 || height < 1) return SOGK_INVALID_ARG;
    const V3 pos{position[0], position[1], position[2]};
    const V3 forward = normalized(sub(V3{target[0], target[1], target[2]}, pos));
    const V3 right = normalized(cross(forward, V3{up[0], up[1], up[2]}));
    const V3 cam_up = cross(right, forward);
    for (int a = 0; a < 3; ++a) {
        out->position[a] = pos[a];
        out->forward[a] = forward[a];
        out->right[a] = right[a];
        out->cam_up[a] = cam_up[a];
    }
    out->tan_half = std::tan(vfov_deg * 0.5 * kPi / 180.0);
    out->aspect = static_cast<double>(width) / height;
    out->t_far = t_far;
    out->width = width;
    out->height = height;
    return SOGK_OK;
}

// host twin of the device raygen (camera.hpp:175-178)
int sogk_camera_rays_host(const sogk_camera* c, int64_t first, int64_t n, double* h_rays) {
    if (!c || first < 0 || n < 0 || (n && !h_rays)) return SOGK_INVALID_ARG;
    if (first + n > int64_t(c->width) * c->height) return SOGK_INVALID_ARG; // out_of_range
    const V3 f{c->forward[0], c->forward[1], c->forward[2]};
    const V3 r{c->right[0], c->right[1], c->right[2]};
    const V3 cu{c->cam_up[0], c->cam_up[1], c->cam_up[2]};
    const V3 pos{c->position[0], c->position[1], c->position[2]};
    for (int64_t i = 0; i < n; ++i) {
        const int64_t pix = first + i;
        const int px = int(pix % c->width), py = int(pix / c->width);
        const double u = ((px + 0.5) / c->width * 2.0 - 1.0) * c->tan_half * c->aspect;
        const double v = (1.0 - (py + 0.5) / c->height * 2.0) * c->tan_half;
        const V3 dir = normalized(add(add(f, mul(r, u)), mul(cu, v)));
        store_ray(pos, dir, 0.0, c->t_far, h_rays + 8 * i);
    }
    return SOGK_OK;
}

} // extern "C"
