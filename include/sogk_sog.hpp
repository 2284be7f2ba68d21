// sogk_sog.hpp — C++ drop-in shim: the reference's own types and entry points
// (namespace sog, /root/reference/proj/include/sog/) on top of the sm_100a
// C-ABI (sogk.h).  Header-only; include it in code that already includes the
// reference library and link libsogk.so:
//
//     #include <sog/sog.hpp>
//     #include "sogk_sog.hpp"
//     sog::gpu::DeviceSparseGrid vdb = sog::gpu::build_sparse(dense);        // sparse.hpp:333
//     sog::gpu::Sampler hdda(vdb, sog::KernelKind::skip, sched);             // make_sampler, bench.hpp:382
//     sog::gpu::PackedSamples out = hdda.sample_rays(rays);                  // batched run_sampler
//     sog::SampleRun one = hdda(ray);                                        // run_sampler, sampling.hpp:182
//
// Errors follow the reference: std::invalid_argument for bad arguments,
// sog::io_error for SOG0/SOG1 problems, std::runtime_error for device failures.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sog/camera.hpp"
#include "sog/distance.hpp"
#include "sog/io.hpp"
#include "sog/render.hpp"
#include "sog/sampling.hpp"
#include "sogk.h"

namespace sog::gpu {

static_assert(sizeof(Ray) == 8 * sizeof(double), "sog::Ray must be 8 packed doubles");

inline void check(int status) {
    if (status == SOGK_OK) return;
    char buf[512];
    sogk_last_error(buf, sizeof buf);
    const std::string msg(buf);
    switch (status) {
        case SOGK_INVALID_ARG: throw std::invalid_argument(msg);
        case SOGK_IO_ERROR: {
            io_errc c = io_errc::corrupt;
            if (msg.find("bad magic") != std::string::npos) c = io_errc::bad_magic;
            else if (msg.find("bad version") != std::string::npos) c = io_errc::bad_version;
            else if (msg.find("truncated") != std::string::npos) c = io_errc::truncated;
            throw io_error(c, msg);
        }
        default: throw std::runtime_error(std::string(sogk_status_string(status)) + ": " + msg);
    }
}

inline sogk_transform to_c(const GridTransform& t) {
    sogk_transform c{};
    for (int a = 0; a < 3; ++a) {
        c.res[a] = t.resolution[a];
        c.world_min[a] = t.world_min[a];
    }
    c.voxel_size = t.voxel_size;
    return c;
}

struct GridDeleter {
    void operator()(sogk_grid* g) const { sogk_grid_destroy(g); }
};
using GridHandle = std::shared_ptr<sogk_grid>;

/// DenseGrid (grid.hpp:120-165) resident in HBM.
class DeviceDenseGrid {
public:
    explicit DeviceDenseGrid(const DenseGrid& d, void* stream = nullptr) : t_(d.transform()) {
        const sogk_transform c = to_c(t_);
        sogk_grid* g = nullptr;
        check(sogk_grid_create_dense(&c, d.payload().data(), d.payload().size(), stream, &g));
        h_.reset(g, GridDeleter{});
    }
    const GridTransform& transform() const { return t_; }
    sogk_grid* handle() const { return h_.get(); }
    DenseGrid to_host() const {
        DenseGrid d(t_);
        check(sogk_grid_download_dense(h_.get(), d.payload().data(), d.payload().size()));
        return d;
    }

private:
    GridTransform t_;
    GridHandle h_;
};

/// SparseGrid (sparse.hpp:141-218) as the GPU VDB layout.
class DeviceSparseGrid {
public:
    DeviceSparseGrid(sogk_grid* g, const GridTransform& t) : t_(t), h_(g, GridDeleter{}) {}
    const GridTransform& transform() const { return t_; }
    sogk_grid* handle() const { return h_.get(); }
    sogk_grid_info info() const {
        sogk_grid_info i{};
        check(sogk_grid_get_info(h_.get(), &i));
        return i;
    }
    std::size_t leaf_count() const { return std::size_t(info().leaf_count); }
    std::size_t memory_bytes() const { return std::size_t(info().memory_bytes); } // io.hpp:227
    /// serialize_sparse (io.hpp:161-181): byte-identical to the reference tree's SOG1
    std::vector<std::uint8_t> serialize() const {
        std::size_t n = 0;
        check(sogk_grid_export_sog1(h_.get(), nullptr, &n));
        std::vector<std::uint8_t> out(n);
        check(sogk_grid_export_sog1(h_.get(), out.data(), &n));
        return out;
    }
    /// the reference tree itself (deserialize_sparse of the exported bytes)
    SparseGrid to_host() const { return deserialize_sparse(serialize()); }

private:
    GridTransform t_;
    GridHandle h_;
};

/// build_sparse (sparse.hpp:333-371) on the GPU.
inline DeviceSparseGrid build_sparse(const DeviceDenseGrid& d, void* stream = nullptr) {
    sogk_grid* g = nullptr;
    check(sogk_grid_build_vdb(d.handle(), stream, &g));
    return DeviceSparseGrid(g, d.transform());
}
inline DeviceSparseGrid build_sparse(const DenseGrid& d, void* stream = nullptr) {
    return build_sparse(DeviceDenseGrid(d, stream), stream);
}

/// DistanceGrid (distance.hpp:15-43) in HBM: the grid the CD analyzer marches.
class DeviceDistanceGrid {
public:
    DeviceDistanceGrid(sogk_grid* g, const GridTransform& t) : t_(t), h_(g, GridDeleter{}) {}
    const GridTransform& transform() const { return t_; }
    sogk_grid* handle() const { return h_.get(); }
    /// the reference DistanceGrid (same values: both transforms are exact)
    DistanceGrid to_host() const {
        std::vector<std::int32_t> d(std::size_t(t_.voxel_count()));
        std::int32_t ae = 0;
        check(sogk_grid_download_distance(h_.get(), d.data(), d.size(), &ae));
        return DistanceGrid(t_, std::move(d), ae != 0);
    }

private:
    GridTransform t_;
    GridHandle h_;
};

/// build_distance (distance.hpp:45-103) on the GPU.
inline DeviceDistanceGrid build_distance(const DeviceDenseGrid& d, void* stream = nullptr) {
    sogk_grid* g = nullptr;
    check(sogk_grid_build_distance(d.handle(), stream, &g));
    return DeviceDistanceGrid(g, d.transform());
}

/// Packed sample intervals of a ray batch (sogk.h output contract).
struct PackedSamples {
    std::vector<std::int64_t> packed_info; // [n][2] offset, count
    std::vector<double> t_starts, t_ends;
    std::vector<std::int32_t> ray_indices;
    std::vector<std::uint32_t> cells;
    std::vector<std::uint8_t> levels;
    std::vector<std::uint8_t> status;
    std::vector<std::int32_t> counters; // [n][3]
    std::int64_t stats[SOGK_STATS_LEN] = {};

    std::size_t size() const { return packed_info.size() / 2; }
    /// the reference SampleBuffer of ray r (sampling.hpp:42)
    SampleBuffer samples(std::size_t r) const {
        const auto off = packed_info[2 * r], cnt = packed_info[2 * r + 1];
        return SampleBuffer(t_starts.begin() + off, t_starts.begin() + off + cnt);
    }
    /// the reference SampleRun of ray r (sampling.hpp:157-164)
    SampleRun run(std::size_t r) const {
        SampleRun out;
        out.samples = samples(r);
        out.analyzer_lookups = counters[3 * r];
        out.analyzer_steps = counters[3 * r + 1];
        out.kernel_lookups = counters[3 * r + 2];
        return out;
    }
};

struct SamplerDeleter {
    void operator()(sogk_sampler* s) const { sogk_sampler_destroy(s); }
};

/// One variant of the reference's variant matrix (bench.hpp:30-64): dense+dda, sparse+hdda or
/// dense+cd (the distance grid), each {branch, skip}, over one grid or a cascade
/// (sampling.hpp:222-462).
class Sampler {
public:
    Sampler(const DeviceDenseGrid& g, KernelKind k, const StepSchedule& s)
        : Sampler({g.handle()}, SOGK_DDA, k, s, false) {}
    Sampler(const DeviceSparseGrid& g, KernelKind k, const StepSchedule& s)
        : Sampler({g.handle()}, SOGK_HDDA, k, s, false) {}
    Sampler(const DeviceDistanceGrid& g, KernelKind k, const StepSchedule& s)
        : Sampler({g.handle()}, SOGK_CD, k, s, false) {}
    Sampler(const std::vector<DeviceDistanceGrid>& cascade, KernelKind k, const StepSchedule& s)
        : Sampler(handles(cascade), SOGK_CD, k, s, true) {}
    Sampler(const std::vector<DeviceDenseGrid>& cascade, KernelKind k, const StepSchedule& s)
        : Sampler(handles(cascade), SOGK_DDA, k, s, true) {}
    Sampler(const std::vector<DeviceSparseGrid>& cascade, KernelKind k, const StepSchedule& s)
        : Sampler(handles(cascade), SOGK_HDDA, k, s, true) {}

    /// Batched run_sampler / run_cascade_sampler: host rays in, host packed samples out.
    PackedSamples sample_rays(std::span<const Ray> rays, std::int64_t ray_index_base = 0,
                              void* stream = nullptr) const {
        const std::int64_t n = std::int64_t(rays.size());
        PackedSamples out;
        out.packed_info.resize(2 * n);
        out.status.resize(n);
        out.counters.resize(3 * n);
        std::int64_t cap = std::max<std::int64_t>(1024, 64 * n);
        for (;;) {
            out.t_starts.resize(cap);
            out.t_ends.resize(cap);
            out.ray_indices.resize(cap);
            out.cells.resize(cap);
            out.levels.resize(cap);
            const int st = sogk_sample_host(
                s_.get(), reinterpret_cast<const double*>(rays.data()), n, ray_index_base, cap,
                out.packed_info.data(), out.t_starts.data(), out.t_ends.data(), out.ray_indices.data(),
                out.cells.data(), out.levels.data(), out.status.data(), out.counters.data(), out.stats,
                stream);
            if (st == SOGK_INSUFFICIENT_CAPACITY) {
                cap = out.stats[SOGK_STAT_TOTAL_SAMPLES];
                continue;
            }
            check(st);
            break;
        }
        const std::size_t total = std::size_t(out.stats[SOGK_STAT_TOTAL_SAMPLES]);
        out.t_starts.resize(total);
        out.t_ends.resize(total);
        out.ray_indices.resize(total);
        out.cells.resize(total);
        out.levels.resize(total);
        if (out.stats[SOGK_STAT_INVALID_RAYS])
            throw std::invalid_argument("ray direction must be unit length and 0 <= t_min < t_max");
        if (out.stats[SOGK_STAT_UNDEFINED_RAYS])
            throw std::runtime_error("reference HDDA does not terminate on some rays (edge-crossing spin)");
        return out;
    }

    /// This rank's share of a ray batch that every rank holds (multi-GPU, one process per
    /// GPU): the contiguous range shard_range(n, world, rank) sampled with global
    /// ray_indices.  Concatenating the ranks' outputs in rank order (offsets shifted by the
    /// earlier ranks' totals) gives sample_rays(rays), for any world size.
    PackedSamples sample_shard(std::span<const Ray> rays, int world, int rank,
                               void* stream = nullptr) const;

    /// run_sampler for one ray (drop-in; prefer sample_rays for throughput)
    SampleRun operator()(const Ray& ray) const { return sample_rays({&ray, 1}).run(0); }

    sogk_sampler* handle() const { return s_.get(); }

private:
    template <class G>
    static std::vector<sogk_grid*> handles(const std::vector<G>& gs) {
        std::vector<sogk_grid*> h;
        for (const auto& g : gs) h.push_back(g.handle());
        return h;
    }
    Sampler(std::vector<sogk_grid*> levels, int analyzer, KernelKind k, const StepSchedule& s,
            bool cascade) {
        sogk_sampler_desc d{};
        d.analyzer = analyzer;
        d.kernel = k == KernelKind::branch ? SOGK_BRANCH : SOGK_SKIP;
        d.schedule = s.kind == StepSchedule::Kind::constant ? SOGK_CONSTANT : SOGK_LINEAR;
        d.dt0 = s.dt0;
        d.growth = s.growth;
        d.cascade = cascade ? 1 : 0;
        sogk_sampler* h = nullptr;
        check(sogk_sampler_create(const_cast<const sogk_grid* const*>(levels.data()),
                                  int(levels.size()), &d, &h));
        s_.reset(h, SamplerDeleter{});
    }
    std::shared_ptr<sogk_sampler> s_;
};

/// Contiguous ray range [first, first + count) of `rank` among `world` ranks: ceil(n / world)
/// rays per rank, the last ranks possibly short or empty.  The reference splits a frame into
/// row chunks the same way (render_frame, bench.hpp:446-450: rows_per = ceil(height / n)), and
/// its output does not depend on the split; rays are independent, so no collective follows.
struct ShardRange {
    std::int64_t first = 0, count = 0;
};
inline ShardRange shard_range(std::int64_t n, int world, int rank) {
    if (world < 1 || rank < 0 || rank >= world || n < 0)
        throw std::invalid_argument("shard_range: need 0 <= rank < world and n >= 0");
    const std::int64_t per = (n + world - 1) / world;
    ShardRange r;
    r.first = std::min<std::int64_t>(n, per * rank);
    r.count = std::min<std::int64_t>(n, r.first + per) - r.first;
    return r;
}

inline PackedSamples Sampler::sample_shard(std::span<const Ray> rays, int world, int rank,
                                           void* stream) const {
    const ShardRange sr = shard_range(std::int64_t(rays.size()), world, rank);
    return sample_rays(rays.subspan(std::size_t(sr.first), std::size_t(sr.count)), sr.first, stream);
}

/// run_sampler overloads (sampling.hpp:166-196) over device grids
inline SampleRun run_sampler(const Ray& ray, const DeviceDenseGrid& g, KernelKind k,
                             const StepSchedule& s) {
    return Sampler(g, k, s)(ray);
}
inline SampleRun run_sampler(const Ray& ray, const DeviceSparseGrid& g, KernelKind k,
                             const StepSchedule& s) {
    return Sampler(g, k, s)(ray);
}

/// make_sampler (bench.hpp:382-413) for the GPU variants: the std::function the
/// reference's render_frame / run_matrix consume.
inline std::function<SampleRun(const Ray&)> make_sampler(const Sampler& s) {
    return [s](const Ray& r) { return s(r); };
}

/// Event streams of a ray batch (the reference's traverse entry points, traversal.hpp:120-359):
/// ray r's events exactly as collect_events(Analyzer(grid, ray)) returns them, and the
/// analyzer's lookup_count() / step_count() after the last one.
struct EventStreams {
    std::vector<std::int64_t> event_info; // [n][2] offset, count
    std::vector<sogk_event> events;
    std::vector<std::uint8_t> status;     // SOGK_RAY_OK / _INVALID / _UNDEFINED
    std::vector<std::int32_t> counters;   // [n][2] lookup_count, step_count
    std::int64_t stats[SOGK_STATS_LEN] = {};

    std::size_t size() const { return event_info.size() / 2; }
    static TraversalEvent to_ref(const sogk_event& e) {
        TraversalEvent t;
        t.ijk = Vec3i{e.ijk[0], e.ijk[1], e.ijk[2]};
        t.level = static_cast<Level>(e.level);
        t.t0 = e.t0;
        t.t1 = e.t1;
        t.occupied = e.occupied != 0;
        return t;
    }
    /// collect_events of ray r (traversal.hpp:339-343)
    std::vector<TraversalEvent> ray_events(std::size_t r) const {
        std::vector<TraversalEvent> out;
        for (std::int64_t k = 0; k < event_info[2 * r + 1]; ++k)
            out.push_back(to_ref(events[std::size_t(event_info[2 * r] + k)]));
        return out;
    }
    /// the CascadeTraversal events of ray r (sampling.hpp:297-299): grid_level included
    std::vector<CascadeEvent> ray_cascade_events(std::size_t r) const {
        std::vector<CascadeEvent> out;
        for (std::int64_t k = 0; k < event_info[2 * r + 1]; ++k) {
            const sogk_event& e = events[std::size_t(event_info[2 * r] + k)];
            CascadeEvent c;
            static_cast<TraversalEvent&>(c) = to_ref(e);
            c.grid_level = e.grid_level;
            out.push_back(c);
        }
        return out;
    }
    long lookup_count(std::size_t r) const { return counters[2 * r]; }
    long step_count(std::size_t r) const { return counters[2 * r + 1]; }
};

/// DdaTraversal / HddaTraversal / CdTraversal / CascadeTraversal (traversal.hpp:120-337,
/// sampling.hpp:305-415) over ray batches on the GPU: the analyzer is the grid's
/// (dense -> DDA, VDB -> HDDA, distance -> CD; a vector of levels -> the cascade).
class Traverser {
public:
    template <class G>
    explicit Traverser(const G& grid) : s_(grid, KernelKind::skip, StepSchedule::constant(1.0)) {}

    EventStreams traverse_rays(std::span<const Ray> rays, void* stream = nullptr) const {
        const std::int64_t n = std::int64_t(rays.size());
        EventStreams out;
        out.event_info.resize(2 * n);
        out.status.resize(n);
        out.counters.resize(2 * n);
        std::int64_t cap = std::max<std::int64_t>(256, 64 * n);
        for (;;) {
            out.events.resize(std::size_t(cap));
            const int st = sogk_traverse_host(s_.handle(), reinterpret_cast<const double*>(rays.data()), n,
                                              cap, out.event_info.data(), out.events.data(), out.status.data(),
                                              out.counters.data(), out.stats, stream);
            if (st == SOGK_INSUFFICIENT_CAPACITY) {
                cap = out.stats[SOGK_STAT_TOTAL_SAMPLES];
                continue;
            }
            check(st);
            break;
        }
        out.events.resize(std::size_t(out.stats[SOGK_STAT_TOTAL_SAMPLES]));
        return out;
    }

    /// collect_events(Analyzer(grid, ray)) for one ray; the reference's next() never returns
    /// on the edge-crossing spin rays: those throw instead of hanging
    std::vector<TraversalEvent> collect_events(const Ray& ray) const {
        const EventStreams e = traverse_rays({&ray, 1});
        if (e.status[0] == SOGK_RAY_UNDEFINED)
            throw std::runtime_error("the reference analyzer never returns on this ray (edge-crossing spin)");
        return e.ray_events(0);
    }

private:
    Sampler s_;
};

/// SparseGrid::query (sparse.hpp:163-171) on the GPU, one point
inline QueryResult query(const DeviceSparseGrid& g, const Vec3i& ijk) {
    const std::int32_t p[3] = {ijk.x, ijk.y, ijk.z};
    sogk_query q{};
    check(sogk_grid_query_host(g.handle(), p, 1, &q));
    QueryResult r;
    r.occupied = q.occupied != 0;
    r.level = static_cast<Level>(q.level);
    r.origin = Vec3i{q.origin[0], q.origin[1], q.origin[2]};
    r.extent = q.extent;
    return r;
}

/// AnalyticScene (render.hpp:58-92) in HBM.
class DeviceScene {
public:
    explicit DeviceScene(const AnalyticScene& scene) {
        scene.validate();
        std::vector<sogk_primitive> p;
        for (const Primitive& q : scene.primitives) {
            sogk_primitive c{};
            c.shape = q.shape == Primitive::Shape::sphere ? SOGK_SPHERE : SOGK_BOX;
            for (int a = 0; a < 3; ++a) {
                c.center[a] = q.center[a];
                c.lo[a] = q.lo[a];
                c.hi[a] = q.hi[a];
                c.color[a] = q.color[a];
            }
            c.radius = q.radius;
            c.density = q.density;
            p.push_back(c);
        }
        const double bg[3] = {scene.background.x, scene.background.y, scene.background.z};
        sogk_scene* h = nullptr;
        check(sogk_scene_create(p.data(), std::int32_t(p.size()), bg, &h));
        h_.reset(h, [](sogk_scene* x) { sogk_scene_destroy(x); });
    }
    sogk_scene* handle() const { return h_.get(); }

private:
    std::shared_ptr<sogk_scene> h_;
};

/// render_frame (bench.hpp:424-461) on the GPU: every pixel sampled and composited
/// (composite_detailed, render.hpp:97-118) in two kernels, the image and the FrameResult
/// counters back on the host.  Pixels agree with the reference within one 8-bit level
/// (CUDA exp vs glibc exp); the counters are exact.
struct GpuFrame {
    Image image;
    long lookups = 0, steps = 0, samples = 0;
};
inline GpuFrame render_frame(const Sampler& s, const DeviceScene& scene, const Camera& cam,
                             void* stream = nullptr) {
    sogk_camera c{};
    const double pos[3] = {cam.position.x, cam.position.y, cam.position.z};
    const double tgt[3] = {cam.target.x, cam.target.y, cam.target.z};
    const double up[3] = {cam.up.x, cam.up.y, cam.up.z};
    check(sogk_camera_setup(pos, tgt, up, cam.vfov_deg, cam.width, cam.height, cam.t_far, &c));
    const std::int64_t n = std::int64_t(cam.width) * cam.height;
    std::vector<std::uint8_t> rgb(std::size_t(n) * 3);
    std::int64_t stats[SOGK_STATS_LEN] = {};
    check(sogk_render_frame_host(s.handle(), scene.handle(), &c, rgb.data(), stats, stream));
    GpuFrame f;
    f.image = Image(cam.width, cam.height);
    for (int y = 0; y < cam.height; ++y)
        for (int x = 0; x < cam.width; ++x) {
            const std::size_t i = (std::size_t(y) * cam.width + x) * 3;
            // Image::set_pixel of the 8-bit value reproduces the byte exactly
            f.image.set_pixel(x, y, Vec3{rgb[i] / 255.0, rgb[i + 1] / 255.0, rgb[i + 2] / 255.0});
        }
    f.lookups = long(stats[SOGK_STAT_ANALYZER_LOOKUPS] + stats[SOGK_STAT_KERNEL_LOOKUPS]);
    f.steps = long(stats[SOGK_STAT_ANALYZER_STEPS]);
    f.samples = long(stats[SOGK_STAT_TOTAL_SAMPLES]);
    return f;
}

} // namespace sog::gpu
