// ref_shim.cpp — C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  This file contains no reference code: it
// #includes /root/reference/proj/include/sog/*.hpp (read-only, never copied)
// and /root/reference/proj/tests/support/test_support.hpp, and exposes them
// through extern "C" so that
//   * tests/golden/make_golden.py can produce golden vectors from the real
//     reference (pinning oracle/sog_oracle.c), and
//   * bench.py --impl reference / cpu_baseline can time the reference's own
//     per-ray sampler (sampling.hpp:166-196, 440-455) on all host cores,
//     split over contiguous ray ranges like render_frame (bench.hpp:424-461)
//     without compositing.
// Built by oracle/Makefile into oracle/_ref/libsogref.so with the reference's
// own flags (-O2 -std=c++20, no -march) plus -ffp-contract=off.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "sog/bench.hpp"  // make_probe_rays (bench.hpp:628-649); needs nlohmann/json.hpp
#include "sog/camera.hpp"
#include "sog/io.hpp"
#include "sog/sampling.hpp"
#include "sog/scene_gen.hpp"
#include "sog/sparse.hpp"
#include "test_support.hpp"

using namespace sog;

namespace {

struct RefSampler {
    DenseCascade dense;
    SparseCascade sparse;
    DistanceCascade distance;
    int cascade = 0;
    int analyzer = 0; // 0 dda, 1 hdda, 2 cd
    KernelKind kernel = KernelKind::skip;
    StepSchedule sched;
};

// Forwarding analyzer that records every event it returns.  sample_skip /
// sample_branch are templates over Analyzer& (sampling.hpp:87-88,105-106),
// so this wrapper runs the unmodified kernels.
template <class A>
struct Recording {
    A inner;
    std::vector<TraversalEvent> events;
    std::vector<int> grid_levels;
    template <class... Args>
    explicit Recording(Args&&... args) : inner(std::forward<Args>(args)...) {}
    bool valid() const { return inner.valid(); }
    double t_enter() const { return inner.t_enter(); }
    double t_exit() const { return inner.t_exit(); }
    long lookup_count() const { return inner.lookup_count(); }
    long step_count() const { return inner.step_count(); }
    auto next() {
        auto ev = inner.next();
        if (ev) {
            events.push_back(static_cast<const TraversalEvent&>(*ev));
            if constexpr (requires { ev->grid_level; })
                grid_levels.push_back(ev->grid_level);
            else
                grid_levels.push_back(0);
        }
        return ev;
    }
};

struct RayOut {
    std::vector<double> t;
    std::vector<double> t_end;
    std::vector<uint32_t> cell;
    std::vector<uint8_t> level;
    long lookups = 0, steps = 0, kernel_lookups = 0;
};

Ray load_ray(const double* p) {
    return Ray({p[0], p[1], p[2]}, {p[3], p[4], p[5]}, p[6], p[7]);
}

template <class An, class ProbeFactory>
void run_recorded(An& an, const RefSampler& s, ProbeFactory make_probe, RayOut& out) {
    SampleBuffer buf;
    if (s.kernel == KernelKind::branch) {
        auto probe = make_probe();
        buf = sample_branch(an, probe, s.sched);
        out.kernel_lookups = probe.lookups;
    } else {
        buf = sample_skip(an, s.sched);
    }
    out.lookups = an.lookup_count();
    out.steps = an.step_count();
    // attribute each sample to the unique recorded event with t0 < t <= t1
    std::size_t j = 0;
    for (double t : buf) {
        while (j < an.events.size() && an.events[j].t1 < t) ++j;
        const TraversalEvent& ev = an.events[j];
        out.t.push_back(t);
        out.t_end.push_back(t + s.sched.step(t)); // the next t_last (sampling.hpp:99,118)
        out.cell.push_back(uint32_t(ev.ijk.x & 1023) | (uint32_t(ev.ijk.y & 1023) << 10) |
                           (uint32_t(ev.ijk.z & 1023) << 20));
        out.level.push_back(uint8_t(int(ev.level) | (an.grid_levels[j] << 2)));
    }
}

void sample_one(const RefSampler& s, const Ray& ray, RayOut& out) {
    const bool cascade = s.cascade || s.dense.levels.size() > 1;
    if (!cascade) {
        if (s.analyzer == 0) {
            Recording<DdaTraversal> an(s.dense.levels[0], ray);
            run_recorded(an, s, [&] { return DenseProbe{&s.dense.levels[0]}; }, out);
        } else if (s.analyzer == 2) { // run_sampler(ray, dense, dist, ...) (sampling.hpp:198-212)
            Recording<CdTraversal> an(s.distance.levels[0], ray);
            run_recorded(an, s, [&] { return DenseProbe{&s.dense.levels[0]}; }, out);
        } else {
            Recording<HddaTraversal> an(s.sparse.levels[0], ray);
            run_recorded(an, s, [&] { return SparseProbe(s.sparse.levels[0]); }, out);
        }
    } else {
        if (s.analyzer == 0) {
            Recording<CascadeTraversal<DenseGrid>> an(s.dense, ray);
            run_recorded(an, s, [&] { return CascadeProbe<DenseGrid>(s.dense); }, out);
        } else if (s.analyzer == 2) {
            Recording<CascadeTraversal<DistanceGrid>> an(s.distance, ray);
            run_recorded(an, s, [&] { return CascadeProbe<DistanceGrid>(s.distance); }, out);
        } else {
            Recording<CascadeTraversal<SparseGrid>> an(s.sparse, ray);
            run_recorded(an, s, [&] { return CascadeProbe<SparseGrid>(s.sparse); }, out);
        }
    }
}

// The plain reference entry points, exactly what make_sampler dispatches to
// (bench.hpp:382-413): used for timing.
std::size_t sample_plain(const RefSampler& s, const Ray& ray) {
    const bool cascade = s.cascade || s.dense.levels.size() > 1;
    if (!cascade) {
        if (s.analyzer == 0) return run_sampler(ray, s.dense.levels[0], s.kernel, s.sched).samples.size();
        if (s.analyzer == 2)
            return run_sampler(ray, s.dense.levels[0], s.distance.levels[0], s.kernel, s.sched).samples.size();
        return run_sampler(ray, s.sparse.levels[0], s.kernel, s.sched).samples.size();
    }
    if (s.analyzer == 0) return run_cascade_sampler(ray, s.dense, s.kernel, s.sched).samples.size();
    if (s.analyzer == 2) return run_cascade_sampler(ray, s.distance, s.kernel, s.sched).samples.size();
    return run_cascade_sampler(ray, s.sparse, s.kernel, s.sched).samples.size();
}

template <class Fn>
void parallel_ranges(int64_t n, int threads, Fn fn) {
    threads = std::max(1, threads);
    if (threads == 1 || n < 2) {
        fn(0, 0, n);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t per = (n + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
        const int64_t a = std::min<int64_t>(n, w * per), b = std::min<int64_t>(n, (w + 1) * per);
        pool.emplace_back(fn, w, a, b);
    }
    for (auto& th : pool) th.join();
}

GridTransform make_transform(const int32_t res[3], const double wmin[3], double voxel) {
    return GridTransform({res[0], res[1], res[2]}, {wmin[0], wmin[1], wmin[2]}, voxel);
}

void copy_bits(const DenseGrid& g, uint8_t* out) {
    std::memcpy(out, g.payload().data(), g.payload().size());
}

} // namespace

extern "C" {

int ref_hardware_concurrency() { return int(std::thread::hardware_concurrency()); }

// scene_gen.hpp:94-192; returns occupancy fraction
double ref_generate_scene(int kind, const int32_t res[3], const double wmin[3], double voxel,
                          uint64_t seed, double fraction, int count, double threshold,
                          uint8_t* out_bits) {
    SceneParams p;
    p.seed = seed;
    p.fraction = fraction;
    p.primitive_count = count;
    p.threshold = threshold;
    const GeneratedScene gen = generate_scene(SceneKind(kind), make_transform(res, wmin, voxel), p);
    copy_bits(gen.grid, out_bits);
    return gen.occupancy;
}

// build_dense_cascade (scene_gen.hpp:196-209); out_bits = levels consecutive payloads,
// out_wmin = levels*3, out_voxel = levels
void ref_dense_cascade(int kind, const int32_t res[3], const double wmin[3], double voxel,
                       uint64_t seed, double fraction, int count, double threshold, int levels,
                       uint8_t* out_bits, double* out_wmin, double* out_voxel) {
    SceneParams p;
    p.seed = seed;
    p.fraction = fraction;
    p.primitive_count = count;
    p.threshold = threshold;
    const GridTransform base = make_transform(res, wmin, voxel);
    const GeneratedScene gen = generate_scene(SceneKind(kind), base, p);
    const DenseCascade c = build_dense_cascade(gen.scene, base, levels, p.threshold);
    std::size_t off = 0;
    for (int b = 0; b < levels; ++b) {
        copy_bits(c.levels[b], out_bits + off);
        off += c.levels[b].payload().size();
        for (int a = 0; a < 3; ++a) out_wmin[3 * b + a] = c.levels[b].transform().world_min[a];
        out_voxel[b] = c.levels[b].transform().voxel_size;
    }
}

// Camera::pixel_ray (camera.hpp:167-179), row-major pixels
void ref_camera_rays(const double pos[3], const double target[3], const double up[3],
                     double vfov_deg, int width, int height, double t_far, double* out) {
    Camera cam;
    cam.position = {pos[0], pos[1], pos[2]};
    cam.target = {target[0], target[1], target[2]};
    cam.up = {up[0], up[1], up[2]};
    cam.vfov_deg = vfov_deg;
    cam.width = width;
    cam.height = height;
    cam.t_far = t_far;
    int64_t i = 0;
    for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x, ++i) {
            const Ray r = cam.pixel_ray(x, y);
            double* o = out + 8 * i;
            o[0] = r.origin.x; o[1] = r.origin.y; o[2] = r.origin.z;
            o[3] = r.direction.x; o[4] = r.direction.y; o[5] = r.direction.z;
            o[6] = r.t_min; o[7] = r.t_max;
        }
}

static void store_ray(const Ray& r, double* o) {
    o[0] = r.origin.x; o[1] = r.origin.y; o[2] = r.origin.z;
    o[3] = r.direction.x; o[4] = r.direction.y; o[5] = r.direction.z;
    o[6] = r.t_min; o[7] = r.t_max;
}

// make_probe_rays (bench.hpp:628-649) over GridTransform(res, wmin, voxel)
void ref_probe_rays(const int32_t res[3], const double wmin[3], double voxel, int count,
                    uint64_t seed, double* out) {
    const std::vector<Ray> rays = make_probe_rays(make_transform(res, wmin, voxel), count, seed);
    for (int i = 0; i < count; ++i) store_ray(rays[i], out + 8 * i);
}

// testsupport::random_ray (test_support.hpp:66-82), n rays from one mt19937_64(seed)
void ref_random_rays(const int32_t res[3], const double wmin[3], double voxel, int count,
                     uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    const GridTransform t = make_transform(res, wmin, voxel);
    for (int i = 0; i < count; ++i) store_ray(testsupport::random_ray(rng, t), out + 8 * i);
}

// testsupport::random_grid / random_blocky_grid (test_support.hpp:29-62)
void ref_random_grid(const int32_t res[3], const double wmin[3], double voxel, uint64_t seed,
                     double fraction, uint8_t* out_bits) {
    std::mt19937_64 rng(seed);
    copy_bits(testsupport::random_grid(rng, make_transform(res, wmin, voxel), fraction), out_bits);
}
void ref_random_blocky_grid(const int32_t res[3], const double wmin[3], double voxel,
                            uint64_t seed, double block_fraction, double noise_fraction,
                            uint8_t* out_bits) {
    std::mt19937_64 rng(seed);
    copy_bits(testsupport::random_blocky_grid(rng, make_transform(res, wmin, voxel), block_fraction,
                                              noise_fraction),
              out_bits);
}

// serialize_sparse(build_sparse(dense)) (io.hpp:161-181, sparse.hpp:333-371);
// returns the byte size (writes only when it fits)
int64_t ref_build_sog1(const int32_t res[3], const double wmin[3], double voxel,
                       const uint8_t* bits, uint8_t* out, int64_t cap) {
    DenseGrid d(make_transform(res, wmin, voxel));
    std::memcpy(d.payload().data(), bits, d.payload().size());
    const std::vector<uint8_t> bytes = serialize_sparse(build_sparse(d));
    if (out && int64_t(bytes.size()) <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return int64_t(bytes.size());
}

// median build_sparse time over reps (bench.hpp:349-356 convention), ms
double ref_build_sparse_ms(const int32_t res[3], const double wmin[3], double voxel,
                           const uint8_t* bits, int reps) {
    DenseGrid d(make_transform(res, wmin, voxel));
    std::memcpy(d.payload().data(), bits, d.payload().size());
    std::vector<double> ms;
    for (int i = 0; i < reps; ++i) {
        const auto a = std::chrono::steady_clock::now();
        SparseGrid s = build_sparse(d);
        const auto b = std::chrono::steady_clock::now();
        ms.push_back(std::chrono::duration<double, std::milli>(b - a).count());
    }
    std::sort(ms.begin(), ms.end());
    return ms[ms.size() / 2];
}

void* ref_sampler_create(int n_levels, int cascade, const int32_t res[3], const double* wmin,
                         const double* voxel, const uint8_t* const* bits, int analyzer,
                         int kernel, int sched_kind, double dt0, double growth) {
    auto* s = new RefSampler;
    for (int b = 0; b < n_levels; ++b) {
        DenseGrid d(make_transform(res, wmin + 3 * b, voxel[b]));
        std::memcpy(d.payload().data(), bits[b], d.payload().size());
        s->dense.levels.push_back(std::move(d));
    }
    if (analyzer == 1)
        for (const auto& d : s->dense.levels) s->sparse.levels.push_back(build_sparse(d));
    if (analyzer == 2)
        for (const auto& d : s->dense.levels) s->distance.levels.push_back(build_distance(d));
    s->cascade = cascade;
    s->analyzer = analyzer;
    s->kernel = kernel == 0 ? KernelKind::branch : KernelKind::skip;
    s->sched = sched_kind == 0 ? StepSchedule::constant(dt0) : StepSchedule::linear(dt0, growth);
    return s;
}

void ref_sampler_free(void* h) { delete static_cast<RefSampler*>(h); }

// Packed outputs for rays not masked by skip (skip[i] != 0 -> status 2, no samples:
// the reference never returns on those rays).  Returns total
// samples; outputs beyond cap are not written.
int64_t ref_sample_batch(void* h, const double* rays, int64_t n, const uint8_t* skip,
                         int threads, int64_t cap, int64_t* packed_info, double* t_starts,
                         double* t_ends, uint32_t* cells, uint8_t* levels, int32_t* counters) {
    const RefSampler& s = *static_cast<RefSampler*>(h);
    std::vector<RayOut> outs(n);
    parallel_ranges(n, threads, [&](int, int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i)
            if (!(skip && skip[i])) sample_one(s, load_ray(rays + 8 * i), outs[i]);
    });
    int64_t off = 0;
    for (int64_t i = 0; i < n; ++i) {
        const RayOut& o = outs[i];
        const int64_t c = int64_t(o.t.size());
        packed_info[2 * i] = off;
        packed_info[2 * i + 1] = c;
        for (int64_t k = 0; k < c && off + k < cap; ++k) {
            t_starts[off + k] = o.t[k];
            t_ends[off + k] = o.t_end[k];
            cells[off + k] = o.cell[k];
            levels[off + k] = o.level[k];
        }
        counters[3 * i] = int32_t(o.lookups);
        counters[3 * i + 1] = int32_t(o.steps);
        counters[3 * i + 2] = int32_t(o.kernel_lookups);
        off += c;
    }
    return off;
}

// Events of one ray through the reference analyzer (collect_events, traversal.hpp:340-345).
// ev_out rows: ijk[3], level, occupied, grid_level (int32) ; t_out rows: t0, t1.
int64_t ref_collect_events(void* h, const double* ray, int64_t cap, int32_t* ev_out,
                           double* t_out, int64_t* counters) {
    const RefSampler& s = *static_cast<RefSampler*>(h);
    const Ray r = load_ray(ray);
    const bool cascade = s.cascade || s.dense.levels.size() > 1;
    int64_t n = 0;
    auto drain = [&](auto& an) {
        while (auto ev = an.next()) {
            if (n < cap) {
                ev_out[6 * n] = ev->ijk.x;
                ev_out[6 * n + 1] = ev->ijk.y;
                ev_out[6 * n + 2] = ev->ijk.z;
                ev_out[6 * n + 3] = int32_t(ev->level);
                ev_out[6 * n + 4] = ev->occupied ? 1 : 0;
                if constexpr (requires { ev->grid_level; })
                    ev_out[6 * n + 5] = ev->grid_level;
                else
                    ev_out[6 * n + 5] = 0;
                t_out[2 * n] = ev->t0;
                t_out[2 * n + 1] = ev->t1;
            }
            ++n;
        }
        counters[0] = an.lookup_count();
        counters[1] = an.step_count();
    };
    if (!cascade) {
        if (s.analyzer == 0) {
            DdaTraversal an(s.dense.levels[0], r);
            drain(an);
        } else if (s.analyzer == 2) {
            CdTraversal an(s.distance.levels[0], r);
            drain(an);
        } else {
            HddaTraversal an(s.sparse.levels[0], r);
            drain(an);
        }
    } else if (s.analyzer == 0) {
        CascadeTraversal<DenseGrid> an(s.dense, r);
        drain(an);
    } else if (s.analyzer == 2) {
        CascadeTraversal<DistanceGrid> an(s.distance, r);
        drain(an);
    } else {
        CascadeTraversal<SparseGrid> an(s.sparse, r);
        drain(an);
    }
    return n;
}

// CPU baseline: the reference's per-ray sampler over rays [0, n) split across
// `threads` contiguous ranges (render_frame, bench.hpp:446-454, minus compositing).
// Returns the median wall time in seconds over reps; *samples = samples per rep.
double ref_time_sampler(void* h, const double* rays, int64_t n, const uint8_t* skip,
                        int threads, int reps, int64_t* samples) {
    const RefSampler& s = *static_cast<RefSampler*>(h);
    std::vector<Ray> rr;
    rr.reserve(n);
    for (int64_t i = 0; i < n; ++i) rr.push_back(load_ray(rays + 8 * i));
    std::vector<double> secs;
    for (int rep = 0; rep < reps; ++rep) {
        std::vector<int64_t> per(std::max(1, threads), 0);
        const auto a = std::chrono::steady_clock::now();
        parallel_ranges(n, threads, [&](int w, int64_t lo, int64_t hi) {
            int64_t c = 0;
            for (int64_t i = lo; i < hi; ++i)
                if (!(skip && skip[i])) c += int64_t(sample_plain(s, rr[i]));
            per[w] = c;
        });
        const auto b = std::chrono::steady_clock::now();
        secs.push_back(std::chrono::duration<double>(b - a).count());
        int64_t tot = 0;
        for (auto c : per) tot += c;
        *samples = tot;
    }
    std::sort(secs.begin(), secs.end());
    return secs[secs.size() / 2];
}

// generate_scene's AnalyticScene (scene_gen.hpp:94-176): 16 doubles per primitive =
// shape, center[3], radius, lo[3], hi[3], density, color[3], 0; returns the count
int ref_scene_primitives(int kind, const int32_t res[3], const double wmin[3], double voxel,
                         uint64_t seed, double fraction, int count, double* out, int cap,
                         double* background) {
    SceneParams p;
    p.seed = seed;
    p.fraction = fraction;
    p.primitive_count = count;
    const GeneratedScene gen = generate_scene(SceneKind(kind), make_transform(res, wmin, voxel), p);
    const auto& prims = gen.scene.primitives;
    for (int a = 0; a < 3; ++a) background[a] = gen.scene.background[a];
    for (int i = 0; i < int(prims.size()) && i < cap; ++i) {
        const Primitive& q = prims[i];
        double* o = out + 16 * i;
        o[0] = q.shape == Primitive::Shape::sphere ? 0.0 : 1.0;
        for (int a = 0; a < 3; ++a) {
            o[1 + a] = q.center[a];
            o[5 + a] = q.lo[a];
            o[8 + a] = q.hi[a];
            o[12 + a] = q.color[a];
        }
        o[4] = q.radius;
        o[11] = q.density;
        o[15] = 0.0;
    }
    return int(prims.size());
}

// render_frame (bench.hpp:424-461) of one bench variant on build_assets(cfg)
// (bench.hpp:306-376): rgb = width*height*3 bytes; stats = lookups, steps, samples
void ref_render_frame(int kind, uint64_t seed, double fraction, int resolution, int cascades,
                      int sched_kind, int width, int height, int grid, int analyzer, int kernel,
                      int threads, uint8_t* rgb, int64_t* stats) {
    BenchConfig cfg;
    cfg.kind = SceneKind(kind);
    cfg.params.seed = seed;
    if (fraction > 0.0) cfg.params.fraction = fraction;
    cfg.resolution = resolution;
    cfg.cascades = cascades;
    cfg.schedule_kind = sched_kind == 0 ? StepSchedule::Kind::constant : StepSchedule::Kind::linear;
    cfg.width = width;
    cfg.height = height;
    const BenchAssets assets = build_assets(cfg);
    const VariantId v{grid == 0 ? GridKind::dense : GridKind::sparse,
                      analyzer == 0 ? AnalyzerKind::dda : AnalyzerKind::hdda,
                      kernel == 0 ? KernelKind::branch : KernelKind::skip};
    const FrameResult f = render_frame(assets, make_sampler(assets, v), threads);
    std::memcpy(rgb, f.image.data().data(), f.image.data().size());
    stats[0] = f.lookups;
    stats[1] = f.steps;
    stats[2] = f.samples;
}

// composite_detailed (render.hpp:97-118) through the reference: prims as 16 doubles each
// (ref_scene_primitives layout); out = color rgb, weight_sum, transmittance
void ref_composite(const double* ray, const double* samples, int64_t n, const double* prims,
                   int n_prims, const double* background, int sched_kind, double dt0,
                   double growth, double* out) {
    AnalyticScene scene;
    scene.background = {background[0], background[1], background[2]};
    for (int i = 0; i < n_prims; ++i) {
        const double* q = prims + 16 * i;
        const Vec3 color{q[12], q[13], q[14]};
        if (q[0] == 0.0)
            scene.primitives.push_back(Primitive::sphere({q[1], q[2], q[3]}, q[4], q[11], color));
        else
            scene.primitives.push_back(
                Primitive::box({q[5], q[6], q[7]}, {q[8], q[9], q[10]}, q[11], color));
    }
    const Ray r({ray[0], ray[1], ray[2]}, {ray[3], ray[4], ray[5]}, ray[6], ray[7]);
    const SampleBuffer buf(samples, samples + n);
    const StepSchedule sched =
        sched_kind == 0 ? StepSchedule::constant(dt0) : StepSchedule::linear(dt0, growth);
    const CompositeResult c = composite_detailed(r, buf, scene, sched);
    out[0] = c.color.x;
    out[1] = c.color.y;
    out[2] = c.color.z;
    out[3] = c.weight_sum;
    out[4] = c.transmittance;
}

// build_distance (distance.hpp:45-103): int32 per voxel; returns all_empty()
int ref_build_distance(const int32_t res[3], const double wmin[3], double voxel, const uint8_t* bits,
                       int32_t* out) {
    DenseGrid d(make_transform(res, wmin, voxel));
    std::memcpy(d.payload().data(), bits, d.payload().size());
    const DistanceGrid g = build_distance(d);
    const Vec3i r = g.transform().resolution;
    int64_t i = 0;
    for (int z = 0; z < r.z; ++z)
        for (int y = 0; y < r.y; ++y)
            for (int x = 0; x < r.x; ++x) out[i++] = g.at({x, y, z});
    return g.all_empty() ? 1 : 0;
}

// run_matrix (bench.hpp:514-553) + emit_csv / emit_json (bench.hpp:563-605) of the reference
// on a small config; returns the bytes needed (json then csv, NUL-separated) or -1 if cap is short
int64_t ref_run_matrix(int kind, uint64_t seed, double fraction, int resolution, int cascades,
                       int sched_kind, int width, int height, int repetitions, char* out,
                       int64_t cap) {
    BenchConfig cfg;
    cfg.kind = SceneKind(kind);
    cfg.params.seed = seed;
    if (fraction > 0.0) cfg.params.fraction = fraction;
    cfg.resolution = resolution;
    cfg.cascades = cascades;
    cfg.schedule_kind = sched_kind == 0 ? StepSchedule::Kind::constant : StepSchedule::Kind::linear;
    cfg.width = width;
    cfg.height = height;
    cfg.repetitions = repetitions;
    cfg.validate();
    const BenchReport rep = run_matrix(cfg);
    const std::string j = emit_json(rep), c = emit_csv(rep);
    const int64_t need = int64_t(j.size() + c.size() + 2);
    if (need > cap) return -need;
    std::memcpy(out, j.data(), j.size());
    out[j.size()] = 0;
    std::memcpy(out + j.size() + 1, c.data(), c.size());
    out[need - 1] = 0;
    return need;
}

} // extern "C"
