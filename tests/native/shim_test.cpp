// Drop-in check of include/sogk_sog.hpp: the unmodified reference library
// (sog::run_sampler, sog::build_sparse + serialize_sparse) against sog::gpu on
// the same inputs.  Built by oracle/Makefile into oracle/_ref/shim_test (it
// compiles the reference headers, so it is test infrastructure); run by
// tests/test_gpu_shim.py on the GPU box.  Exit 0 = bit-exact everywhere.
#include <cstdio>
#include <sstream>
#include <vector>

#include "sog/sog.hpp"
#include "sogk_sog.hpp"

using namespace sog;

static int failures = 0;
#define EXPECT(c, ...)                           \
    do {                                         \
        if (!(c)) {                              \
            ++failures;                          \
            std::printf("FAIL: " __VA_ARGS__);   \
            std::printf("\n");                   \
        }                                        \
    } while (0)

int main() {
    const GridTransform t = GridTransform::cube(64, {-1, -1, -1}, 2.0);
    SceneParams p;
    p.seed = 1;
    const GeneratedScene gen = generate_scene(SceneKind::shell, t, p);
    const DenseGrid& dense = gen.grid;
    const SparseGrid sparse = build_sparse(dense);

    // GPU build == reference build, byte for byte (io.hpp:161-181)
    gpu::DeviceDenseGrid ddense(dense);
    gpu::DeviceSparseGrid dvdb = gpu::build_sparse(ddense);
    EXPECT(dvdb.serialize() == serialize_sparse(sparse), "SOG1 bytes differ");
    EXPECT(dvdb.memory_bytes() == memory_bytes(sparse), "memory_bytes differ");
    EXPECT(dvdb.leaf_count() == sparse.leaf_count(), "leaf_count differs");
    EXPECT(dvdb.to_host().structurally_equal(sparse), "round trip differs");

    Camera cam;
    cam.position = {1.9, 1.4, 2.3};
    cam.vfov_deg = 42.0;
    cam.width = 80;
    cam.height = 60;
    std::vector<Ray> rays;
    for (int y = 0; y < cam.height; ++y)
        for (int x = 0; x < cam.width; ++x) rays.push_back(cam.pixel_ray(x, y));

    const StepSchedule scheds[] = {StepSchedule::constant(0.5 * t.voxel_size),
                                   StepSchedule::linear(0.011, 1.0 / 128.0)};
    for (const auto& sched : scheds)
        for (KernelKind k : {KernelKind::branch, KernelKind::skip}) {
            const gpu::Sampler sd(ddense, k, sched), sh(dvdb, k, sched);
            const gpu::PackedSamples od = sd.sample_rays(rays), oh = sh.sample_rays(rays);
            long mism = 0;
            for (std::size_t r = 0; r < rays.size(); ++r) {
                const SampleRun rd = run_sampler(rays[r], dense, k, sched);
                const SampleRun rh = run_sampler(rays[r], sparse, k, sched);
                const SampleRun gd = od.run(r), gh = oh.run(r);
                mism += gd.samples != rd.samples || gd.analyzer_lookups != rd.analyzer_lookups ||
                        gd.analyzer_steps != rd.analyzer_steps || gd.kernel_lookups != rd.kernel_lookups;
                mism += gh.samples != rh.samples || gh.analyzer_lookups != rh.analyzer_lookups ||
                        gh.analyzer_steps != rh.analyzer_steps || gh.kernel_lookups != rh.kernel_lookups;
            }
            EXPECT(mism == 0, "%ld ray mismatches (kernel %d)", mism, int(k));
        }
    // rank shards (multi-GPU row split): concatenated shards == the whole batch, global ray_indices
    {
        const gpu::Sampler sh(dvdb, KernelKind::skip, scheds[1]);
        const gpu::PackedSamples whole = sh.sample_rays(rays);
        for (int world : {1, 3, 7}) {
            long sm = 0;
            std::int64_t covered = 0;
            for (int rank = 0; rank < world; ++rank) {
                const gpu::ShardRange sr = gpu::shard_range(std::int64_t(rays.size()), world, rank);
                const gpu::PackedSamples part = sh.sample_shard(rays, world, rank);
                sm += std::int64_t(part.size()) != sr.count;
                for (std::int64_t r = 0; r < sr.count && sm == 0; ++r) {
                    const std::size_t g = std::size_t(sr.first + r);
                    sm += part.run(std::size_t(r)).samples != whole.run(g).samples;
                    const auto off = part.packed_info[2 * r], cnt = part.packed_info[2 * r + 1];
                    for (std::int64_t k = 0; k < cnt; ++k)
                        sm += part.ray_indices[std::size_t(off + k)] != std::int32_t(g);
                }
                covered += sr.count;
            }
            EXPECT(sm == 0 && covered == std::int64_t(rays.size()), "world %d: shards differ from the batch",
                   world);
        }
    }
    // single-ray drop-in
    const gpu::Sampler one(dvdb, KernelKind::skip, scheds[0]);
    EXPECT(one(rays[1234]).samples == run_sampler(rays[1234], sparse, KernelKind::skip, scheds[0]).samples,
           "single-ray run_sampler differs");
    // cascade (run_cascade_sampler, sampling.hpp:440-455)
    const DenseCascade dc = build_dense_cascade(gen.scene, t, 3, p.threshold);
    const SparseCascade sc = build_sparse_cascade(dc);
    std::vector<gpu::DeviceSparseGrid> gl;
    for (const auto& l : dc.levels) gl.push_back(gpu::build_sparse(l));
    const StepSchedule lin = StepSchedule::linear(0.5 * t.voxel_size, 1.0 / 256.0);
    const gpu::PackedSamples oc = gpu::Sampler(gl, KernelKind::skip, lin).sample_rays(rays);
    long cm = 0;
    for (std::size_t r = 0; r < rays.size(); ++r)
        cm += oc.samples(r) != run_cascade_sampler(rays[r], sc, KernelKind::skip, lin).samples;
    EXPECT(cm == 0, "%ld cascade ray mismatches", cm);
    // CD analyzer (run_sampler(ray, dense, dist, ...), sampling.hpp:198-212) and build_distance
    const DistanceGrid dist = build_distance(dense);
    const gpu::DeviceDistanceGrid ddist = gpu::build_distance(ddense);
    {
        const DistanceGrid back = ddist.to_host();
        long dm = 0;
        for (int z = 0; z < 64; ++z)
            for (int y = 0; y < 64; ++y)
                for (int x = 0; x < 64; ++x) dm += back.at({x, y, z}) != dist.at({x, y, z});
        EXPECT(dm == 0 && back.all_empty() == dist.all_empty(), "%ld distance values differ", dm);
        for (KernelKind k : {KernelKind::branch, KernelKind::skip}) {
            const gpu::PackedSamples o = gpu::Sampler(ddist, k, scheds[0]).sample_rays(rays);
            long m = 0;
            for (std::size_t r = 0; r < rays.size(); ++r) {
                const SampleRun a = run_sampler(rays[r], dense, dist, k, scheds[0]);
                const SampleRun b = o.run(r);
                m += a.samples != b.samples || a.analyzer_lookups != b.analyzer_lookups ||
                     a.analyzer_steps != b.analyzer_steps || a.kernel_lookups != b.kernel_lookups;
            }
            EXPECT(m == 0, "%ld CD ray mismatches (kernel %d)", m, int(k));
        }
    }
    // render_frame (bench.hpp:424-461): the reference's image vs the GPU frame
    {
        BenchAssets assets;
        assets.scene = gen.scene;
        assets.dense.levels.push_back(dense);
        assets.camera = cam;
        assets.schedule = scheds[0];
        const FrameResult ref = render_frame(assets, [&](const Ray& r) {
            return run_sampler(r, sparse, KernelKind::skip, scheds[0]);
        }, 1);
        const gpu::GpuFrame g = gpu::render_frame(gpu::Sampler(dvdb, KernelKind::skip, scheds[0]),
                                                  gpu::DeviceScene(gen.scene), cam);
        EXPECT(psnr(g.image, ref.image) >= 40.0, "render PSNR %.1f dB", psnr(g.image, ref.image));
        EXPECT(g.lookups == ref.lookups && g.steps == ref.steps && g.samples == ref.samples,
               "frame counters differ");
    }
    // traverse: collect_events + dump_trace (traversal.hpp:339-357) for every analyzer, and
    // SparseGrid::query
    {
        auto dump = [](const std::vector<TraversalEvent>& ev) {
            std::ostringstream os;
            dump_trace(os, ev);
            return os.str();
        };
        const gpu::EventStreams ed = gpu::Traverser(ddense).traverse_rays(rays);
        const gpu::EventStreams eh = gpu::Traverser(dvdb).traverse_rays(rays);
        const gpu::EventStreams ec = gpu::Traverser(ddist).traverse_rays(rays);
        long tm = 0;
        for (std::size_t r = 0; r < rays.size(); ++r) {
            DdaTraversal a(dense, rays[r]);
            HddaTraversal b(sparse, rays[r]);
            CdTraversal c(dist, rays[r]);
            const auto ea = collect_events(a), eb = collect_events(b), ecd = collect_events(c);
            tm += dump(ed.ray_events(r)) != dump(ea) || ed.lookup_count(r) != a.lookup_count() ||
                  ed.step_count(r) != a.step_count();
            tm += dump(eh.ray_events(r)) != dump(eb) || eh.lookup_count(r) != b.lookup_count() ||
                  eh.step_count(r) != b.step_count();
            tm += dump(ec.ray_events(r)) != dump(ecd) || ec.lookup_count(r) != c.lookup_count() ||
                  ec.step_count(r) != c.step_count();
        }
        EXPECT(tm == 0, "%ld event-stream (dump_trace) mismatches", tm);
        const gpu::EventStreams es = gpu::Traverser(gl).traverse_rays(rays);
        long cmx = 0;
        for (std::size_t r = 0; r < rays.size(); ++r) {
            CascadeTraversal<SparseGrid> ct(sc, rays[r]);
            std::vector<CascadeEvent> ref; // collect_events slices to TraversalEvent: drain by hand
            while (auto ev = ct.next()) ref.push_back(*ev);
            const auto got = es.ray_cascade_events(r);
            bool same = ref.size() == got.size();
            for (std::size_t k = 0; same && k < ref.size(); ++k)
                same = ref[k].ijk == got[k].ijk && ref[k].level == got[k].level && ref[k].t0 == got[k].t0 &&
                       ref[k].t1 == got[k].t1 && ref[k].occupied == got[k].occupied &&
                       ref[k].grid_level == got[k].grid_level;
            cmx += !same || es.lookup_count(r) != ct.lookup_count() || es.step_count(r) != ct.step_count();
        }
        EXPECT(cmx == 0, "%ld cascade event-stream mismatches", cmx);
        EXPECT(dump(gpu::Traverser(ddense).collect_events(rays[777])) ==
                   dump(collect_events(DdaTraversal(dense, rays[777]))), "single-ray collect_events");
        long qm = 0;
        for (int z = -70; z < 140; z += 7)
            for (int y = -9; y < 80; y += 5)
                for (int x = -130; x < 200; x += 11) {
                    const QueryResult a = sparse.query({x, y, z});
                    const QueryResult b = gpu::query(dvdb, {x, y, z});
                    qm += a.occupied != b.occupied || a.level != b.level || !(a.origin == b.origin) ||
                          a.extent != b.extent;
                }
        EXPECT(qm == 0, "%ld query mismatches", qm);
    }
    // errors like the reference
    bool threw = false;
    try {
        gpu::Sampler bad(dvdb, KernelKind::skip, StepSchedule{StepSchedule::Kind::constant, -1.0, 0.0});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "negative step did not throw std::invalid_argument");
    std::printf("%s: %zu rays x 4 variants x 2 schedules + cascade + CD + render + traverse/query, %d failures\n",
                failures ? "FAILED" : "OK", rays.size(), failures);
    return failures ? 1 : 0;
}
