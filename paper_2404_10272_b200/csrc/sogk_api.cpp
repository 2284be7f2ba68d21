// sogk_api.cpp — the C-ABI (include/sogk.h): grid and sampler handles, SOG0/SOG1
// I/O, validation with the reference's error semantics, and the launchers.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <array>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sogk.h"
#include "sogk_internal.h"

using namespace sogk;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_err;

int fail(int status, const std::string& msg) {
    g_err = msg;
    return status;
}

// Rays are read as 16-byte pairs and packed_info / event_info are {offset, count} pairs read and
// written as one 16-byte access: a misaligned base would fault the kernel (a sticky context
// error), so the entry points refuse it up front.
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
const char* const kAlign16 = "device rays and packed_info / event_info must be 16-byte aligned";

int cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        return fail(SOGK_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
        return fail(SOGK_NO_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
    return fail(SOGK_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr, what)                                   \
    do {                                                 \
        cudaError_t _e = (expr);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

bool valid_transform(const sogk_transform* t) { // GridTransform ctor, grid.hpp:24-30
    return t && t->res[0] >= 1 && t->res[1] >= 1 && t->res[2] >= 1 && t->voxel_size > 0.0;
}
uint64_t voxel_count(const sogk_transform& t) { return uint64_t(t.res[0]) * t.res[1] * t.res[2]; }
uint64_t payload_bytes(const sogk_transform& t) { return (voxel_count(t) + 7) / 8; }

template <class T>
cudaError_t dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) return cudaSuccess;
    return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

// Grid storage comes from the device's stream-ordered pool, which keeps freed blocks
// (release threshold = max) so rebuilding a grid does not pay cudaMalloc / cudaFree page
// mapping -- the reference's conversion times are plain heap allocations.  The pool is
// trimmed by sogk_release_workspaces.
cudaError_t retain_pool() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && !done[dev]) {
        cudaMemPool_t pool;
        if ((e = cudaDeviceGetDefaultMemPool(&pool, dev)) != cudaSuccess) return e;
        uint64_t keep = UINT64_MAX;
        if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess)
            return e;
        done[dev] = true;
    }
    return cudaSuccess;
}

template <class T>
cudaError_t galloc(T** p, size_t count, cudaStream_t st) {
    *p = nullptr;
    if (count == 0) return cudaSuccess;
    cudaError_t e = retain_pool();
    if (e != cudaSuccess) return e;
    return cudaMallocAsync(reinterpret_cast<void**>(p), count * sizeof(T), st);
}

struct RootEntry { // one record of the reference root map (sparse.hpp:143-150)
    int32_t origin[3];
    uint8_t kind; // 0 empty tile, 1 occupied tile, 2 internal
    int32_t node; // region slot for internal entries
};

struct RegionOrder { // sparse.hpp:119-125
    bool operator()(const std::array<int32_t, 3>& a, const std::array<int32_t, 3>& b) const {
        if (a[2] != b[2]) return a[2] < b[2];
        if (a[1] != b[1]) return a[1] < b[1];
        return a[0] < b[0];
    }
};
} // namespace

struct sogk_grid {
    int kind = SOGK_GRID_DENSE;
    sogk_transform t{};
    int device = 0;
    // dense
    uint8_t* bits = nullptr;
    uint64_t nbytes = 0;
    // vdb
    int R[3] = {0, 0, 0};
    int64_t nreg = 0;
    int32_t* root = nullptr;
    uint64_t* child_mask = nullptr;
    uint64_t* value_mask = nullptr;
    uint32_t* prefix = nullptr;
    uint64_t* leaves = nullptr;
    int32_t* table = nullptr;
    uint32_t* region_leaves = nullptr;
    uint32_t* total_leaves = nullptr;
    uint64_t leaf_capacity = 0;
    // distance
    int32_t* dist = nullptr;
    unsigned* dist_any = nullptr; // device flag: some voxel occupied (!all_empty)
    // host-side root map when loaded from SOG1 (entries that do not map to an
    // in-grid aligned region are kept for export only); empty for built grids
    std::vector<RootEntry> extra_entries;
    bool from_file = false;
    // lazily materialized metadata
    mutable bool meta_ready = false;
    mutable std::vector<int32_t> h_root;
    mutable int64_t leaf_count = 0;

    // build completion on the build stream: host reads (metadata, downloads, exports) wait on it
    cudaEvent_t ready = nullptr;
    cudaError_t mark(cudaStream_t st) {
        cudaError_t e = ready ? cudaSuccess : cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
        return e == cudaSuccess ? cudaEventRecord(ready, st) : e;
    }
    cudaError_t wait_ready() const { return ready ? cudaEventSynchronize(ready) : cudaSuccess; }

    ~sogk_grid() { // pool blocks (galloc); like cudaFree, wait for work that may still read them
        void* ps[] = {bits, root, child_mask, value_mask, prefix, table, leaves, region_leaves,
                      total_leaves, dist, dist_any};
        bool any = false;
        for (void* p : ps) any |= p != nullptr;
        if (!any) return;
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != device) cudaSetDevice(device);
        cudaDeviceSynchronize();
        for (void* p : ps)
            if (p) cudaFreeAsync(p, 0);
        if (cur != device) cudaSetDevice(cur);
        if (ready) cudaEventDestroy(ready);
    }

    GridDev dev() const {
        GridDev g{};
        for (int a = 0; a < 3; ++a) {
            g.res[a] = t.res[a];
            g.wmin[a] = t.world_min[a];
            g.R[a] = R[a];
        }
        g.voxel = t.voxel_size;
        g.inv_voxel = 1.0 / t.voxel_size;
        {
            int e = 0;
            const double m = std::frexp(t.voxel_size, &e);
            // exact reciprocal and no subnormal products for grid-scale values
            g.voxel_pow2 = (m == 0.5 && e > -900 && e < 900) ? 1 : 0;
        }
        const double h = t.voxel_size * 0.5; // center_bounds, sampling.hpp:248-251
        for (int a = 0; a < 3; ++a) {
            g.clo[a] = t.world_min[a] + h;
            g.chi[a] = (t.world_min[a] + double(t.res[a]) * t.voxel_size) - h;
        }
        g.bits = bits;
        g.root = root;
        g.child_mask = child_mask;
        g.value_mask = value_mask;
        g.prefix = prefix;
        g.leaves = leaves;
        g.table = table;
        g.node0 = kNodeMulti;
        g.dist = dist;
        return g;
    }

    int fetch_meta() const {
        if (meta_ready) return SOGK_OK;
        if (kind != SOGK_GRID_VDB) {
            meta_ready = true;
            return SOGK_OK;
        }
        CK(wait_ready(), "build completion");
        h_root.resize(nreg);
        CK(cudaMemcpy(h_root.data(), root, nreg * sizeof(int32_t), cudaMemcpyDeviceToHost), "root D2H");
        uint32_t tl = 0;
        CK(cudaMemcpy(&tl, total_leaves, sizeof(uint32_t), cudaMemcpyDeviceToHost), "leaf count D2H");
        leaf_count = tl;
        meta_ready = true;
        return SOGK_OK;
    }
};

// Pass-1 -> pass-2 workspaces, one per (device, stream): work on one stream is ordered, so
// samplers can share it; a sampler's slabs stay valid until another count on that stream.
struct Workspace {
    void* ptr = nullptr;
    size_t bytes = 0;
    // the count whose slabs it holds: its token (sogk_sample_count_ex), the sampler id and the
    // rays / packed_info it ran on
    uint64_t token = 0;
    uint64_t owner = 0;
    const void* packed = nullptr;
    const void* rays = nullptr;
    int64_t first = -1, n = -1;
    bool cam = false;
    int64_t C = 0; // run records per ray the slabs are laid out with (set by the claiming count)
};
static std::atomic<uint64_t> g_sampler_ids{0};
static std::atomic<uint64_t> g_count_tokens{0};
// Pass-1 slab budget for a workspace that has to grow: SOGK_SLAB_BUDGET_GB, else 40 % of the
// device memory free at that moment (counting the workspace's own current block, which is
// released first) and at least 2 GiB.  Asked only when the full slab (C = SOGK_SLAB, 128) does
// not fit the workspace already held; a smaller slab only sends more rays to tail_kernel.
static double slab_budget_bytes(size_t held) {
    if (const char* e = std::getenv("SOGK_SLAB_BUDGET_GB")) return std::max(0.0, std::atof(e)) * double(1ull << 30);
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return 8.0 * double(1ull << 30);
    }
    return std::max(2.0 * double(1ull << 30), 0.4 * (double(fr) + double(held)));
}
static std::mutex g_ws_mu;
static std::map<std::pair<int, void*>, Workspace>& ws_registry() {
    static auto* m = new std::map<std::pair<int, void*>, Workspace>(); // never destroyed
    return *m;
}
static Workspace* workspace_peek(void* stream) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = ws_registry().find({dev, stream});
    return it == ws_registry().end() ? nullptr : &it->second;
}
// Render scratch, one per (device, stream) like the workspaces (work on a stream is ordered;
// the mutex covers host threads sharing a stream): [stats 256 B | packed n x 16 | rays n x 64]
// and, per sample, t 8 B | ray index 4 B | shaded 32 B.
struct RenderScratch {
    static constexpr double kSampleBytes = 44.0;
    std::mutex mu;
    void* rb = nullptr;
    int64_t rb_n = 0;
    void* sb = nullptr;
    int64_t smp_cap = 0;
    // smallest camera bound found not to fit a quarter of free memory: larger bounds skip the
    // cudaMemGetInfo query (a driver call per frame whose latency varies run to run)
    int64_t unfit_bound = INT64_MAX;
    int64_t* h_total = nullptr; // pinned
    static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
    int ensure_rays(int64_t n) {
        if (!h_total) CK(cudaMallocHost(&h_total, 64), "pinned total");
        if (n <= rb_n && rb) return SOGK_OK;
        cudaFree(rb); // synchronous: earlier frames that read it have finished
        rb = nullptr;
        rb_n = 0;
        const int64_t m = std::max<int64_t>(n, 1);
        CK(cudaMalloc(&rb, 256 + al(size_t(m) * 16) + size_t(m) * 64), "render scratch");
        rb_n = m;
        return SOGK_OK;
    }
    int ensure_samples(int64_t cap, void*) {
        if (cap <= smp_cap && sb) return SOGK_OK;
        cudaFree(sb);
        sb = nullptr;
        smp_cap = 0;
        const int64_t m = std::max<int64_t>(cap, 1);
        CK(cudaMalloc(&sb, al(size_t(m) * 8) + al(size_t(m) * 4) + size_t(m) * 32), "render sample scratch");
        smp_cap = m;
        return SOGK_OK;
    }
    int64_t* stats() const { return static_cast<int64_t*>(rb); }
    int64_t* packed() const { return reinterpret_cast<int64_t*>(static_cast<char*>(rb) + 256); }
    double* rays_buf() const {
        return reinterpret_cast<double*>(static_cast<char*>(rb) + 256 + al(size_t(rb_n) * 16));
    }
    double* ts() const { return static_cast<double*>(sb); }
    int32_t* ri() const { return reinterpret_cast<int32_t*>(static_cast<char*>(sb) + al(size_t(smp_cap) * 8)); }
    void* shaded() const {
        return static_cast<char*>(sb) + al(size_t(smp_cap) * 8) + al(size_t(smp_cap) * 4);
    }
    void release() {
        cudaFree(rb);
        cudaFree(sb);
        if (h_total) cudaFreeHost(h_total);
        rb = sb = nullptr;
        h_total = nullptr;
        rb_n = smp_cap = 0;
        unfit_bound = INT64_MAX;
    }
};
static std::map<std::pair<int, void*>, RenderScratch*>& render_registry() {
    static auto* m = new std::map<std::pair<int, void*>, RenderScratch*>(); // never destroyed
    return *m;
}
static RenderScratch* render_scratch_for(void* stream) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    RenderScratch*& r = render_registry()[{dev, stream}];
    if (!r) r = new RenderScratch;
    return r;
}

struct sogk_sampler {
    Variant v{};
    SamplerDev dev{};
    sogk_sampler_desc desc{};
    int n_levels = 0;
    // the grids (immutable, caller-owned): launches on a stream first wait for their builds
    const sogk_grid* lv[SOGK_MAX_LEVELS] = {};
    int max_res = 0;
    // serializes the calls that use per-sampler host state (sogk_sample_host, render): the
    // reference's render_frame calls one make_sampler function from many threads
    std::mutex host_mu;
    // sogk_sample_host scratch, pipeline streams and pinned per-chunk stats
    void* hb = nullptr;
    size_t hb_bytes = 0;
    bool lanes_ready = false;
    cudaStream_t lanes[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t lane_ev[3] = {nullptr, nullptr, nullptr};
    int64_t* h_chunk_stats = nullptr;
    std::vector<cudaEvent_t> done_ev; // per chunk: its downloads finished (host expansion waits)

    ~sogk_sampler() {
        for (cudaEvent_t e : done_ev) cudaEventDestroy(e);
        cudaFree(hb);
        if (lanes_ready) {
            for (int l = 0; l < 3; ++l) {
                cudaStreamDestroy(lanes[l]);
                cudaEventDestroy(lane_ev[l]);
            }
            cudaFreeHost(h_chunk_stats);
        }
    }

    // order `stream` after the builds of every level (grids built on another stream: their
    // pool storage and contents are valid in that stream's order only)
    int wait_levels(void* stream) const {
        for (int b = 0; b < n_levels; ++b)
            if (lv[b] && lv[b]->ready) CK(cudaStreamWaitEvent(S(stream), lv[b]->ready, 0), "grid build wait");
        return SOGK_OK;
    }

    // pass 1 -> pass 2 handshake: the run slabs of a count live in the workspace of the
    // (device, stream) it ran on, tagged with a token, the sampler and the rays; a write on that
    // stream that presents the token (or, through the token-less API, the same sampler, rays and
    // packed_info) uses them, anything else takes the exact cold path
    const uint64_t id = ++g_sampler_ids;
    int ray_order = 0; // 1: pass 1 processes buffer rays binned by entry cell and direction
    int64_t slab_cap = 128; // C: run records per ray (SOGK_SLAB; 0 = resume-only)

    int64_t cap_for(int64_t n, double budget) const {
        // keep the slabs within the budget; a smaller slab only sends more rays to
        // tail_kernel (exact either way)
        int64_t c = slab_cap;
        while (c > 0 && double(n) * double(c) * 16.0 > budget) c -= 4;
        return c < 0 ? 0 : c;
    }
    static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
    // workspace = [scan tile states | counters (64 B) | resume states | overflow list |
    //              run counts | run slabs (C per ray) | ray-binning scratch]
    size_t need_bytes(int64_t n, int64_t C) const {
        const size_t e = size_t(n) * size_t(C);
        return scan_off(n) + al(resume_bytes(n)) + 2 * al(size_t(n) * 4) + al(e * sizeof(RunRec)) +
               (ray_order ? bin_scratch_bytes(n) : 0);
    }
    // ray-binning scratch, after the slabs
    void* bin_scratch(const Workspace* w, int64_t n) const {
        const size_t e = size_t(n) * size_t(w->C);
        return static_cast<char*>(w->ptr) + scan_off(n) + al(resume_bytes(n)) + 2 * al(size_t(n) * 4) +
               al(e * sizeof(RunRec));
    }
    // the (device, stream) workspace, grown to fit n rays and tagged for this count
    int claim_ws(int64_t n, void* stream, const void* rays, const void* packed, bool cam,
                 int64_t first, Workspace** out) {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(g_ws_mu);
        Workspace& w = ws_registry()[{dev, stream}];
        int64_t C = slab_cap;
        size_t need = need_bytes(n, C);
        if (w.bytes < need) { // the full slab does not fit what is held: size it from free memory
            C = cap_for(n, slab_budget_bytes(w.bytes));
            int64_t fit = slab_cap; // or keep the largest slab the held block already fits
            while (fit > C && need_bytes(n, fit) > w.bytes) fit -= 4;
            C = std::max(C, fit);
            need = need_bytes(n, C);
        }
        if (w.bytes < need) {
            cudaFree(w.ptr); // synchronous: work still reading it has finished
            w.ptr = nullptr;
            w.bytes = 0;
            CK(cudaMalloc(&w.ptr, need), "sampler workspace");
            w.bytes = need;
        }
        w.C = C;
        w.token = ++g_count_tokens;
        w.owner = id;
        w.rays = rays;
        w.packed = packed;
        w.cam = cam;
        w.first = first;
        w.n = n;
        *out = &w;
        return SOGK_OK;
    }
    // the workspace holding this sampler's slabs for these rays, or nullptr; token != 0 must
    // match the count's token, token == 0 (the token-less API) matches on the buffers
    Workspace* owned_ws(void* stream, uint64_t token, const void* rays, const void* packed, bool cam,
                        int64_t first, int64_t n) const {
        Workspace* w = workspace_peek(stream);
        if (!w || w->owner != id || w->n != n || w->cam != cam) return nullptr;
        if (token) return w->token == token ? w : nullptr;
        if (w->packed != packed) return nullptr;
        if (cam ? w->first != first : w->rays != rays) return nullptr;
        return w;
    }
    static size_t scan_off(int64_t n) { return ((size_t(scan_tiles(n)) * 8 + 64 + 255) / 256) * 256; }
    static uint64_t* tiles(const Workspace* w) { return static_cast<uint64_t*>(w->ptr); }
    // counters: [scan tile counter (u32 in a u64 slot) | overflow counter]
    static unsigned* ovf_ctr(const Workspace* w, int64_t n) {
        return reinterpret_cast<unsigned*>(tiles(w) + scan_tiles(n) + 1);
    }
    SlabDev slab(const Workspace* w, int64_t n) const {
        char* p = static_cast<char*>(w->ptr) + scan_off(n);
        SlabDev S{};
        S.C = w->C;
        S.resume = reinterpret_cast<Resume*>(p);
        p += al(resume_bytes(n));
        S.ovf_list = reinterpret_cast<uint32_t*>(p);
        p += al(size_t(n) * 4);
        S.nruns = reinterpret_cast<int32_t*>(p);
        p += al(size_t(n) * 4);
        S.runs = reinterpret_cast<RunRec*>(p);
        S.ovf_ctr = ovf_ctr(w, n);
        return S;
    }

    // Upper bound on the samples of one camera ray (render scratch sizing without a host
    // round trip), or -1 when none is cheap to state.  Every sample lies in the clipped range
    // of the outermost level box, consecutive samples are >= dt0 - ulp(D)/2 apart (the ladder
    // adds step(t) >= dt0 and rounds once, t <= D = the camera's farthest box corner).
    int64_t max_points_per_camera_ray(const sogk_camera& c) const {
        const GridDev& g = dev.lv[n_levels - 1];
        double chord2 = 0.0, far2 = 0.0;
        for (int a = 0; a < 3; ++a) {
            const double lo = g.wmin[a], hi = g.wmin[a] + double(g.res[a]) * g.voxel;
            chord2 += (hi - lo) * (hi - lo);
            const double f = std::max(std::fabs(c.position[a] - lo), std::fabs(c.position[a] - hi));
            far2 += f * f;
        }
        const double D = std::sqrt(far2) * (1.0 + 1e-9) + 1.0;
        const double ulpD = std::nextafter(D, DBL_MAX) - D;
        if (!(ulpD < dev.dt0 * 0x1p-20) || !std::isfinite(D)) return -1;
        const double m = dev.dt0 - ulpD;
        const double k = std::floor(std::sqrt(chord2) * (1.0 + 1e-9) / m) + 2.0;
        return k < 1e12 ? int64_t(k) : -1;
    }
};

// ---------------------------------------------------------------------------
// library
// ---------------------------------------------------------------------------
extern "C" {

const char* sogk_version(void) { return "sogk 0.1.0 (sm_100a)"; }
int sogk_abi_version(void) { return SOGK_ABI_VERSION; }

const char* sogk_status_string(int s) {
    switch (s) {
        case SOGK_OK: return "ok";
        case SOGK_INVALID_ARG: return "invalid argument";
        case SOGK_CUDA_ERROR: return "CUDA error";
        case SOGK_OOM: return "out of device memory";
        case SOGK_INSUFFICIENT_CAPACITY: return "insufficient output capacity";
        case SOGK_IO_ERROR: return "I/O error";
        case SOGK_NO_DEVICE: return "no CUDA device";
        default: return "unknown status";
    }
}

int sogk_last_error_set(int status, const char* msg) { return fail(status, msg ? msg : ""); }

int sogk_last_error(char* buf, size_t len) {
    if (buf && len) {
        const size_t n = std::min(len - 1, g_err.size());
        std::memcpy(buf, g_err.data(), n);
        buf[n] = 0;
    }
    return int(g_err.size());
}

int sogk_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ---------------------------------------------------------------------------
// grids
// ---------------------------------------------------------------------------
static int create_dense(const sogk_transform* t, const uint8_t* bits, size_t nbytes, bool host,
                        void* stream, sogk_grid** out) {
    if (!out) return fail(SOGK_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!valid_transform(t))
        return fail(SOGK_INVALID_ARG, "grid resolution components must be >= 1 and voxel size positive");
    if (!bits) return fail(SOGK_INVALID_ARG, "bit payload is NULL");
    if (nbytes != payload_bytes(*t))
        return fail(SOGK_INVALID_ARG, "payload size must be ceil(voxel_count / 8) bytes");
    auto* g = new sogk_grid;
    g->kind = SOGK_GRID_DENSE;
    g->t = *t;
    g->nbytes = nbytes;
    cudaGetDevice(&g->device);
    cudaError_t e = galloc(&g->bits, nbytes, S(stream));
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(g->bits, bits, nbytes,
                            host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, S(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream)); // caller may free its buffer
    if (e != cudaSuccess) {
        delete g;
        return cuda_fail(e, "dense grid upload");
    }
    *out = g;
    return SOGK_OK;
}

int sogk_grid_create_dense(const sogk_transform* t, const uint8_t* h_bits, size_t nbytes,
                           void* stream, sogk_grid** out) {
    return create_dense(t, h_bits, nbytes, true, stream, out);
}

int sogk_grid_create_dense_device(const sogk_transform* t, const uint8_t* d_bits, size_t nbytes,
                                  void* stream, sogk_grid** out) {
    return create_dense(t, d_bits, nbytes, false, stream, out);
}

static cudaError_t alloc_vdb(sogk_grid* g, cudaStream_t st) {
    for (int a = 0; a < 3; ++a) g->R[a] = (g->t.res[a] + 127) / 128;
    g->nreg = int64_t(g->R[0]) * g->R[1] * g->R[2];
    g->leaf_capacity = uint64_t(g->nreg) * 4096;
    cudaError_t e;
    if ((e = galloc(&g->root, g->nreg, st)) != cudaSuccess) return e;
    if ((e = galloc(&g->child_mask, g->nreg * 64, st)) != cudaSuccess) return e;
    if ((e = galloc(&g->value_mask, g->nreg * 64, st)) != cudaSuccess) return e;
    if ((e = galloc(&g->prefix, g->nreg * 64, st)) != cudaSuccess) return e;
    if ((e = galloc(&g->table, g->nreg * 4096, st)) != cudaSuccess) return e;
    if ((e = galloc(&g->region_leaves, g->nreg, st)) != cudaSuccess) return e;
    if ((e = galloc(&g->total_leaves, 1, st)) != cudaSuccess) return e;
    return cudaSuccess;
}

int sogk_grid_build_vdb(const sogk_grid* d, void* stream, sogk_grid** out) {
    if (!out) return fail(SOGK_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!d || d->kind != SOGK_GRID_DENSE)
        return fail(SOGK_INVALID_ARG, "build_vdb needs a dense grid");
    if (d->t.res[0] > 1024 * 128 || d->t.res[1] > 1024 * 128 || d->t.res[2] > 1024 * 128)
        return fail(SOGK_INVALID_ARG, "resolution too large");
    auto* g = new sogk_grid;
    g->kind = SOGK_GRID_VDB;
    g->t = d->t;
    g->device = d->device;
    cudaError_t e = alloc_vdb(g, S(stream));
    if (e == cudaSuccess) e = galloc(&g->leaves, g->leaf_capacity * 8, S(stream));
    if (e != cudaSuccess) {
        delete g;
        return cuda_fail(e, "vdb allocation");
    }
    VdbBuildArgs a{};
    a.dense = d->dev();
    for (int k = 0; k < 3; ++k) a.R[k] = g->R[k];
    a.root = g->root;
    a.child_mask = g->child_mask;
    a.value_mask = g->value_mask;
    a.prefix = g->prefix;
    a.table = g->table;
    a.leaves = g->leaves;
    a.region_leaves = g->region_leaves;
    a.total_leaves = g->total_leaves;
    e = launch_vdb_build(a, S(stream));
    if (e == cudaSuccess) e = g->mark(S(stream));
    if (e != cudaSuccess) {
        delete g;
        return cuda_fail(e, "vdb build launch");
    }
    *out = g;
    return SOGK_OK;
}

int sogk_grid_build_distance(const sogk_grid* d, void* stream, sogk_grid** out) {
    if (!out) return fail(SOGK_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!d || d->kind != SOGK_GRID_DENSE)
        return fail(SOGK_INVALID_ARG, "build_distance needs a dense grid");
    for (int a = 0; a < 3; ++a)
        if (d->t.res[a] > 2047) return fail(SOGK_INVALID_ARG, "distance lines are limited to 2047 voxels");
    auto* g = new sogk_grid;
    g->kind = SOGK_GRID_DISTANCE;
    g->t = d->t;
    g->device = d->device;
    const uint64_t n = voxel_count(d->t);
    int32_t* scratch = nullptr;
    cudaError_t e = galloc(&g->dist, n, S(stream));
    if (e == cudaSuccess) e = galloc(&g->dist_any, 1, S(stream));
    if (e == cudaSuccess) e = galloc(&scratch, n, S(stream));
    if (e == cudaSuccess) e = launch_distance_build(d->dev(), g->dist, scratch, g->dist_any, S(stream));
    if (scratch) cudaFreeAsync(scratch, S(stream)); // stream-ordered: after the passes
    if (e == cudaSuccess) e = g->mark(S(stream));
    if (e != cudaSuccess) {
        delete g;
        return cuda_fail(e, "distance build");
    }
    *out = g;
    return SOGK_OK;
}

int sogk_grid_download_distance(const sogk_grid* g, int32_t* h_dist, size_t count,
                                int32_t* all_empty) {
    if (!g || g->kind != SOGK_GRID_DISTANCE) return fail(SOGK_INVALID_ARG, "not a distance grid");
    const uint64_t n = voxel_count(g->t);
    CK(g->wait_ready(), "build completion");
    if (h_dist) {
        if (count < n) return fail(SOGK_INSUFFICIENT_CAPACITY, "buffer smaller than the grid");
        CK(cudaMemcpy(h_dist, g->dist, n * sizeof(int32_t), cudaMemcpyDeviceToHost), "distance D2H");
    }
    if (all_empty) {
        unsigned any = 0;
        CK(cudaMemcpy(&any, g->dist_any, sizeof(unsigned), cudaMemcpyDeviceToHost), "flag D2H");
        *all_empty = any ? 0 : 1;
    }
    return SOGK_OK;
}

int sogk_grid_destroy(sogk_grid* g) {
    delete g;
    return SOGK_OK;
}

int sogk_grid_get_info(const sogk_grid* g, sogk_grid_info* out) {
    if (!g || !out) return fail(SOGK_INVALID_ARG, "NULL argument");
    int st = g->fetch_meta();
    if (st) return st;
    std::memset(out, 0, sizeof(*out));
    out->kind = g->kind;
    out->transform = g->t;
    if (g->kind == SOGK_GRID_DENSE) {
        out->memory_bytes = int64_t(g->nbytes); // io.hpp:223-225
        out->device_bytes = int64_t(g->nbytes);
        return SOGK_OK;
    }
    if (g->kind == SOGK_GRID_DISTANCE) { // variant_memory_bytes: voxel_count * 4 (bench.hpp:468-470)
        out->memory_bytes = int64_t(voxel_count(g->t)) * 4;
        out->device_bytes = out->memory_bytes;
        return SOGK_OK;
    }
    int64_t internal = 0;
    for (int32_t r : g->h_root) internal += r >= 0;
    const int64_t entries = g->from_file
                                ? int64_t(std::count_if(g->h_root.begin(), g->h_root.end(),
                                                        [](int32_t r) { return r != -3; })) +
                                      int64_t(g->extra_entries.size())
                                : g->nreg;
    out->root_entries = entries;
    out->internal_nodes = internal;
    out->leaf_count = g->leaf_count;
    // memory_bytes(SparseGrid) == SOG1 size (io.hpp:227-238)
    out->memory_bytes = (4 + 4 + 12 + 24 + 8 + 4) + entries * 13 + internal * 4096 +
                        g->leaf_count * 64;
    out->device_bytes = g->nreg * (4 + 64 * (8 + 8 + 4) + 4 + 4096 * 4) + 4 + int64_t(g->leaf_capacity) * 64;
    return SOGK_OK;
}

// ---------------------------------------------------------------------------
// SOG0 / SOG1 (io.hpp:134-214)
// ---------------------------------------------------------------------------
namespace {
struct Writer {
    std::vector<uint8_t> out;
    void bytes(const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        out.insert(out.end(), b, b + n);
    }
    void u8(uint8_t v) { out.push_back(v); }
    void u32(uint32_t v) {
        for (int i = 0; i < 4; ++i) out.push_back(uint8_t(v >> (8 * i)));
    }
    void f64(double v) {
        uint64_t b;
        std::memcpy(&b, &v, 8);
        for (int i = 0; i < 8; ++i) out.push_back(uint8_t(b >> (8 * i)));
    }
    void transform(const sogk_transform& t) { // write_transform io.hpp:308-316
        for (int a = 0; a < 3; ++a) u32(uint32_t(t.res[a]));
        for (int a = 0; a < 3; ++a) f64(t.world_min[a]);
        f64(t.voxel_size);
    }
};

struct Reader { // ByteReader io.hpp:272-306; returns false + message on error
    const uint8_t* p;
    size_t n, pos = 0;
    std::string err;
    int code = 0; // 0 ok, 1 bad magic, 2 bad version, 3 truncated, 4 corrupt
    bool need(size_t k) {
        if (pos + k > n) {
            if (!code) {
                code = 3;
                err = "unexpected end of data (truncated)";
            }
            return false;
        }
        return true;
    }
    uint8_t u8() { return need(1) ? p[pos++] : 0; }
    uint32_t u32() {
        if (!need(4)) return 0;
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= uint32_t(p[pos + i]) << (8 * i);
        pos += 4;
        return v;
    }
    double f64() {
        if (!need(8)) return 0;
        uint64_t b = 0;
        for (int i = 0; i < 8; ++i) b |= uint64_t(p[pos + i]) << (8 * i);
        pos += 8;
        double v;
        std::memcpy(&v, &b, 8);
        return v;
    }
    bool corrupt(const char* what) {
        if (!code) {
            code = 4;
            err = std::string(what) + " (corrupt)";
        }
        return false;
    }
    bool magic(const char* m) {
        if (!need(4)) return false;
        if (std::memcmp(p + pos, m, 4) != 0) {
            code = 1;
            err = "not a grid file (bad magic)";
            return false;
        }
        pos += 4;
        return true;
    }
    bool version() {
        const uint32_t v = u32();
        if (code) return false;
        if (v != 1) {
            code = 2;
            err = "unsupported version (bad version)";
            return false;
        }
        return true;
    }
    bool transform(sogk_transform& t) { // read_transform io.hpp:318-333
        const uint32_t rx = u32(), ry = u32(), rz = u32();
        t.world_min[0] = f64();
        t.world_min[1] = f64();
        t.world_min[2] = f64();
        t.voxel_size = f64();
        if (code) return false;
        if (rx < 1 || ry < 1 || rz < 1 || !(t.voxel_size > 0.0))
            return corrupt("invalid grid transform");
        if (uint64_t(rx) * ry * rz > (uint64_t(1) << 33)) return corrupt("resolution too large");
        t.res[0] = int32_t(rx);
        t.res[1] = int32_t(ry);
        t.res[2] = int32_t(rz);
        return true;
    }
};

int io_fail(const Reader& r) { return fail(SOGK_IO_ERROR, r.err); }
} // namespace

int sogk_grid_export_sog0(const sogk_grid* g, uint8_t* buf, size_t* len) {
    if (!g || !len) return fail(SOGK_INVALID_ARG, "NULL argument");
    if (g->kind != SOGK_GRID_DENSE) return fail(SOGK_INVALID_ARG, "SOG0 export needs a dense grid");
    const size_t need = 4 + 4 + 12 + 24 + 8 + g->nbytes;
    if (!buf) {
        *len = need;
        return SOGK_OK;
    }
    if (*len < need) {
        *len = need;
        return fail(SOGK_INSUFFICIENT_CAPACITY, "buffer too small for SOG0");
    }
    Writer w;
    w.bytes("SOG0", 4);
    w.u32(1);
    w.transform(g->t);
    std::memcpy(buf, w.out.data(), w.out.size());
    CK(cudaMemcpy(buf + w.out.size(), g->bits, g->nbytes, cudaMemcpyDeviceToHost), "payload D2H");
    *len = need;
    return SOGK_OK;
}

int sogk_grid_load_sog0(const uint8_t* bytes, size_t len, void* stream, sogk_grid** out) {
    if (!out || (!bytes && len)) return fail(SOGK_INVALID_ARG, "NULL argument");
    *out = nullptr;
    Reader r{bytes, len};
    sogk_transform t{};
    if (!r.magic("SOG0") || !r.version() || !r.transform(t)) return io_fail(r);
    const uint64_t nb = payload_bytes(t);
    if (!r.need(nb)) return io_fail(r);
    if (r.pos + nb != len) { // expect_end
        r.corrupt("trailing bytes after payload");
        return io_fail(r);
    }
    return sogk_grid_create_dense(&t, bytes + r.pos, nb, stream, out);
}

int sogk_grid_export_sog1(const sogk_grid* g, uint8_t* buf, size_t* len) {
    if (!g || !len) return fail(SOGK_INVALID_ARG, "NULL argument");
    if (g->kind != SOGK_GRID_VDB) return fail(SOGK_INVALID_ARG, "SOG1 export needs a VDB grid");
    int st = g->fetch_meta();
    if (st) return st;
    std::vector<uint64_t> cm(g->nreg * 64), vm(g->nreg * 64);
    std::vector<uint32_t> pf(g->nreg * 64);
    std::vector<uint64_t> lv(size_t(g->leaf_count) * 8);
    CK(cudaMemcpy(cm.data(), g->child_mask, cm.size() * 8, cudaMemcpyDeviceToHost), "mask D2H");
    CK(cudaMemcpy(vm.data(), g->value_mask, vm.size() * 8, cudaMemcpyDeviceToHost), "mask D2H");
    CK(cudaMemcpy(pf.data(), g->prefix, pf.size() * 4, cudaMemcpyDeviceToHost), "prefix D2H");
    if (!lv.empty())
        CK(cudaMemcpy(lv.data(), g->leaves, lv.size() * 8, cudaMemcpyDeviceToHost), "leaves D2H");
    // root entries in map order: in-grid regions (absent ones skipped for loaded files) + extras
    std::map<std::array<int32_t, 3>, RootEntry, RegionOrder> entries;
    for (int64_t r = 0; r < g->nreg; ++r) {
        const int32_t node = g->h_root[r];
        if (node == -3) continue; // region absent from a loaded file
        RootEntry e{};
        e.origin[0] = int32_t(r % g->R[0]) * 128;
        e.origin[1] = int32_t((r / g->R[0]) % g->R[1]) * 128;
        e.origin[2] = int32_t(r / (int64_t(g->R[0]) * g->R[1])) * 128;
        e.kind = node == kRootEmpty ? 0 : (node == kRootOccupied ? 1 : 2);
        e.node = node;
        entries[{e.origin[0], e.origin[1], e.origin[2]}] = e;
    }
    for (const RootEntry& e : g->extra_entries) entries[{e.origin[0], e.origin[1], e.origin[2]}] = e;
    Writer w; // serialize_sparse io.hpp:161-181
    w.bytes("SOG1", 4);
    w.u32(1);
    w.transform(g->t);
    w.u32(uint32_t(entries.size()));
    for (const auto& kv : entries) {
        const RootEntry& e = kv.second;
        w.u32(uint32_t(e.origin[0]));
        w.u32(uint32_t(e.origin[1]));
        w.u32(uint32_t(e.origin[2]));
        w.u8(e.kind);
        if (e.kind != 2) continue;
        if (e.node < 0) return fail(SOGK_INVALID_ARG, "internal root entry outside the grid");
        for (int ci = 0; ci < 4096; ++ci) {
            const int64_t wi = int64_t(e.node) * 64 + (ci >> 6);
            const int b = ci & 63;
            if ((cm[wi] >> b) & 1ull) {
                w.u8(2);
                const uint64_t leaf =
                    pf[wi] + uint64_t(__builtin_popcountll(cm[wi] & ((1ull << b) - 1ull)));
                w.bytes(&lv[leaf * 8], 64); // little-endian words == LeafNode bytes
            } else {
                w.u8(uint8_t((vm[wi] >> b) & 1ull));
            }
        }
    }
    if (!buf) {
        *len = w.out.size();
        return SOGK_OK;
    }
    if (*len < w.out.size()) {
        *len = w.out.size();
        return fail(SOGK_INSUFFICIENT_CAPACITY, "buffer too small for SOG1");
    }
    std::memcpy(buf, w.out.data(), w.out.size());
    *len = w.out.size();
    return SOGK_OK;
}

int sogk_grid_load_sog1(const uint8_t* bytes, size_t len, void* stream, sogk_grid** out) {
    if (!out || (!bytes && len)) return fail(SOGK_INVALID_ARG, "NULL argument");
    *out = nullptr;
    Reader r{bytes, len};
    sogk_transform t{};
    if (!r.magic("SOG1") || !r.version() || !r.transform(t)) return io_fail(r);
    const uint32_t n_entries = r.u32();
    if (r.code) return io_fail(r);
    auto* g = new sogk_grid;
    g->kind = SOGK_GRID_VDB;
    g->t = t;
    g->from_file = true;
    cudaGetDevice(&g->device);
    for (int a = 0; a < 3; ++a) g->R[a] = (t.res[a] + 127) / 128;
    g->nreg = int64_t(g->R[0]) * g->R[1] * g->R[2];
    std::vector<int32_t> root(g->nreg, -3); // -3: absent region (queries read empty internal tile)
    std::vector<uint64_t> cm(g->nreg * 64, 0), vm(g->nreg * 64, 0);
    std::vector<uint32_t> pf(g->nreg * 64, 0);
    std::vector<uint64_t> leaves;
    std::vector<std::array<int32_t, 3>> seen;
    std::map<std::array<int32_t, 3>, int, RegionOrder> dup;
    for (uint32_t e = 0; e < n_entries; ++e) {
        std::array<int32_t, 3> o;
        o[0] = int32_t(r.u32());
        o[1] = int32_t(r.u32());
        o[2] = int32_t(r.u32());
        const uint8_t kind = r.u8();
        if (r.code) break;
        if (kind > 2) {
            r.corrupt("invalid root entry kind");
            break;
        }
        if (dup.count(o)) {
            r.corrupt("duplicate root entry");
            break;
        }
        dup[o] = 1;
        // an entry is reachable by queries only at a 128-aligned in-grid origin
        const bool mapped = o[0] >= 0 && o[1] >= 0 && o[2] >= 0 && o[0] % 128 == 0 &&
                            o[1] % 128 == 0 && o[2] % 128 == 0 && o[0] / 128 < g->R[0] &&
                            o[1] / 128 < g->R[1] && o[2] / 128 < g->R[2];
        const int64_t reg = mapped ? (int64_t(o[2] / 128) * g->R[1] + o[1] / 128) * g->R[0] + o[0] / 128 : -1;
        int32_t node = kind == 0 ? kRootEmpty : kRootOccupied;
        std::vector<uint8_t> kinds;
        std::vector<uint64_t> node_leaves;
        if (kind == 2) {
            kinds.resize(4096);
            for (int ci = 0; ci < 4096 && !r.code; ++ci) {
                const uint8_t ck = r.u8();
                if (r.code) break;
                if (ck > 2) {
                    r.corrupt("invalid child kind");
                    break;
                }
                kinds[ci] = ck;
                if (ck == 2) {
                    if (!r.need(64)) break;
                    uint64_t w8[8];
                    std::memcpy(w8, bytes + r.pos, 64);
                    r.pos += 64;
                    node_leaves.insert(node_leaves.end(), w8, w8 + 8);
                }
            }
            if (r.code) break;
        }
        if (!mapped) {
            RootEntry x{{o[0], o[1], o[2]}, kind, -1};
            if (kind == 2) { // unreachable node: keep it for export in a private slot
                r.corrupt("internal root entry outside the grid is not supported");
                break;
            }
            g->extra_entries.push_back(x);
            continue;
        }
        if (kind == 2) {
            node = int32_t(reg);
            uint32_t base = uint32_t(leaves.size() / 8);
            for (int w = 0; w < 64; ++w) {
                pf[reg * 64 + w] = base;
                for (int b = 0; b < 64; ++b) {
                    const uint8_t ck = kinds[w * 64 + b];
                    if (ck == 2) {
                        cm[reg * 64 + w] |= 1ull << b;
                        ++base;
                    } else if (ck == 1) {
                        vm[reg * 64 + w] |= 1ull << b;
                    }
                }
            }
            leaves.insert(leaves.end(), node_leaves.begin(), node_leaves.end());
        }
        root[reg] = node;
    }
    if (!r.code && r.pos != len) r.corrupt("trailing bytes after payload");
    if (r.code) {
        delete g;
        return io_fail(r);
    }
    // absent regions answer like an empty internal tile (sparse.hpp:166-168)
    std::vector<int32_t> dev_root(root);
    for (auto& x : dev_root)
        if (x == -3) x = kRootEmpty;
    g->leaf_capacity = leaves.size() / 8;
    // legacy stream: the synchronous uploads below are ordered after the allocations
    cudaError_t e = alloc_vdb(g, nullptr);
    if (e == cudaSuccess) e = galloc(&g->leaves, std::max<size_t>(leaves.size(), 8), nullptr);
    const uint32_t tl = uint32_t(leaves.size() / 8);
    if (e == cudaSuccess) e = cudaMemcpy(g->root, dev_root.data(), dev_root.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->child_mask, cm.data(), cm.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->value_mask, vm.data(), vm.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->prefix, pf.data(), pf.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !leaves.empty())
        e = cudaMemcpy(g->leaves, leaves.data(), leaves.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->total_leaves, &tl, 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        VdbBuildArgs a{};
        for (int k = 0; k < 3; ++k) a.R[k] = g->R[k];
        a.root = g->root;
        a.child_mask = g->child_mask;
        a.value_mask = g->value_mask;
        a.prefix = g->prefix;
        a.table = g->table;
        e = launch_vdb_table(a, S(stream));
        if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
    }
    if (e != cudaSuccess) {
        delete g;
        return cuda_fail(e, "SOG1 upload");
    }
    g->h_root = root;
    g->leaf_count = tl;
    g->meta_ready = true;
    *out = g;
    return SOGK_OK;
}

int sogk_grid_download_dense(const sogk_grid* g, uint8_t* h_bits, size_t nbytes) {
    if (!g || !h_bits) return fail(SOGK_INVALID_ARG, "NULL argument");
    if (nbytes != payload_bytes(g->t)) return fail(SOGK_INVALID_ARG, "payload size mismatch");
    if (g->kind == SOGK_GRID_DENSE) {
        CK(cudaMemcpy(h_bits, g->bits, nbytes, cudaMemcpyDeviceToHost), "payload D2H");
        return SOGK_OK;
    }
    CK(g->wait_ready(), "build completion");
    uint8_t* d = nullptr;
    CK(cudaMalloc(&d, nbytes), "to_dense scratch");
    cudaError_t e = launch_vdb_to_dense(g->dev(), d, int64_t(nbytes), nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(h_bits, d, nbytes, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "to_dense");
    return SOGK_OK;
}

// ---------------------------------------------------------------------------
// samplers
// ---------------------------------------------------------------------------
int sogk_sampler_create(const sogk_grid* const* levels, int n_levels,
                        const sogk_sampler_desc* desc, sogk_sampler** out) {
    if (!out) return fail(SOGK_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!levels || !desc) return fail(SOGK_INVALID_ARG, "NULL argument");
    if (n_levels < 1) return fail(SOGK_INVALID_ARG, "cascade has no levels");
    if (n_levels > SOGK_MAX_LEVELS) return fail(SOGK_INVALID_ARG, "too many cascade levels");
    if (desc->analyzer != SOGK_DDA && desc->analyzer != SOGK_HDDA && desc->analyzer != SOGK_CD)
        return fail(SOGK_INVALID_ARG, "unknown analyzer");
    if (desc->kernel != SOGK_BRANCH && desc->kernel != SOGK_SKIP)
        return fail(SOGK_INVALID_ARG, "unknown kernel");
    // StepSchedule::constant / linear validation (sampling.hpp:25-34)
    if (desc->schedule != SOGK_CONSTANT && desc->schedule != SOGK_LINEAR)
        return fail(SOGK_INVALID_ARG, "unknown schedule");
    if (!(desc->dt0 > 0.0)) return fail(SOGK_INVALID_ARG, "step size must be positive");
    if (desc->schedule == SOGK_LINEAR && desc->growth < 0.0)
        return fail(SOGK_INVALID_ARG, "growth must be non-negative");
    const int want = desc->analyzer == SOGK_DDA    ? SOGK_GRID_DENSE
                     : desc->analyzer == SOGK_HDDA ? SOGK_GRID_VDB
                                                   : SOGK_GRID_DISTANCE;
    for (int b = 0; b < n_levels; ++b) {
        if (!levels[b]) return fail(SOGK_INVALID_ARG, "NULL grid level");
        if (levels[b]->kind != want)
            return fail(SOGK_INVALID_ARG, "analyzers are bound to their grid: dda marches dense "
                                          "grids, hdda VDBs, cd distance grids");
    }
    const bool cascade = desc->cascade || n_levels > 1;
    if (cascade) { // validate_cascade (sampling.hpp:253-273)
        const sogk_transform& base = levels[0]->t;
        for (int b = 0; b < n_levels; ++b) {
            const sogk_transform& t = levels[b]->t;
            if (t.res[0] != base.res[0] || t.res[1] != base.res[1] || t.res[2] != base.res[2])
                return fail(SOGK_INVALID_ARG, "cascade levels must share one resolution");
            const double expected = base.voxel_size * static_cast<double>(1u << b);
            if (std::abs(t.voxel_size - expected) > 1e-12 * expected)
                return fail(SOGK_INVALID_ARG, "cascade voxel sizes must double per level");
            if (b > 0) {
                const sogk_transform& p = levels[b - 1]->t;
                for (int a = 0; a < 3; ++a) {
                    const double lo = t.world_min[a], hi = lo + double(t.res[a]) * t.voxel_size;
                    const double plo = p.world_min[a],
                                 phi = plo + double(p.res[a]) * p.voxel_size;
                    if (plo < lo || phi > hi)
                        return fail(SOGK_INVALID_ARG, "cascade level bounds must nest");
                }
            }
        }
    }
    auto* s = new sogk_sampler;
    s->desc = *desc;
    s->n_levels = n_levels;
    s->v.analyzer = desc->analyzer;
    s->v.cascade = cascade ? 1 : 0;
    s->v.branch = desc->kernel == SOGK_BRANCH ? 1 : 0;
    s->v.linear = desc->schedule == SOGK_LINEAR ? 1 : 0;
    if (const char* e = std::getenv("SOGK_SLAB")) s->slab_cap = std::max(0, std::atoi(e));
    for (int b = 0; b < n_levels; ++b) {
        s->dev.lv[b] = levels[b]->dev();
        s->lv[b] = levels[b];
        // a single-region VDB (128^3 and below): its one root entry goes into the sampler's
        // constant parameters, so the query's dependent chain is child table -> leaf word
        const sogk_grid* L = levels[b];
        if (SOGK_NODE0 && L->kind == SOGK_GRID_VDB && L->R[0] == 1 && L->R[1] == 1 && L->R[2] == 1 && L->root) {
            int32_t r0 = 0;
            cudaError_t e = L->wait_ready();
            if (e == cudaSuccess) e = cudaMemcpy(&r0, L->root, sizeof r0, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                delete s;
                return cuda_fail(e, "root entry");
            }
            s->dev.lv[b].node0 = r0;
        }
        for (int a = 0; a < 3; ++a) s->max_res = std::max(s->max_res, levels[b]->t.res[a]);
    }
    s->dev.n_levels = n_levels;
    s->dev.spin_cap = desc->spin_cap > 0 ? desc->spin_cap : SOGK_DEFAULT_SPIN_CAP;
    s->dev.dt0 = desc->dt0;
    s->dev.inv_dt0 = 1.0 / desc->dt0;
    s->dev.growth = desc->schedule == SOGK_LINEAR ? desc->growth : 0.0;
    // largest t with fl(growth * t) <= dt0: below it the linear step is the constant dt0
    if (s->dev.growth > 0.0) {
        double x = desc->dt0 / s->dev.growth;
        while (s->dev.growth * x > desc->dt0) x = std::nextafter(x, 0.0);
        while (s->dev.growth * std::nextafter(x, DBL_MAX) <= desc->dt0) x = std::nextafter(x, DBL_MAX);
        s->dev.t_switch = x;
    } else {
        s->dev.t_switch = DBL_MAX;
    }
    *out = s;
    return SOGK_OK;
}

int sogk_release_workspaces(void) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    CK(cudaDeviceSynchronize(), "release sync");
    for (auto& kv : ws_registry()) cudaFree(kv.second.ptr);
    ws_registry().clear();
    for (auto& kv : render_registry()) {
        std::lock_guard<std::mutex> r(kv.second->mu);
        kv.second->release();
    }
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolTrimTo(pool, 0); // grid blocks kept by the pool
    return SOGK_OK;
}

int sogk_sampler_set_ray_order(sogk_sampler* s, int order) {
    if (!s || (order != 0 && order != 1)) return fail(SOGK_INVALID_ARG, "ray order must be 0 or 1");
    s->ray_order = order;
    return SOGK_OK;
}

int sogk_sampler_destroy(sogk_sampler* s) {
    delete s;
    return SOGK_OK;
}

static CameraDev to_dev(const sogk_camera& c) {
    CameraDev d{};
    for (int a = 0; a < 3; ++a) {
        d.position[a] = c.position[a];
        d.forward[a] = c.forward[a];
        d.right[a] = c.right[a];
        d.cam_up[a] = c.cam_up[a];
    }
    d.tan_half = c.tan_half;
    d.aspect = c.aspect;
    d.t_far = c.t_far;
    d.width = c.width;
    d.height = c.height;
    return d;
}

static int count_impl(sogk_sampler* s, const double* d_rays, const sogk_camera* cam,
                      int64_t first, int64_t n, int64_t* d_packed, int64_t* d_stats,
                      uint8_t* d_status, int32_t* d_counters, void* stream, uint64_t* token = nullptr) {
    if (token) *token = 0;
    if (!s) return fail(SOGK_INVALID_ARG, "sampler is NULL");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative ray count");
    if (n >= (int64_t(1) << 32)) return fail(SOGK_INVALID_ARG, "at most 2^32 - 1 rays per call");
    if (!d_stats) return fail(SOGK_INVALID_ARG, "stats buffer is NULL");
    if (n > 0 && (!d_packed || (!cam && !d_rays)))
        return fail(SOGK_INVALID_ARG, "NULL device buffer");
    if (n > 0 && (!aligned16(d_packed) || (!cam && !aligned16(d_rays)))) return fail(SOGK_INVALID_ARG, kAlign16);
    int st = s->wait_levels(stream);
    if (st) return st;
    CK(cudaMemsetAsync(d_stats, 0, SOGK_STATS_LEN * sizeof(int64_t), S(stream)), "stats reset");
    if (n == 0) return SOGK_OK;
    Workspace* w = nullptr;
    st = s->claim_ws(n, stream, cam ? nullptr : d_rays, d_packed, cam != nullptr, first, &w);
    if (st) return st;
    const int64_t tiles = scan_tiles(n);
    CK(cudaMemsetAsync(w->ptr, 0, size_t(tiles) * 8 + 64, S(stream)), "workspace reset");
    CameraDev cd{};
    if (cam) cd = to_dev(*cam);
    const SlabDev slab = s->slab(w, n);
    uint32_t* perm = nullptr;
    if (s->ray_order && !cam)
        CK(launch_ray_binning(s->dev, d_rays, n, s->bin_scratch(w, n), &perm, S(stream)), "ray binning");
    // SOGK_L2_PERSIST=1 (experiment; measured no gain): pass 1 of a single VDB runs
    // with an L2 persisting access-policy window over its child tables + leaves' first MBs
    static const bool l2p = std::getenv("SOGK_L2_PERSIST") != nullptr;
    const sogk_grid* g0 = s->lv[0];
    const bool persist = l2p && s->n_levels == 1 && g0 && g0->kind == SOGK_GRID_VDB;
    if (persist) {
        static std::once_flag once;
        std::call_once(once, [] {
            int dev = 0, mx = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
            if (mx > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(mx));
            cudaGetLastError();
        });
        cudaStreamAttrValue av{};
        av.accessPolicyWindow.base_ptr = g0->table;
        av.accessPolicyWindow.num_bytes = size_t(g0->nreg) * 4096 * sizeof(int32_t);
        av.accessPolicyWindow.hitRatio = 1.0f;
        av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CK(cudaStreamSetAttribute(S(stream), cudaStreamAttributeAccessPolicyWindow, &av), "L2 window");
    }
    CK(launch_count(s->v, s->dev, d_rays, cam ? &cd : nullptr, first, n, d_packed, d_stats,
                    d_status, d_counters, slab, S(stream), perm),
       "count launch");
    if (persist) { // restore the caller's stream
        cudaStreamAttrValue av{};
        av.accessPolicyWindow.num_bytes = 0;
        CK(cudaStreamSetAttribute(S(stream), cudaStreamAttributeAccessPolicyWindow, &av), "L2 window");
    }
    CK(launch_scan(n, d_packed, d_stats, sogk_sampler::tiles(w),
                   reinterpret_cast<unsigned int*>(sogk_sampler::tiles(w) + tiles), S(stream)),
       "scan launch");
    if (token) *token = w->token;
    return SOGK_OK;
}

static bool camera_range_ok(const sogk_camera* cam, int64_t first, int64_t n) {
    return cam && cam->width >= 1 && cam->height >= 1 && first >= 0 &&
           first + n <= int64_t(cam->width) * cam->height;
}

int sogk_sample_count(sogk_sampler* s, const double* d_rays, int64_t n, int64_t* d_packed_info,
                      int64_t* d_stats, uint8_t* d_status, int32_t* d_counters, void* stream) {
    return count_impl(s, d_rays, nullptr, 0, n, d_packed_info, d_stats, d_status, d_counters,
                      stream);
}

int sogk_sample_count_ex(sogk_sampler* s, const double* d_rays, int64_t n, int64_t* d_packed_info,
                         int64_t* d_stats, uint8_t* d_status, int32_t* d_counters, void* stream,
                         uint64_t* token) {
    return count_impl(s, d_rays, nullptr, 0, n, d_packed_info, d_stats, d_status, d_counters,
                      stream, token);
}

int sogk_sample_count_camera(sogk_sampler* s, const sogk_camera* cam, int64_t first_pixel,
                             int64_t n, int64_t* d_packed_info, int64_t* d_stats,
                             uint8_t* d_status, int32_t* d_counters, void* stream) {
    if (!camera_range_ok(cam, first_pixel, n)) return fail(SOGK_INVALID_ARG, "pixel outside image");
    return count_impl(s, nullptr, cam, first_pixel, n, d_packed_info, d_stats, d_status,
                      d_counters, stream);
}

static int write_impl(sogk_sampler* s, const double* d_rays, const sogk_camera* cam, int64_t first,
                      int64_t n, const int64_t* d_packed, uint64_t token, int64_t base, double* ts,
                      double* te, int32_t* ri, uint32_t* ce, uint8_t* lv, void* stream) {
    if (!s) return fail(SOGK_INVALID_ARG, "sampler is NULL");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative ray count");
    if (n >= (int64_t(1) << 32)) return fail(SOGK_INVALID_ARG, "at most 2^32 - 1 rays per call");
    if (ri && (base < 0 || base + n - 1 > int64_t(INT32_MAX)))
        return fail(SOGK_INVALID_ARG, "ray_indices are int32: ray_index_base + n - 1 must be <= INT32_MAX");
    if (ce && s->max_res > 1024)
        return fail(SOGK_INVALID_ARG, "cells pack 10 bits per axis: grids above 1024 voxels per axis "
                                      "cannot export cells");
    if (n == 0) return SOGK_OK;
    if (!d_packed || !ts || (!cam && !d_rays)) return fail(SOGK_INVALID_ARG, "NULL device buffer");
    if (!aligned16(d_packed) || (!cam && !aligned16(d_rays))) return fail(SOGK_INVALID_ARG, kAlign16);
    int st = s->wait_levels(stream);
    if (st) return st;
    CameraDev cd{};
    if (cam) cd = to_dev(*cam);
    // the slabs are valid when pass 1 ran on this sampler, stream and rays
    const Workspace* w = s->owned_ws(stream, token, cam ? nullptr : d_rays, d_packed, cam != nullptr, first, n);
    const bool same = w != nullptr;
    const SlabDev slab = same ? s->slab(w, n) : SlabDev{};
    CK(launch_write(s->v, s->dev, d_rays, cam ? &cd : nullptr, first, n, d_packed,
                    same ? &slab : nullptr, base, ts, te, ri, ce, lv, S(stream)),
       "write launch");
    return SOGK_OK;
}

int sogk_sample_write(sogk_sampler* s, const double* d_rays, int64_t n,
                      const int64_t* d_packed_info, int64_t ray_index_base, double* d_t_starts,
                      double* d_t_ends, int32_t* d_ray_indices, uint32_t* d_cells,
                      uint8_t* d_levels, void* stream) {
    return write_impl(s, d_rays, nullptr, 0, n, d_packed_info, 0, ray_index_base, d_t_starts,
                      d_t_ends, d_ray_indices, d_cells, d_levels, stream);
}

int sogk_sample_write_ex(sogk_sampler* s, const double* d_rays, int64_t n,
                         const int64_t* d_packed_info, uint64_t token, int64_t ray_index_base,
                         double* d_t_starts, double* d_t_ends, int32_t* d_ray_indices,
                         uint32_t* d_cells, uint8_t* d_levels, void* stream) {
    return write_impl(s, d_rays, nullptr, 0, n, d_packed_info, token ? token : ~uint64_t(0),
                      ray_index_base, d_t_starts, d_t_ends, d_ray_indices, d_cells, d_levels, stream);
}

int sogk_sample_write_camera(sogk_sampler* s, const sogk_camera* cam, int64_t first_pixel,
                             int64_t n, const int64_t* d_packed_info, int64_t ray_index_base,
                             double* d_t_starts, double* d_t_ends, int32_t* d_ray_indices,
                             uint32_t* d_cells, uint8_t* d_levels, void* stream) {
    if (!camera_range_ok(cam, first_pixel, n)) return fail(SOGK_INVALID_ARG, "pixel outside image");
    return write_impl(s, nullptr, cam, first_pixel, n, d_packed_info, 0, ray_index_base, d_t_starts,
                      d_t_ends, d_ray_indices, d_cells, d_levels, stream);
}

// ---- traverse ----------------------------------------------------------------
int sogk_traverse_count(sogk_sampler* s, const double* d_rays, int64_t n, int64_t* d_event_info,
                        int64_t* d_stats, uint8_t* d_status, int32_t* d_counters, void* stream) {
    if (!s) return fail(SOGK_INVALID_ARG, "sampler is NULL");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative ray count");
    if (!d_stats) return fail(SOGK_INVALID_ARG, "stats buffer is NULL");
    if (n > 0 && (!d_rays || !d_event_info)) return fail(SOGK_INVALID_ARG, "NULL device buffer");
    if (n > 0 && (!aligned16(d_rays) || !aligned16(d_event_info))) return fail(SOGK_INVALID_ARG, kAlign16);
    int st = s->wait_levels(stream);
    if (st) return st;
    CK(cudaMemsetAsync(d_stats, 0, SOGK_STATS_LEN * sizeof(int64_t), S(stream)), "stats reset");
    if (n == 0) return SOGK_OK;
    CK(launch_traverse_count(s->v, s->dev, d_rays, n, d_event_info, d_stats, d_status, d_counters,
                             S(stream)),
       "traverse launch");
    // the scan's look-back tiles come from the stream-ordered pool (not the sampling workspace,
    // whose slabs a pending write may still need)
    const int64_t tiles = scan_tiles(n);
    uint64_t* t = nullptr;
    CK(retain_pool(), "pool");
    CK(cudaMallocAsync(reinterpret_cast<void**>(&t), size_t(tiles + 2) * 8, S(stream)), "scan tiles");
    cudaError_t e = cudaMemsetAsync(t, 0, size_t(tiles + 2) * 8, S(stream));
    if (e == cudaSuccess)
        e = launch_scan(n, d_event_info, d_stats, t, reinterpret_cast<unsigned int*>(t + tiles), S(stream));
    cudaFreeAsync(t, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "traverse scan");
    return SOGK_OK;
}

int sogk_traverse_write(sogk_sampler* s, const double* d_rays, int64_t n,
                        const int64_t* d_event_info, sogk_event* d_events, void* stream) {
    if (!s) return fail(SOGK_INVALID_ARG, "sampler is NULL");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative ray count");
    if (n == 0) return SOGK_OK;
    if (!d_rays || !d_event_info || !d_events) return fail(SOGK_INVALID_ARG, "NULL device buffer");
    if (!aligned16(d_rays) || !aligned16(d_event_info) || (reinterpret_cast<uintptr_t>(d_events) & 7))
        return fail(SOGK_INVALID_ARG, "device rays / event_info must be 16-byte aligned, events 8-byte");
    int st = s->wait_levels(stream);
    if (st) return st;
    CK(launch_traverse_write(s->v, s->dev, d_rays, n, d_event_info, d_events, S(stream)), "traverse launch");
    return SOGK_OK;
}

int sogk_traverse_host(sogk_sampler* s, const double* h_rays, int64_t n, int64_t capacity,
                       int64_t* h_event_info, sogk_event* h_events, uint8_t* h_status,
                       int32_t* h_counters, int64_t* h_stats, void* stream) {
    if (!s || !h_stats) return fail(SOGK_INVALID_ARG, "NULL argument");
    if (n < 0 || capacity < 0) return fail(SOGK_INVALID_ARG, "negative size");
    if (n > 0 && (!h_rays || !h_event_info)) return fail(SOGK_INVALID_ARG, "NULL host buffer");
    std::lock_guard<std::mutex> hold(s->host_mu);
    for (int k = 0; k < SOGK_STATS_LEN; ++k) h_stats[k] = 0;
    if (n == 0) return SOGK_OK;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t b_rays = al(size_t(n) * 64), b_info = al(size_t(n) * 16), b_stats = 256,
                 b_status = al(size_t(n)), b_ctr = al(size_t(n) * 8);
    char* p = nullptr;
    CK(cudaMalloc(&p, b_rays + b_info + b_stats + b_status + b_ctr), "traverse scratch");
    double* d_rays = reinterpret_cast<double*>(p);
    int64_t* d_info = reinterpret_cast<int64_t*>(p + b_rays);
    int64_t* d_stats = reinterpret_cast<int64_t*>(p + b_rays + b_info);
    uint8_t* d_status = reinterpret_cast<uint8_t*>(p + b_rays + b_info + b_stats);
    int32_t* d_ctr = reinterpret_cast<int32_t*>(p + b_rays + b_info + b_stats + b_status);
    sogk_event* d_ev = nullptr;
    int rc = SOGK_OK;
    cudaError_t e = cudaMemcpyAsync(d_rays, h_rays, size_t(n) * 64, cudaMemcpyHostToDevice, S(stream));
    if (e == cudaSuccess) {
        rc = sogk_traverse_count(s, d_rays, n, d_info, d_stats, d_status, d_ctr, stream);
        if (rc == SOGK_OK) {
            e = cudaMemcpyAsync(h_stats, d_stats, SOGK_STATS_LEN * 8, cudaMemcpyDeviceToHost, S(stream));
            if (e == cudaSuccess) e = cudaMemcpyAsync(h_event_info, d_info, size_t(n) * 16, cudaMemcpyDeviceToHost, S(stream));
            if (e == cudaSuccess && h_status) e = cudaMemcpyAsync(h_status, d_status, size_t(n), cudaMemcpyDeviceToHost, S(stream));
            if (e == cudaSuccess && h_counters) e = cudaMemcpyAsync(h_counters, d_ctr, size_t(n) * 8, cudaMemcpyDeviceToHost, S(stream));
            if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
            const int64_t total = h_stats[SOGK_STAT_TOTAL_SAMPLES];
            if (e == cudaSuccess && total > capacity) {
                rc = fail(SOGK_INSUFFICIENT_CAPACITY, "event capacity below the event total");
            } else if (e == cudaSuccess && total > 0) {
                if (!h_events) {
                    rc = fail(SOGK_INVALID_ARG, "NULL host event buffer");
                } else {
                    e = cudaMalloc(&d_ev, size_t(total) * sizeof(sogk_event));
                    if (e == cudaSuccess) {
                        rc = sogk_traverse_write(s, d_rays, n, d_info, d_ev, stream);
                        if (rc == SOGK_OK)
                            e = cudaMemcpyAsync(h_events, d_ev, size_t(total) * sizeof(sogk_event),
                                                cudaMemcpyDeviceToHost, S(stream));
                        if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
                    }
                }
            }
        }
    }
    cudaFree(d_ev);
    cudaFree(p);
    if (e != cudaSuccess) return cuda_fail(e, "traverse host path");
    return rc;
}

int sogk_grid_query(const sogk_grid* g, const int32_t* d_ijk, int64_t n, sogk_query* d_out,
                    void* stream) {
    if (!g) return fail(SOGK_INVALID_ARG, "grid is NULL");
    if (g->kind == SOGK_GRID_DISTANCE) return fail(SOGK_INVALID_ARG, "query needs a dense or VDB grid");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative point count");
    if (n == 0) return SOGK_OK;
    if (!d_ijk || !d_out) return fail(SOGK_INVALID_ARG, "NULL device buffer");
    if (g->ready) CK(cudaStreamWaitEvent(S(stream), g->ready, 0), "grid build wait");
    CK(launch_query(g->dev(), g->kind == SOGK_GRID_VDB ? 1 : 0, d_ijk, n, d_out, S(stream)), "query launch");
    return SOGK_OK;
}

int sogk_grid_query_host(const sogk_grid* g, const int32_t* h_ijk, int64_t n, sogk_query* h_out) {
    if (!g) return fail(SOGK_INVALID_ARG, "grid is NULL");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative point count");
    if (n == 0) return SOGK_OK;
    if (!h_ijk || !h_out) return fail(SOGK_INVALID_ARG, "NULL host buffer");
    char* p = nullptr;
    const size_t b_in = (size_t(n) * 12 + 255) & ~size_t(255);
    CK(cudaMalloc(&p, b_in + size_t(n) * sizeof(sogk_query)), "query scratch");
    cudaError_t e = cudaMemcpy(p, h_ijk, size_t(n) * 12, cudaMemcpyHostToDevice);
    int rc = SOGK_OK;
    if (e == cudaSuccess) rc = sogk_grid_query(g, reinterpret_cast<int32_t*>(p), n,
                                               reinterpret_cast<sogk_query*>(p + b_in), nullptr);
    if (e == cudaSuccess && rc == SOGK_OK)
        e = cudaMemcpy(h_out, p + b_in, size_t(n) * sizeof(sogk_query), cudaMemcpyDeviceToHost);
    cudaFree(p);
    if (e != cudaSuccess) return cuda_fail(e, "query");
    return rc;
}

// ---- compositing consumer ------------------------------------------------
struct sogk_scene {
    SceneDev dev{};
    sogk_primitive* d_prims = nullptr;
    int* d_grid = nullptr;
    ~sogk_scene() {
        cudaFree(d_prims);
        cudaFree(d_grid);
    }
};

// Candidate grid (SceneDev): a cube of kCells^3 cells around the union of the primitive
// bounding boxes; a primitive is listed in every cell its box (grown by one cell on each
// side, far above rounding in Primitive::contains) touches.
static void build_candidate_grid(const sogk_primitive* p, int32_t n, SceneDev& d,
                                 std::vector<int>& cstart, std::vector<int>& cand) {
    d.gres = 0;
    if (n < 4) return; // a loop over a few primitives is as cheap as the lookup
    double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
    auto box = [&](const sogk_primitive& q, double* b0, double* b1) {
        for (int a = 0; a < 3; ++a) {
            b0[a] = q.shape == SOGK_SPHERE ? q.center[a] - q.radius : q.lo[a];
            b1[a] = q.shape == SOGK_SPHERE ? q.center[a] + q.radius : q.hi[a];
        }
    };
    for (int32_t i = 0; i < n; ++i) {
        double b0[3], b1[3];
        box(p[i], b0, b1);
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], b0[a]);
            hi[a] = std::max(hi[a], b1[a]);
        }
    }
    double ext = 0.0;
    for (int a = 0; a < 3; ++a) ext = std::max(ext, hi[a] - lo[a]);
    if (!(ext > 0.0) || !std::isfinite(ext)) return;
    constexpr int kCells = 32;
    const double cell = ext / kCells;
    d.gres = kCells;
    d.ginv = 1.0 / cell;
    for (int a = 0; a < 3; ++a) d.glo[a] = lo[a];
    std::vector<std::vector<int>> lists(size_t(kCells) * kCells * kCells);
    for (int32_t i = 0; i < n; ++i) {
        double b0[3], b1[3];
        box(p[i], b0, b1);
        int c0[3], c1[3];
        for (int a = 0; a < 3; ++a) {
            c0[a] = std::max(0, int(std::floor((b0[a] - lo[a]) / cell)) - 1);
            c1[a] = std::min(kCells - 1, int(std::floor((b1[a] - lo[a]) / cell)) + 1);
        }
        for (int z = c0[2]; z <= c1[2]; ++z)
            for (int y = c0[1]; y <= c1[1]; ++y)
                for (int x = c0[0]; x <= c1[0]; ++x)
                    lists[(size_t(z) * kCells + y) * kCells + x].push_back(i); // ascending i
    }
    cstart.assign(lists.size() + 1, 0);
    for (size_t c = 0; c < lists.size(); ++c) cstart[c + 1] = cstart[c] + int(lists[c].size());
    cand.clear();
    cand.reserve(size_t(cstart.back()));
    for (const auto& l : lists) cand.insert(cand.end(), l.begin(), l.end());
}

int sogk_scene_create(const sogk_primitive* h_prims, int32_t n, const double background[3],
                      sogk_scene** out) {
    if (!out || n < 0 || (n > 0 && !h_prims) || !background)
        return fail(SOGK_INVALID_ARG, "sogk_scene_create: NULL argument or negative count");
    for (int32_t i = 0; i < n; ++i) { // AnalyticScene::validate (render.hpp:62-70)
        const sogk_primitive& p = h_prims[i];
        if (p.shape != SOGK_SPHERE && p.shape != SOGK_BOX)
            return fail(SOGK_INVALID_ARG, "primitive shape must be sphere or box");
        if (p.density < 0.0) return fail(SOGK_INVALID_ARG, "primitive density must be >= 0");
        for (int c = 0; c < 3; ++c)
            if (p.color[c] < 0.0 || p.color[c] > 1.0)
                return fail(SOGK_INVALID_ARG, "primitive color must lie in [0,1]");
    }
    auto* sc = new sogk_scene;
    if (n > 0) {
        cudaError_t e = cudaMalloc(&sc->d_prims, size_t(n) * sizeof(sogk_primitive));
        if (e == cudaSuccess)
            e = cudaMemcpy(sc->d_prims, h_prims, size_t(n) * sizeof(sogk_primitive), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            delete sc;
            return cuda_fail(e, "scene upload");
        }
    }
    sc->dev.prims = sc->d_prims;
    sc->dev.n = n;
    for (int a = 0; a < 3; ++a) sc->dev.bg[a] = background[a];
    std::vector<int> cstart, cand;
    build_candidate_grid(h_prims, n, sc->dev, cstart, cand);
    if (sc->dev.gres > 0) {
        const size_t nb = (cstart.size() + cand.size()) * sizeof(int);
        cudaError_t e = cudaMalloc(&sc->d_grid, nb);
        if (e == cudaSuccess)
            e = cudaMemcpy(sc->d_grid, cstart.data(), cstart.size() * sizeof(int), cudaMemcpyHostToDevice);
        if (e == cudaSuccess && !cand.empty())
            e = cudaMemcpy(sc->d_grid + cstart.size(), cand.data(), cand.size() * sizeof(int),
                           cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            delete sc;
            return cuda_fail(e, "scene grid upload");
        }
        sc->dev.cstart = sc->d_grid;
        sc->dev.cand = sc->d_grid + cstart.size();
    }
    *out = sc;
    return SOGK_OK;
}

int sogk_scene_destroy(sogk_scene* scene) {
    delete scene;
    return SOGK_OK;
}

int sogk_composite(const sogk_sampler* s, const sogk_scene* scene, const double* d_rays, int64_t n,
                   const int64_t* d_packed_info, const double* d_t_starts, double* d_result,
                   uint8_t* d_rgb8, void* stream) {
    if (!s || !scene) return fail(SOGK_INVALID_ARG, "sampler or scene is NULL");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative ray count");
    if (n == 0) return SOGK_OK;
    if (!d_rays || !d_packed_info || (!d_result && !d_rgb8))
        return fail(SOGK_INVALID_ARG, "NULL device buffer");
    if (!aligned16(d_rays) || !aligned16(d_packed_info)) return fail(SOGK_INVALID_ARG, kAlign16);
    CK(launch_composite(s->v, s->dev, scene->dev, d_rays, n, d_packed_info, d_t_starts, d_result,
                        d_rgb8, S(stream)),
       "composite launch");
    return SOGK_OK;
}

int sogk_render_camera(sogk_sampler* s, const sogk_scene* scene, const sogk_camera* cam,
                       int64_t first_pixel, int64_t n, double* d_result, uint8_t* d_rgb8,
                       int64_t* d_stats, void* stream) {
    if (!s || !scene) return fail(SOGK_INVALID_ARG, "sampler or scene is NULL");
    if (n < 0) return fail(SOGK_INVALID_ARG, "negative ray count");
    if (!camera_range_ok(cam, first_pixel, n)) return fail(SOGK_INVALID_ARG, "pixel outside image");
    if (!d_result && !d_rgb8) return fail(SOGK_INVALID_ARG, "NULL device buffer");
    std::lock_guard<std::mutex> hold(s->host_mu);
    RenderScratch* rs = render_scratch_for(stream);
    std::lock_guard<std::mutex> hold_rs(rs->mu);
    int st = rs->ensure_rays(n);
    if (st) return st;
    int64_t* stats = d_stats ? d_stats : rs->stats();
    int64_t* packed = rs->packed();
    // Sample capacity: the camera's bound when it fits in a quarter of free memory (allocated
    // once per stream; the frame then runs without any host round trip), else the exact total
    // read back after pass 1 (one sync), with geometric growth.
    const bool force_sync = std::getenv("SOGK_RENDER_SYNC") != nullptr; // tests: the sync path
    const int64_t per = force_sync ? -1 : s->max_points_per_camera_ray(*cam);
    bool fixed = false;
    if (per >= 0 && n > 0 && per <= INT64_MAX / 64 / n) {
        const int64_t bound = per * n;
        if (bound <= rs->smp_cap) {
            fixed = true;
        } else if (bound < rs->unfit_bound) {
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) cudaGetLastError();
            if (double(bound) * RenderScratch::kSampleBytes <= 0.25 * double(fr)) {
                st = rs->ensure_samples(bound, stream);
                if (st) return st;
                fixed = true;
            } else {
                rs->unfit_bound = bound;
            }
        }
    }
    uint64_t tok = 0;
    st = count_impl(s, nullptr, cam, first_pixel, n, packed, stats, nullptr, nullptr, stream, &tok);
    if (st) return st;
    if (n == 0) return SOGK_OK;
    int64_t hint = rs->smp_cap;
    if (!fixed) {
        CK(cudaMemcpyAsync(rs->h_total, stats + SOGK_STAT_TOTAL_SAMPLES, 8, cudaMemcpyDeviceToHost, S(stream)),
           "total D2H");
        CK(cudaStreamSynchronize(S(stream)), "count sync");
        hint = *rs->h_total;
        if (hint > rs->smp_cap) {
            st = rs->ensure_samples(hint + hint / 2, stream);
            if (st) return st;
        }
    }
    // pass 2 (t_starts, ray_indices), the ray buffer for shading, then shade + accumulate
    if (hint > 0) {
        st = write_impl(s, nullptr, cam, first_pixel, n, packed, tok, 0, rs->ts(), nullptr, rs->ri(),
                        nullptr, nullptr, stream);
        if (st) return st;
    }
    const CameraDev cd = to_dev(*cam);
    CK(launch_raygen(cd, first_pixel, n, rs->rays_buf(), S(stream)), "raygen");
    CK(launch_shade_accumulate(s->v, s->dev, scene->dev, rs->rays_buf(), n, packed, rs->ts(), rs->ri(),
                               stats + SOGK_STAT_TOTAL_SAMPLES, hint, 0, rs->shaded(), d_result, d_rgb8,
                               S(stream)),
       "render shade");
    return SOGK_OK;
}

int sogk_render_frame_host(sogk_sampler* s, const sogk_scene* scene, const sogk_camera* cam,
                           uint8_t* h_rgb8, int64_t* h_stats, void* stream) {
    if (!s || !scene || !cam || !h_rgb8) return fail(SOGK_INVALID_ARG, "NULL argument");
    const int64_t n = int64_t(cam->width) * cam->height;
    uint8_t* d_rgb = nullptr;
    int64_t* d_stats = nullptr;
    cudaError_t e = dalloc(&d_rgb, size_t(n) * 3);
    if (e == cudaSuccess) e = dalloc(&d_stats, SOGK_STATS_LEN);
    int st = e == cudaSuccess ? SOGK_OK : cuda_fail(e, "render buffers");
    if (st == SOGK_OK)
        st = sogk_render_camera(s, scene, cam, 0, n, nullptr, d_rgb, d_stats, stream);
    if (st == SOGK_OK) {
        e = cudaMemcpyAsync(h_rgb8, d_rgb, size_t(n) * 3, cudaMemcpyDeviceToHost, S(stream));
        if (e == cudaSuccess && h_stats)
            e = cudaMemcpyAsync(h_stats, d_stats, SOGK_STATS_LEN * 8, cudaMemcpyDeviceToHost, S(stream));
        if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
        if (e != cudaSuccess) st = cuda_fail(e, "render D2H");
    }
    cudaFree(d_rgb);
    cudaFree(d_stats);
    return st;
}

int sogk_camera_rays(const sogk_camera* cam, int64_t first_pixel, int64_t n, double* d_rays,
                     void* stream) {
    if (!camera_range_ok(cam, first_pixel, n) || (n && !d_rays))
        return fail(SOGK_INVALID_ARG, "pixel outside image");
    CK(launch_raygen(to_dev(*cam), first_pixel, n, d_rays, S(stream)), "raygen launch");
    return SOGK_OK;
}

int sogk_sample_host(sogk_sampler* s, const double* h_rays, int64_t n, int64_t ray_index_base,
                     int64_t capacity, int64_t* h_packed_info, double* h_t_starts,
                     double* h_t_ends, int32_t* h_ray_indices, uint32_t* h_cells,
                     uint8_t* h_levels, uint8_t* h_status, int32_t* h_counters,
                     int64_t* h_stats, void* stream) {
    if (!s || !h_stats) return fail(SOGK_INVALID_ARG, "NULL argument");
    if (n < 0 || capacity < 0) return fail(SOGK_INVALID_ARG, "negative size");
    if (n > 0 && (!h_rays || !h_packed_info)) return fail(SOGK_INVALID_ARG, "NULL host buffer");
    if (h_ray_indices && (ray_index_base < 0 || ray_index_base + n - 1 > int64_t(INT32_MAX)))
        return fail(SOGK_INVALID_ARG, "ray_indices are int32: ray_index_base + n - 1 must be <= INT32_MAX");
    std::lock_guard<std::mutex> hold(s->host_mu); // per-sampler scratch, lanes and pinned stats
    // Chunked pipeline over kLanes internal streams: chunk c's upload and pass 1 overlap the
    // pass 2 and download of chunk c-1 (each stream has its own pass-1 -> pass-2 workspace).
    // Offsets are made global on the device before download; the call is synchronous.
    constexpr int kLanes = 3;
    static const int64_t kChunks = [] { // chunks per call (pipeline depth), SOGK_HOST_CHUNKS
        const char* e = std::getenv("SOGK_HOST_CHUNKS");
        const long v = e ? std::atol(e) : 0;
        return int64_t(v >= 1 && v <= 64 ? v : 8);
    }();
    // t_ends and ray_indices are functions of t_starts and packed_info (t_end = t + step(t),
    // sampling.hpp:99,118; ray_indices = ray_index_base + r over each ray's range): when the
    // caller also takes t_starts they are expanded on host threads from the downloaded
    // t_starts / packed_info of each finished chunk, while the next chunks are on the GPU and
    // the PCIe link -- the device->host link is the bound of this call, and this cuts its bytes
    // per sample from 20 to 8.  Same IEEE operation (one add, no FMA), so the bytes are
    // identical to the device's.  SOGK_HOST_EXPAND: "all" (both), "ri" (ray_indices only,
    // t_ends downloaded), "t" (t_ends only, ray_indices downloaded), "0" (download both);
    // default "t" (the balance of PCIe and host memory traffic that measured best)
    static const int kExpand = [] { // bit 0: ray_indices on the host, bit 1: t_ends on the host
        const char* e = std::getenv("SOGK_HOST_EXPAND");
        if (!e) return 2;
        if (e[0] == '0') return 0;
        if (e[0] == 'r') return 1;
        if (e[0] == 't') return 2;
        return 3;
    }();
    static const int kExpandThreads = [] {
        const char* e = std::getenv("SOGK_HOST_THREADS");
        const long v = e ? std::atol(e) : 0;
        const int hw = int(std::thread::hardware_concurrency());
        return int(v >= 1 && v <= 64 ? v : std::max(1, std::min(8, hw / 4)));
    }();
    const bool exp_ri = (kExpand & 1) && h_t_starts && h_ray_indices;
    const bool exp_te = (kExpand & 2) && h_t_starts && h_t_ends;
    const bool expand = exp_ri || exp_te;
    // n / 8 rays per chunk, at most 512 K: big calls get a deeper pipeline (shorter fill and
    // drain; 2^24 probe rays: 32 chunks, +4.5 % e2e over 8)
    const int64_t chunk = std::max<int64_t>(65536, std::min<int64_t>((n + kChunks - 1) / kChunks, 1 << 19));
    const int64_t nchunks = n > 0 ? (n + chunk - 1) / chunk : 0;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t b_rays = al(size_t(n) * 64), b_packed = al(size_t(n) * 16),
                 b_stats = al(size_t(std::max<int64_t>(nchunks, 1)) * SOGK_STATS_LEN * 8),
                 b_status = al(size_t(n)), b_ctr = al(size_t(n) * 12);
    const size_t b_ts = al(size_t(capacity) * 8), b_te = exp_te ? 0 : al(size_t(capacity) * 8),
                 b_ri = exp_ri ? 0 : al(size_t(capacity) * 4), b_ce = al(size_t(capacity) * 4),
                 b_lv = al(size_t(capacity));
    const size_t need = b_rays + b_packed + b_stats + b_status + b_ctr + b_ts + b_te + b_ri + b_ce + b_lv;
    if (need > s->hb_bytes) {
        cudaFree(s->hb);
        s->hb = nullptr;
        s->hb_bytes = 0;
        CK(cudaMalloc(&s->hb, need), "host-path scratch");
        s->hb_bytes = need;
    }
    if (!s->lanes_ready) {
        for (int l = 0; l < kLanes; ++l) {
            CK(cudaStreamCreateWithFlags(&s->lanes[l], cudaStreamNonBlocking), "stream");
            CK(cudaEventCreateWithFlags(&s->lane_ev[l], cudaEventDisableTiming), "event");
        }
        CK(cudaMallocHost(&s->h_chunk_stats, 64 * SOGK_STATS_LEN * 8), "pinned stats");
        s->lanes_ready = true;
    }
    while (int64_t(s->done_ev.size()) < nchunks) {
        cudaEvent_t e = nullptr;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        s->done_ev.push_back(e);
    }
    char* p = static_cast<char*>(s->hb);
    double* d_rays = reinterpret_cast<double*>(p);
    p += b_rays;
    int64_t* d_packed = reinterpret_cast<int64_t*>(p);
    p += b_packed;
    int64_t* d_stats = reinterpret_cast<int64_t*>(p);
    p += b_stats;
    uint8_t* d_status = reinterpret_cast<uint8_t*>(p);
    p += b_status;
    int32_t* d_ctr = reinterpret_cast<int32_t*>(p);
    p += b_ctr;
    double* d_ts = reinterpret_cast<double*>(p);
    p += b_ts;
    double* d_te = reinterpret_cast<double*>(p);
    p += b_te;
    int32_t* d_ri = reinterpret_cast<int32_t*>(p);
    p += b_ri;
    uint32_t* d_ce = reinterpret_cast<uint32_t*>(p);
    p += b_ce;
    uint8_t* d_lv = reinterpret_cast<uint8_t*>(p);

    // order after the caller's prior work on `stream`
    cudaEvent_t start_ev = s->lane_ev[0];
    CK(cudaEventRecord(start_ev, S(stream)), "event");
    for (int l = 0; l < kLanes; ++l) CK(cudaStreamWaitEvent(s->lanes[l], start_ev, 0), "wait");

    for (int k = 0; k < SOGK_STATS_LEN; ++k) h_stats[k] = 0;
    std::vector<int64_t> chunk_stats(size_t(nchunks) * SOGK_STATS_LEN, 0);
    std::vector<uint64_t> tokens(size_t(nchunks), 0);
    std::vector<int64_t> chunk_base(size_t(nchunks), -1); // output offset of a written chunk
    int64_t base = 0;
    bool fits = true;
    int rc = SOGK_OK;
    // host expansion of t_ends / ray_indices, chunk by chunk as their downloads finish
    const double dt0 = s->dev.dt0, growth = s->dev.growth;
    const bool linear = s->v.linear != 0;
    // chunks whose write + downloads are issued (the expander sleeps on the condition variable
    // until the next one is, then on that chunk's download event: no spinning host thread)
    int64_t issued = 0;
    bool abort_exp = false;
    std::mutex exp_mu;
    std::condition_variable exp_cv;
    auto expand_chunk = [&](int64_t c) {
        const int64_t r0 = c * chunk, m = std::min(chunk, n - r0);
        auto work = [&](int64_t a, int64_t b) { // rays [a, b) of the chunk
            if (a >= b) return;
            const int64_t lo = h_packed_info[2 * (r0 + a)];
            const int64_t hi = h_packed_info[2 * (r0 + b - 1)] + h_packed_info[2 * (r0 + b - 1) + 1];
            if (exp_ri) {
                for (int64_t r = r0 + a; r < r0 + b; ++r) {
                    const int64_t off = h_packed_info[2 * r], cnt = h_packed_info[2 * r + 1];
                    std::fill_n(h_ray_indices + off, cnt, int32_t(ray_index_base + r));
                }
            }
            if (exp_te) {
                const double* ts = h_t_starts;
                double* te = h_t_ends;
                if (linear) {
                    for (int64_t i = lo; i < hi; ++i) {
                        const double t = ts[i], g = growth * t;
                        te[i] = t + ((dt0 < g) ? g : dt0); // std::max(dt0, growth * t)
                    }
                } else {
                    for (int64_t i = lo; i < hi; ++i) te[i] = ts[i] + dt0;
                }
            }
        };
        const int T = int(std::min<int64_t>(kExpandThreads, std::max<int64_t>(1, m / 4096)));
        if (T <= 1) {
            work(0, m);
            return;
        }
        std::vector<std::thread> th;
        for (int i = 1; i < T; ++i) th.emplace_back(work, m * i / T, m * (i + 1) / T);
        work(0, m / T);
        for (auto& x : th) x.join();
    };
    std::thread expander;
    if (expand && nchunks > 0) {
        expander = std::thread([&] {
            for (int64_t c = 0; c < nchunks; ++c) {
                {
                    std::unique_lock<std::mutex> lk(exp_mu);
                    exp_cv.wait(lk, [&] { return issued > c || abort_exp; });
                    if (abort_exp) return;
                }
                if (cudaEventSynchronize(s->done_ev[c]) != cudaSuccess) return;
                if (chunk_base[size_t(c)] >= 0) expand_chunk(c);
            }
        });
    }
    // pass 1 of chunk c (upload, count, scan, stats download) on lane c % kLanes
    auto issue_count = [&](int64_t c) -> int {
        cudaStream_t L = s->lanes[c % kLanes];
        const int64_t r0 = c * chunk, m = std::min(chunk, n - r0);
        CK(cudaMemcpyAsync(d_rays + 8 * r0, h_rays + 8 * r0, size_t(m) * 64, cudaMemcpyHostToDevice, L), "rays H2D");
        const int st = count_impl(s, d_rays + 8 * r0, nullptr, 0, m, d_packed + 2 * r0,
                                  d_stats + c * SOGK_STATS_LEN, h_status ? d_status + r0 : nullptr,
                                  h_counters ? d_ctr + 3 * r0 : nullptr, L, &tokens[size_t(c)]);
        if (st) return st;
        int64_t* hs = s->h_chunk_stats + (c % 64) * SOGK_STATS_LEN;
        CK(cudaMemcpyAsync(hs, d_stats + c * SOGK_STATS_LEN, SOGK_STATS_LEN * 8, cudaMemcpyDeviceToHost, L), "stats D2H");
        CK(cudaEventRecord(s->lane_ev[c % kLanes], L), "event");
        return SOGK_OK;
    };
    // pass 2 of chunk c (global offsets, write, downloads) once its total is known
    auto issue_write = [&](int64_t c) -> int {
        cudaStream_t L = s->lanes[c % kLanes];
        CK(cudaEventSynchronize(s->lane_ev[c % kLanes]), "count sync");
        const int64_t r0 = c * chunk, m = std::min(chunk, n - r0);
        const int64_t* hs = s->h_chunk_stats + (c % 64) * SOGK_STATS_LEN;
        for (int k = 0; k < SOGK_STATS_LEN; ++k) chunk_stats[size_t(c) * SOGK_STATS_LEN + k] = hs[k];
        const int64_t tot = hs[SOGK_STAT_TOTAL_SAMPLES];
        CK(launch_add_offset(d_packed + 2 * r0, m, base, L), "offsets");
        if (fits && base + tot <= capacity) {
            chunk_base[size_t(c)] = base;
            if (tot > 0) {
                const int st = write_impl(s, d_rays + 8 * r0, nullptr, 0, m, d_packed + 2 * r0,
                                          tokens[size_t(c)], ray_index_base + r0, d_ts,
                                          (h_t_ends && !exp_te) ? d_te : nullptr,
                                          (h_ray_indices && !exp_ri) ? d_ri : nullptr, h_cells ? d_ce : nullptr,
                                          h_levels ? d_lv : nullptr, L);
                if (st) return st;
                const size_t o = size_t(base), tb = size_t(tot);
                if (h_t_starts) CK(cudaMemcpyAsync(h_t_starts + o, d_ts + o, tb * 8, cudaMemcpyDeviceToHost, L), "D2H");
                if (h_t_ends && !exp_te) CK(cudaMemcpyAsync(h_t_ends + o, d_te + o, tb * 8, cudaMemcpyDeviceToHost, L), "D2H");
                if (h_ray_indices && !exp_ri) CK(cudaMemcpyAsync(h_ray_indices + o, d_ri + o, tb * 4, cudaMemcpyDeviceToHost, L), "D2H");
                if (h_cells) CK(cudaMemcpyAsync(h_cells + o, d_ce + o, tb * 4, cudaMemcpyDeviceToHost, L), "D2H");
                if (h_levels) CK(cudaMemcpyAsync(h_levels + o, d_lv + o, tb, cudaMemcpyDeviceToHost, L), "D2H");
            }
        } else {
            fits = false;
        }
        CK(cudaMemcpyAsync(h_packed_info + 2 * r0, d_packed + 2 * r0, size_t(m) * 16, cudaMemcpyDeviceToHost, L), "D2H");
        if (h_status) CK(cudaMemcpyAsync(h_status + r0, d_status + r0, size_t(m), cudaMemcpyDeviceToHost, L), "D2H");
        if (h_counters) CK(cudaMemcpyAsync(h_counters + 3 * r0, d_ctr + 3 * r0, size_t(m) * 12, cudaMemcpyDeviceToHost, L), "D2H");
        CK(cudaEventRecord(s->done_ev[c], L), "event");
        {
            std::lock_guard<std::mutex> lk(exp_mu);
            issued = c + 1;
        }
        exp_cv.notify_one();
        base += tot;
        return SOGK_OK;
    };
    for (int64_t c = 0; c < nchunks && rc == SOGK_OK; ++c) {
        rc = issue_count(c);
        if (rc == SOGK_OK && c > 0) rc = issue_write(c - 1);
        if (c + 1 == nchunks && rc == SOGK_OK) rc = issue_write(c);
    }
    if (rc != SOGK_OK) {
        {
            std::lock_guard<std::mutex> lk(exp_mu);
            abort_exp = true;
        }
        exp_cv.notify_one();
    }
    for (int l = 0; l < kLanes; ++l) {
        const cudaError_t e = cudaStreamSynchronize(s->lanes[l]);
        if (e != cudaSuccess && rc == SOGK_OK) rc = cuda_fail(e, "pipeline sync");
    }
    if (expander.joinable()) expander.join();
    if (rc) return rc;
    for (int64_t c = 0; c < nchunks; ++c)
        for (int k = 0; k < SOGK_STATS_LEN; ++k) {
            if (k == SOGK_STAT_TOTAL_SAMPLES || k == SOGK_STAT_INVALID_RAYS || k == SOGK_STAT_UNDEFINED_RAYS ||
                k == SOGK_STAT_ANALYZER_LOOKUPS || k == SOGK_STAT_ANALYZER_STEPS ||
                k == SOGK_STAT_KERNEL_LOOKUPS || k == SOGK_STAT_SLAB_OVERFLOW_RAYS)
                h_stats[k] += chunk_stats[size_t(c) * SOGK_STATS_LEN + k];
        }
    if (!fits) return fail(SOGK_INSUFFICIENT_CAPACITY, "output capacity below the sample total");
    return SOGK_OK;
}

} // extern "C"
