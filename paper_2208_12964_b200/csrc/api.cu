// C ABI of uscg_b200 (include/uscg_b200.h): host orchestration in C++.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/uscg_b200.h"
#include "kernels.h"
#include "schedule.h"

namespace ub {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DomainError : std::domain_error {
    using std::domain_error::domain_error;
};
// a nested C-ABI call's failure, passed through with its status
struct StatusError : std::runtime_error {
    uscg_status code;
    StatusError(uscg_status c, const char* msg) : std::runtime_error(msg ? msg : "error"), code(c) {}
};

double norm360(double deg) {  // geometry.cpp:48-55
    deg = std::fmod(deg, 360.0);
    if (deg < 0)
        deg += 360.0;
    if (deg >= 360.0)
        deg = 0.0;
    return deg;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count == n && p)
            return;
        release();
        if (count == 0)
            return;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e != cudaSuccess) {
            p = nullptr;
            throw CudaError(std::string("cudaMalloc ") + std::to_string(count * sizeof(T)) +
                            " bytes: " + cudaGetErrorString(e));
        }
        n = count;
    }
    uint64_t bytes() const { return uint64_t(n) * sizeof(T); }
    void ensure(size_t count) {
        if (count > n)
            alloc(count);
    }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
    }
};
}  // namespace

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_error(const std::string& msg) { g_last_error = msg; }

}  // namespace ub

using namespace ub;

struct ResampleCache;
struct MetricsWork;

struct uscg_ctx_s {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    ResampleCache* resample = nullptr;  // ring table + bin-point map of the last resample grid
    MetricsWork* metrics = nullptr;     // uscg_image_metrics scratch (grown, never shrunk)
};


struct uscg_tracer_s {
    uscg_ctx ctx = nullptr;
    int device = 0;
    // grid
    int n_rings = 0, n_slices = 1, volume = 0;
    double ring_spacing = 0, slice_height = 0;
    std::vector<uint32_t> counts;
    std::vector<RingRow> rings;  // index = ring
    uint32_t cps = 0;
    uint64_t cells = 0;
    // scan
    int lines = 0, views = 0;
    std::vector<double> thetas;
    uint64_t records = 0;
    int max_recs = 0, max_cells = 0;
    std::vector<uint32_t> h_cells;  // per unit
    uint64_t cells_per_sweep = 0;
    // device
    DevBuf<RingRow> d_rings;
    DevBuf<uint32_t> d_off;
    DevBuf<double> d_rays;  // first-view rays [src: lines*3][det: lines*3] (length-weighted model)
    DevBuf<double> d_pa, d_pb;
    DevBuf<uint32_t> d_key;
    DevBuf<double> d_theta;
    DevBuf<uint32_t> d_cells;
    DevBuf<uint8_t> d_crossed;
    bool crossed_built = false;
    // schedule
    bool sched_built = false;
    std::vector<uint32_t> level_off;
    DevBuf<uint32_t> d_order;
    DevBuf<uint32_t> d_level_off;
    DevBuf<unsigned> d_bar;
    DevBuf<uint32_t> d_pred_off, d_preds, d_succ_off, d_succs, d_npred_x;
    int run = 1, n_runs = 0, runs_per_view = 0;  // run-granular schedule (dataflow)
    uint64_t n_preds = 0, n_succs = 0;
    DevBuf<unsigned> d_done;  // dataflow flags [units * nchunks]
    DevBuf<uint32_t> w_slab;  // dataflow trace slab
    DevBuf<unsigned> w_slab_ctl;
    int done_chunks = 0;
    unsigned epoch = 0;
    double schedule_seconds = 0;
    // wave executor (2D stacks): every line's traced list and its other-view
    // requirements (mart_sweep.cu), progress counters [views * nchunks]
    bool wave_built = false;
    DevBuf<uint32_t> d_wpos, d_wdep_off, d_wdeps;
    DevBuf<uint2> d_went, d_wsplit;
    DevBuf<uint32_t> d_wspos;
    uint32_t wave_split_longest = 0;
    int wave_split_parts = 0;
    DevBuf<unsigned> d_wprog, d_wnext;
    int wave_chunks = 0;
    unsigned wave_epoch = 0;
    int wave_ctas = 0;  // CTAs per view task of the last wave solve
    uint64_t wave_deps = 0;
    double wave_seconds = 0;
    double generator_ms = 0;  // device time of the first-view generator
    int executor = -1;        // MART executor of the last reconstruction (uscg_tracer_info)
    // flow executor, one problem: every (view, line)'s traced list (built once
    // per geometry when it fits in device memory)
    bool lists_built = false, lists_off = false;
    DevBuf<uint32_t> d_lists;
    DevBuf<unsigned long long> d_lpos;
    double lists_seconds = 0;
    // tile executor (one small problem): the lines in ASAP level order
    bool tile_built = false, tile_off = false;
    // level executor (mart_levels.cu): every line sorted by ASAP level of the
    // line DAG (run = 1), its level offsets, and per-call scratch for the
    // compaction to the lines with a non-zero measurement
    bool lv_built = false;
    DevBuf<uint32_t> d_lv_order, d_lv_off, w_lv_flags, w_lv_pos, w_lv_live, w_lv_live_off;
    std::vector<uint32_t> lv_off;
    double lv_seconds = 0;
    LevelGraphCache lv_graph;  // a sweep's launches, replayed while the same solve comes back
    DevBuf<uint4> d_tmeta;
    DevBuf<uint32_t> d_tlevel;
    int tile_levels = 0;
    // MART workspace
    DevBuf<float> w_field, w_proj, w_prev, w_stage;
    DevBuf<double> w_pfloor, w_stats;
    DevBuf<uint8_t> w_active;
    DevBuf<unsigned long long> w_clamps, w_updates, w_tmp;
    DevBuf<unsigned int> w_resid;
    // uscg_reconstruct_batch: double-buffered staging and its copy streams
    DevBuf<float> w_bin[4], w_bout[4];
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    // ... and two solve slots, so that one stack's solve starts while the
    // previous one drains (wave executor): a slot's per-solve workspaces and
    // wave progress counters are swapped into the tracer for its solve
    struct SolveSlot {
        DevBuf<float> w_proj, w_field;
        DevBuf<double> w_stats, w_pfloor;
        DevBuf<uint8_t> w_active;
        DevBuf<unsigned long long> w_clamps, w_updates, w_tmp;
        DevBuf<unsigned> d_wprog, d_wnext;
        int wave_chunks = 0;
        unsigned wave_epoch = 0;
        cudaStream_t st = nullptr;
    };
    SolveSlot slots[4];
    void swap_slot(SolveSlot& o) {
        w_proj.swap(o.w_proj);
        w_field.swap(o.w_field);
        w_stats.swap(o.w_stats);
        w_pfloor.swap(o.w_pfloor);
        w_active.swap(o.w_active);
        w_clamps.swap(o.w_clamps);
        w_updates.swap(o.w_updates);
        w_tmp.swap(o.w_tmp);
        d_wprog.swap(o.d_wprog);
        d_wnext.swap(o.d_wnext);
        std::swap(wave_chunks, o.wave_chunks);
        std::swap(wave_epoch, o.wave_epoch);
    }
    ~uscg_tracer_s() {
        if (copy_in)
            cudaStreamDestroy(copy_in);
        if (copy_out)
            cudaStreamDestroy(copy_out);
        for (auto& sl : slots)
            if (sl.st)
                cudaStreamDestroy(sl.st);
    }

    DevGrid dev_grid() const {
        DevGrid g;
        g.n_rings = n_rings;
        g.n_slices = volume ? n_slices : 1;
        g.volume = volume;
        g.ring_spacing = ring_spacing;
        g.slice_height = slice_height;
        g.radius = 0.5 * (2 * n_rings) * ring_spacing;
        g.eps = 1e-9 * g.radius;
        const double z_extent = volume ? n_slices * slice_height : slice_height;
        g.zoff = 0.5 * z_extent;
        g.cells_per_slice = cps;
        g.rings = d_rings.p;
        return g;
    }
    TraceArgs trace_args() const {
        TraceArgs a;
        a.off = d_off.p;
        a.pa = d_pa.p;
        a.pb = d_pb.p;
        a.key = d_key.p;
        a.rings = d_rings.p;
        a.theta = d_theta.p;
        a.cells_per_slice = cps;
        a.lines = lines;
        return a;
    }
    cudaStream_t st() const { return ctx->stream; }
    uint64_t units() const { return uint64_t(lines) * uint64_t(views); }
};

// uscg_image_metrics scratch, kept by the context so repeated scoring does
// not allocate (cudaFree synchronizes the device)
struct MetricsWork {
    DevBuf<double> part, mom, c1c2, spart, sout;
};

// uscg_resample's per-grid state, kept by the context so that repeated calls
// on one grid (a volume resampled slab by slab, or every iteration) allocate
// and build nothing
struct ResampleCache {
    int n_rings = -1, n_slices = 0, volume = 0, npix = 0;
    double ring_spacing = 0, slice_height = 0;
    std::vector<uint32_t> counts;  // empty: the reference law
    std::unique_ptr<uscg_tracer_s> grid;
    DevBuf<uint32_t> map;
    // tiled plan (npix % 32 == 0): per 32x32 tile its distinct cells, per
    // pixel (tile-major) the slot of its cell in that list
    bool tiled = false;
    DevBuf<uint32_t> toff, tcells;
    DevBuf<uint16_t> slot;
    bool matches(const uscg_grid* g, int n) const {
        if (!grid || g->n_rings != n_rings || (g->volume ? g->n_slices : 1) != n_slices ||
            (g->volume ? 1 : 0) != volume || n != npix || g->ring_spacing != ring_spacing ||
            g->slice_height != slice_height || (g->ring_counts == nullptr) != counts.empty())
            return false;
        return !g->ring_counts ||
               std::equal(counts.begin(), counts.end(), g->ring_counts);
    }
};

namespace {

// The tiled resample plan from the pixel -> cell map (bin-point map, or the
// inverse permutation): once per (grid, npix), on the host from the map.
void build_resample_plan(ResampleCache& rc, bool perm, int npix, cudaStream_t st) {
    const size_t npx = size_t(npix) * npix;
    DevBuf<uint32_t> pm;
    const uint32_t* dmap = rc.map.p;
    if (perm) {
        pm.alloc(npx);
        launch_perm_map(npix, pm.p, st);
        dmap = pm.p;
    }
    std::vector<uint32_t> map(npx);
    UB_CUDA(cudaMemcpyAsync(map.data(), dmap, sizeof(uint32_t) * npx, cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    const int T = 32, tx = npix / T, tiles = tx * tx;
    std::vector<uint32_t> toff(size_t(tiles) + 1, 0), tcells, cells;
    std::vector<uint16_t> slot(npx);
    tcells.reserve(npx);
    for (int tile = 0; tile < tiles; ++tile) {
        const int r0 = (tile / tx) * T, c0 = (tile % tx) * T;
        cells.clear();
        for (int i = 0; i < T * T; ++i) {
            const uint32_t c = map[size_t(r0 + i / T) * npix + c0 + i % T];
            if (c != 0xFFFFFFFFu)
                cells.push_back(c);
        }
        std::sort(cells.begin(), cells.end());
        cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
        for (int i = 0; i < T * T; ++i) {
            const uint32_t c = map[size_t(r0 + i / T) * npix + c0 + i % T];
            slot[size_t(tile) * T * T + i] =
                c == 0xFFFFFFFFu ? uint16_t(0xFFFF)
                                 : uint16_t(std::lower_bound(cells.begin(), cells.end(), c) - cells.begin());
        }
        tcells.insert(tcells.end(), cells.begin(), cells.end());
        toff[size_t(tile) + 1] = uint32_t(tcells.size());
    }
    rc.toff.alloc(toff.size());
    rc.tcells.alloc(std::max<size_t>(tcells.size(), 1));
    rc.slot.alloc(slot.size());
    UB_CUDA(cudaMemcpyAsync(rc.toff.p, toff.data(), sizeof(uint32_t) * toff.size(), cudaMemcpyHostToDevice, st));
    if (!tcells.empty())
        UB_CUDA(cudaMemcpyAsync(rc.tcells.p, tcells.data(), sizeof(uint32_t) * tcells.size(), cudaMemcpyHostToDevice,
                                st));
    UB_CUDA(cudaMemcpyAsync(rc.slot.p, slot.data(), sizeof(uint16_t) * slot.size(), cudaMemcpyHostToDevice, st));
    UB_CUDA(cudaStreamSynchronize(st));
}

template <class F>
uscg_status guarded(F&& f) {
    try {
        f();
        return USCG_OK;
    } catch (const InvalidArgument& e) {
        set_error(e.what());
        return USCG_ERR_INVALID_ARGUMENT;
    } catch (const DomainError& e) {
        set_error(e.what());
        return USCG_ERR_DOMAIN;
    } catch (const NoDevice& e) {
        set_error(e.what());
        return USCG_ERR_NO_DEVICE;
    } catch (const StatusError& e) {
        set_error(e.what());
        return e.code;
    } catch (const CudaError& e) {
        set_error(e.what());
        return USCG_ERR_CUDA;
    } catch (const std::bad_alloc& e) {
        set_error("host allocation failed");
        return USCG_ERR_ALLOC;
    } catch (const std::exception& e) {
        set_error(e.what());
        return USCG_ERR_CUDA;
    }
}

void need(bool cond, const char* msg) {
    if (!cond)
        throw InvalidArgument(msg);
}

void bind(uscg_ctx ctx) {
    need(ctx != nullptr, "null context");
    UB_CUDA(cudaSetDevice(ctx->device));
}

// GridSpec::validate (grid.cpp:9-16) on the generalized grid
void validate_grid(const uscg_grid* g) {
    need(g != nullptr, "null grid");
    if (g->n_rings < 1)
        throw InvalidArgument("grid size must be an even integer >= 2, got " +
                              std::to_string(2 * g->n_rings));
    need(g->n_rings <= kMaxRings, "at most 4095 rings are supported");
    need(g->ring_spacing > 0, "ring spacing must be positive");
    need(g->slice_height > 0, "slice height must be positive");
    if (g->volume)
        need(g->n_slices >= 1 && g->n_slices <= kMaxSlices, "slice count out of range");
    if (g->ring_counts)
        for (int k = 0; k < g->n_rings; ++k)
            need(g->ring_counts[k] >= 1 && g->ring_counts[k] <= 4096,
                 "ring sector counts must lie in [1, 4096]");
}

// ScanGeometry::validate (scan.cpp:9-24)
void validate_scan(const uscg_scan* s) {
    need(s != nullptr, "null scan");
    need(s->views >= 1, "number of views must be >= 1");
    need(s->det_u >= 1 && s->det_v >= 1, "detector counts must be >= 1");
    need(s->spacing_u > 0, "detector spacing must be positive");
    need(!(s->det_v > 1 && !(s->spacing_v > 0)), "detector row spacing must be positive");
    need(s->detector >= USCG_DET_FLAT && s->detector <= USCG_DET_PARALLEL, "unknown detector kind");
    const double dot = s->source[0] * s->detector_center[0] + s->source[1] * s->detector_center[1];
    need(dot < 0, "source and detector must sit on opposite sides of the origin");
    const double ax = s->detector_center[0] - s->source[0];
    const double ay = s->detector_center[1] - s->source[1];
    need(!(ax * ax + ay * ay == 0), "central ray must not be axial");
}

void fill_grid(uscg_tracer_s* t, const uscg_grid* g) {
    t->n_rings = g->n_rings;
    t->ring_spacing = g->ring_spacing;
    t->n_slices = g->volume ? g->n_slices : 1;
    t->slice_height = g->slice_height;
    t->volume = g->volume ? 1 : 0;
    t->counts.resize(g->n_rings);
    for (int k = 1; k <= g->n_rings; ++k)
        t->counts[k - 1] = g->ring_counts ? g->ring_counts[k - 1] : uint32_t(4 * (2 * k - 1));
    t->rings.assign(size_t(g->n_rings) + 1, RingRow{0, 0, 0});
    uint64_t head = 0;
    for (int k = 1; k <= g->n_rings; ++k) {
        RingRow& r = t->rings[k];
        r.count = t->counts[k - 1];
        r.head = uint32_t(head);
        r.inv_step = r.count / 360.0;  // grid.cpp:68
        head += r.count;
    }
    need(head * uint64_t(t->n_slices) < (1ull << 32), "cell count must fit in 32 bits");
    t->cps = uint32_t(head);
    t->cells = head * uint64_t(t->n_slices);
    t->d_rings.alloc(t->rings.size());
    UB_CUDA(cudaMemcpy(t->d_rings.p, t->rings.data(), sizeof(RingRow) * t->rings.size(),
                       cudaMemcpyHostToDevice));
}

void fill_views(uscg_tracer_s* t, int views, const double* angles) {
    need(views >= 1, "number of views must be >= 1");
    t->views = views;
    t->thetas.resize(views);
    const double step = 360.0 / views;  // ScanGeometry::step_deg
    for (int v = 0; v < views; ++v)
        t->thetas[v] = norm360(angles ? angles[v] : v * step);
    t->d_theta.alloc(views);
    UB_CUDA(cudaMemcpy(t->d_theta.p, t->thetas.data(), sizeof(double) * views,
                       cudaMemcpyHostToDevice));
}

// max records per line, per-unit cell counts, cells per sweep
void finish_tracer(uscg_tracer_s* t, const std::vector<uint32_t>& off,
                   cudaEvent_t annotated = nullptr) {
    t->max_recs = 0;
    for (int l = 0; l < t->lines; ++l)
        t->max_recs = std::max<int>(t->max_recs, int(off[l + 1] - off[l]));
    launch_annotate(t->lines, t->d_off.p, t->d_pa.p, t->d_pb.p, t->d_key.p, t->d_rings.p, t->st());
    if (annotated)
        UB_CUDA(cudaEventRecord(annotated, t->st()));
    const uint64_t units = t->units();
    need(units < (1ull << 32), "views * lines must fit in 32 bits");
    t->d_cells.alloc(units);
    launch_trace_counts(t->trace_args(), t->views, t->max_recs, t->d_cells.p, t->st());
    t->h_cells.resize(units);
    UB_CUDA(cudaMemcpyAsync(t->h_cells.data(), t->d_cells.p, sizeof(uint32_t) * units,
                            cudaMemcpyDeviceToHost, t->st()));
    UB_CUDA(cudaStreamSynchronize(t->st()));
    t->max_cells = 1;
    t->cells_per_sweep = 0;
    for (uint32_t c : t->h_cells) {
        t->max_cells = std::max<int>(t->max_cells, int(c));
        t->cells_per_sweep += c;
    }
}

void first_view_rays(const uscg_scan* s, double* src, double* det) {
    // ScanGeometry::detector_position (scan.cpp:27-36); the arc and parallel
    // generators reuse its in-plane u direction
    const double ax = s->detector_center[0] - s->source[0];
    const double ay = s->detector_center[1] - s->source[1];
    const double alen = std::sqrt(ax * ax + ay * ay);
    const double ux = -ay / alen;
    const double uy = ax / alen;
    const double pi = 3.141592653589793238462643383279502884;
    for (int iv = 0; iv < s->det_v; ++iv)
        for (int iu = 0; iu < s->det_u; ++iu) {
            const size_t l = size_t(iv) * s->det_u + iu;
            const double du = (iu - 0.5 * (s->det_u - 1)) * s->spacing_u;
            const double dv = (iv - 0.5 * (s->det_v - 1)) * s->spacing_v;
            double* o = src + 3 * l;
            double* q = det + 3 * l;
            o[0] = s->source[0];
            o[1] = s->source[1];
            o[2] = s->source[2];
            if (s->detector == USCG_DET_FLAT) {
                q[0] = s->detector_center[0] + du * ux;
                q[1] = s->detector_center[1] + du * uy;
                q[2] = s->detector_center[2] + dv;
            } else if (s->detector == USCG_DET_ARC) {
                // element iu at angle du (degrees) from the central ray, on
                // the circle about the source through the detector centre
                const double a0 = std::atan2(ay, ax);
                const double g = a0 + du * (pi / 180.0);
                q[0] = s->source[0] + alen * std::cos(g);
                q[1] = s->source[1] + alen * std::sin(g);
                q[2] = s->detector_center[2] + dv;
            } else {
                o[0] = s->source[0] + du * ux;
                o[1] = s->source[1] + du * uy;
                o[2] = s->source[2] + dv;
                q[0] = s->detector_center[0] + du * ux;
                q[1] = s->detector_center[1] + du * uy;
                q[2] = s->detector_center[2] + dv;
            }
        }
}

uscg_tracer_s* build_from_rays(uscg_ctx ctx, const uscg_grid* grid, int lines, const double* src,
                               const double* det, int views, const double* angles) {
    validate_grid(grid);
    need(lines >= 1, "line count must be >= 1");
    need(src && det, "null ray arrays");
    std::unique_ptr<uscg_tracer_s> t(new uscg_tracer_s);
    t->ctx = ctx;
    t->device = ctx->device;
    fill_grid(t.get(), grid);
    fill_views(t.get(), views, angles);
    t->lines = lines;
    DevBuf<double>& d_rays = t->d_rays;
    d_rays.alloc(size_t(lines) * 6);
    UB_CUDA(cudaMemcpyAsync(d_rays.p, src, sizeof(double) * 3 * lines, cudaMemcpyHostToDevice,
                            t->st()));
    UB_CUDA(cudaMemcpyAsync(d_rays.p + 3 * size_t(lines), det, sizeof(double) * 3 * lines,
                            cudaMemcpyHostToDevice, t->st()));
    const DevGrid g = t->dev_grid();
    DevBuf<uint32_t> d_cnt;
    d_cnt.alloc(size_t(lines));
    t->d_off.alloc(size_t(lines) + 1);
    // generator device time: the passes before and after the host allocation
    // of the record store (the allocation itself is not counted)
    cudaEvent_t ev[6];  // [0,1] count or bound, [4,5] slot pass, [2,3] write or compaction + annotate
    for (auto& e : ev)
        UB_CUDA(cudaEventCreate(&e));
    bool timed_slots = false;
    const double* src_d = d_rays.p;
    const double* det_d = d_rays.p + 3 * size_t(lines);
    std::vector<uint32_t> off(size_t(lines) + 1);
    // One pass (default): bounded slots, then compaction. The bound is at most
    // 2 n_rings + n_slices + 4 records per ray; the slot scratch must fit in u32
    // offsets and in device memory, else (or on a slot overflow) the exact
    // count pass runs first.
    bool one_pass = std::getenv("USCG_GEN_TWO_PASS") == nullptr &&
                    uint64_t(lines) * uint64_t(2 * t->n_rings + (t->volume ? t->n_slices : 0) + 4) < (1ull << 32);
    DevBuf<uint32_t> d_boff, d_skey;
    DevBuf<double> d_spa, d_spb;
    DevBuf<unsigned> d_flag;
    if (one_pass) {
        UB_CUDA(cudaEventRecord(ev[0], t->st()));
        launch_generate_bound(g, lines, src_d, det_d, d_cnt.p, t->st());
        d_boff.alloc(size_t(lines) + 1);
        launch_exclusive_scan_u32(d_cnt.p, d_boff.p, lines, t->st());
        UB_CUDA(cudaEventRecord(ev[1], t->st()));
        uint32_t slots = 0;
        UB_CUDA(cudaMemcpy(&slots, d_boff.p + lines, sizeof(uint32_t), cudaMemcpyDeviceToHost));
        size_t free_b = 0, total_b = 0;
        UB_CUDA(cudaMemGetInfo(&free_b, &total_b));
        one_pass = double(slots) * 40.0 < 0.8 * double(free_b);  // slots + the packed store
        if (one_pass) {
            const size_t n = std::max<size_t>(slots, 1);
            d_spa.alloc(n);
            d_spb.alloc(n);
            d_skey.alloc(n);
            d_flag.alloc(1);
            UB_CUDA(cudaMemsetAsync(d_flag.p, 0, sizeof(unsigned), t->st()));
            UB_CUDA(cudaEventRecord(ev[4], t->st()));
            launch_generate_slots(g, lines, src_d, det_d, d_boff.p, d_spa.p, d_spb.p, d_skey.p, d_cnt.p, d_flag.p,
                                  t->st());
            launch_exclusive_scan_u32(d_cnt.p, t->d_off.p, lines, t->st());
            UB_CUDA(cudaEventRecord(ev[5], t->st()));
            timed_slots = true;
            unsigned overflow = 0;
            UB_CUDA(cudaMemcpyAsync(&overflow, d_flag.p, sizeof(unsigned), cudaMemcpyDeviceToHost, t->st()));
            UB_CUDA(cudaMemcpyAsync(off.data(), t->d_off.p, sizeof(uint32_t) * (lines + 1), cudaMemcpyDeviceToHost,
                                    t->st()));
            UB_CUDA(cudaStreamSynchronize(t->st()));
            one_pass = overflow == 0;
        }
    }
    if (!one_pass) {
        d_spa.release();
        d_spb.release();
        d_skey.release();
        timed_slots = false;
        UB_CUDA(cudaEventRecord(ev[0], t->st()));
        launch_generate_count(g, lines, src_d, det_d, d_cnt.p, t->st());
        launch_exclusive_scan_u32(d_cnt.p, t->d_off.p, lines, t->st());
        UB_CUDA(cudaEventRecord(ev[1], t->st()));
        UB_CUDA(cudaMemcpyAsync(off.data(), t->d_off.p, sizeof(uint32_t) * (lines + 1), cudaMemcpyDeviceToHost,
                                t->st()));
        UB_CUDA(cudaStreamSynchronize(t->st()));
    }
    t->records = off[lines];
    const size_t R = std::max<size_t>(t->records, 1);
    t->d_pa.alloc(R);
    t->d_pb.alloc(R);
    t->d_key.alloc(R);
    UB_CUDA(cudaEventRecord(ev[2], t->st()));
    if (one_pass)
        launch_compact_records(lines, d_boff.p, t->d_off.p, d_spa.p, d_spb.p, d_skey.p, t->d_pa.p, t->d_pb.p,
                               t->d_key.p, t->st());
    else
        launch_generate_write(g, lines, src_d, det_d, t->d_off.p, t->d_pa.p, t->d_pb.p, t->d_key.p, t->st());
    finish_tracer(t.get(), off, ev[3]);
    float a = 0, b = 0, c = 0;
    UB_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
    UB_CUDA(cudaEventElapsedTime(&b, ev[2], ev[3]));
    if (timed_slots)
        UB_CUDA(cudaEventElapsedTime(&c, ev[4], ev[5]));
    t->generator_ms = double(a) + double(b) + double(c);
    for (auto& e : ev)
        cudaEventDestroy(e);
    return t.release();
}

void ensure_crossed(uscg_tracer_s* t) {
    if (t->crossed_built)
        return;
    t->d_crossed.alloc(t->cells);
    UB_CUDA(cudaMemsetAsync(t->d_crossed.p, 0, t->cells, t->st()));
    launch_crossed(t->trace_args(), t->views, t->max_recs, t->max_cells, t->d_crossed.p, t->st());
    t->crossed_built = true;
}

// MART executor (USCG_MART_MODE): 0 "flow" dataflow over run dependency
// counters; 3 "wave" one task per (view, problem chunk) ordered by per-view
// progress counters (2D stacks); 4 "tile" one CTA with the field in shared
// memory (one small problem). Unset: "auto" (-1), the wave executor where it
// applies (2D grid, chunks of 4-32 problems, lines within its cover, the
// traced lists within a memory budget), the tile executor for one problem
// whose field and line metadata fit in shared memory, else flow.
int mart_mode() {
    const char* e = std::getenv("USCG_MART_MODE");
    const std::string m = e ? e : "auto";
    if (m == "flow")
        return 0;
    if (m == "wave")
        return 3;
    if (m == "tile")
        return 4;
    if (m == "levels")
        return 5;
    return -1;
}

// lines per run for the dataflow executor (USCG_RUN; default 4 for 2D grids,
// whose adjacent lines always overlap, and 2 for volumes: two neighbouring
// detector pixels of a row share most of their cells' 32-byte sectors, so
// the second line's gathers hit L2; measured C4 119 -> 88 ms, C3 5.9 -> 5.4 ms
// per iteration, while runs of 4 or 8 cost single-warp occupancy: their
// staged lists fill shared memory): the largest divisor of the lines per
// view not above the request
int run_length(int lines, bool volume) {
    int want = volume ? 2 : 4;
    if (const char* e = std::getenv("USCG_RUN"))
        want = std::max(1, std::atoi(e));
    for (int r = std::min(want, lines); r > 1; --r)
        if (lines % r == 0)
            return r;
    return 1;
}

// The run DAG of the host builder (AsapSchedule, USCG_HOST_SCHEDULE=1)
struct RunSchedule {
    std::vector<uint32_t> order, level_off, pred_off, preds, npred_x, succ_off, succs;
    uint32_t levels = 0;
};

// the host builder (schedule.cpp): traces copied back in batches
void host_schedule(uscg_tracer_s* t, RunSchedule& R) {
    AsapSchedule sched(t->cells, uint32_t(t->lines), uint32_t(t->run));
    const uint64_t units = t->units();
    const uint64_t batch_cells = 1ull << 25;  // 128 MiB of indices per batch
    std::vector<uint32_t> pos, idx;
    DevBuf<uint32_t> d_pos, d_idx;
    uint64_t u0 = 0;
    while (u0 < units) {
        uint64_t u1 = u0, tot = 0;
        while (u1 < units && (u1 == u0 || tot + t->h_cells[u1] <= batch_cells)) {
            tot += t->h_cells[u1];
            ++u1;
        }
        const uint32_t n = uint32_t(u1 - u0);
        pos.resize(size_t(n) + 1);
        pos[0] = 0;
        for (uint32_t i = 0; i < n; ++i)
            pos[i + 1] = pos[i] + t->h_cells[u0 + i];
        d_pos.ensure(pos.size());
        d_idx.ensure(std::max<uint64_t>(tot, 1));
        UB_CUDA(cudaMemcpyAsync(d_pos.p, pos.data(), sizeof(uint32_t) * pos.size(), cudaMemcpyHostToDevice, t->st()));
        launch_trace_dump(t->trace_args(), uint32_t(u0), n, t->max_recs, t->max_cells, d_pos.p, d_idx.p, t->st());
        idx.resize(std::max<uint64_t>(tot, 1));
        UB_CUDA(cudaMemcpyAsync(idx.data(), d_idx.p, sizeof(uint32_t) * tot, cudaMemcpyDeviceToHost, t->st()));
        UB_CUDA(cudaStreamSynchronize(t->st()));
        sched.add(idx.data(), pos.data(), n);
        u0 = u1;
    }
    sched.done();
    sched.finish(R.order, R.level_off);
    R.levels = sched.levels();
    R.pred_off = sched.pred_off();
    R.preds = sched.preds();
    sched.cross(R.npred_x, R.succ_off, R.succs);
}

template <class T>
void upload(DevBuf<T>& d, const std::vector<T>& h) {
    d.alloc(std::max<size_t>(h.size(), 1));
    if (!h.empty())
        UB_CUDA(cudaMemcpy(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
}

void build_schedule(uscg_tracer_s* t) {
    if (t->sched_built)
        return;
    const auto h0 = std::chrono::steady_clock::now();
    t->run = run_length(t->lines, t->volume != 0);
    // a run's index lists live in shared memory (4 groups per CTA): keep the
    // per-group lists under ~48 KiB
    while (t->run > 1 && size_t(t->run) * size_t(t->max_cells) * 4 > 48 * 1024) {
        int r = t->run - 1;
        while (r > 1 && t->lines % r != 0)
            --r;
        t->run = r;
    }
    t->runs_per_view = t->lines / t->run;
    t->n_runs = t->views * t->runs_per_view;
    const char* host = std::getenv("USCG_HOST_SCHEDULE");
    if (host && std::atoi(host)) {
        RunSchedule R;
        host_schedule(t, R);
        t->level_off = R.level_off;
        upload(t->d_order, R.order);
        upload(t->d_level_off, t->level_off);
        upload(t->d_pred_off, R.pred_off);
        upload(t->d_preds, R.preds);
        t->n_preds = R.preds.size();
        upload(t->d_npred_x, R.npred_x);
        upload(t->d_succ_off, R.succ_off);
        upload(t->d_succs, R.succs);
        t->n_succs = R.succs.size();
    } else {
        // edges, CSR lists, levels and order all on the device (schedule_gpu.cu)
        GpuSchedule G;
        G.alloc = [t](GpuSchedule::Array a, size_t n) -> uint32_t* {
            DevBuf<uint32_t>* d[] = {&t->d_order,  &t->d_level_off, &t->d_pred_off, &t->d_preds,
                                     &t->d_npred_x, &t->d_succ_off,  &t->d_succs};
            d[a]->alloc(n);
            return d[a]->p;
        };
        gpu_schedule_build(t->trace_args(), t->views, t->max_recs, t->max_cells, t->cells, t->cells_per_sweep,
                           uint32_t(t->run), uint32_t(t->runs_per_view), G, t->st());
        t->level_off = std::move(G.level_off);
        t->n_preds = G.n_preds;
        t->n_succs = G.n_succs;
        if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
            std::fprintf(stderr,
                         "schedule: %zu runs, %u levels, %llu preds, %llu succs; edges %.3f s, lists %.3f s, "
                         "levels %.3f s, order %.3f s\n",
                         size_t(t->n_runs), unsigned(t->level_off.size() - 1), (unsigned long long)G.n_preds,
                         (unsigned long long)G.n_succs, G.seconds[0], G.seconds[1], G.seconds[2], G.seconds[3]);
    }
    t->d_bar.alloc(2);
    t->sched_built = true;
    t->schedule_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
}

// The wave executor's inputs (mart_sweep.cu): every (view, line)'s traced
// index list, kept on the device, and per line the progress each other view
// must have reached before the line may run. In-sweep: the line's earlier
// toucher of each cell, if in another view (same-view order is the task's
// own). Cross-sweep: where the line is the first toucher of a cell in a
// sweep, the previous sweep's last toucher. A view's own previous-sweep task
// is awaited at task start, so same-view requirements are dropped; so is
// every requirement an earlier line of the view already implies (progress
// counters are monotone and a view's lines become ready in order).
constexpr uint64_t kWaveIdxBudget = uint64_t(1) << 27;  // traced entries: 2 x 1 GiB of device lists, host build ~3 GB

bool wave_fits(const uscg_tracer_s* t) {
    return !t->volume && t->cells_per_sweep > 0 && t->cells_per_sweep <= kWaveIdxBudget &&
           t->cells < (uint64_t(1) << 31);
}

// The host builder (USCG_HOST_WAVE=1; the reference for the device build's
// test): the traced lists copied back, then one pass in sweep order.
void build_wave_host(uscg_tracer_s* t, const std::vector<uint32_t>& pos, const uint32_t* d_idx) {
    const uint64_t units = t->units();
    const uint32_t L = uint32_t(t->lines);
    const uint64_t total = pos[units];
    std::vector<uint32_t> idx(std::max<uint64_t>(total, 1));
    UB_CUDA(cudaMemcpyAsync(idx.data(), d_idx, sizeof(uint32_t) * total, cudaMemcpyDeviceToHost, t->st()));
    UB_CUDA(cudaStreamSynchronize(t->st()));
    // entries: {cell | also in the previous line of the view << 31, position
    // in the next line of the view or 0xFFFF} (the executor's hand-overs)
    {
        constexpr uint32_t kNone = ~0u;
        std::vector<uint2> ent(std::max<uint64_t>(total, 1));
        std::vector<uint32_t> stamp(t->cells, kNone), where(t->cells);
        for (uint64_t u = 0; u < units; ++u) {
            for (uint32_t k = pos[u]; k < pos[u + 1]; ++k) {
                ent[k] = make_uint2(idx[k], 0xFFFFu);
                stamp[idx[k]] = uint32_t(u);
                where[idx[k]] = k - pos[u];
            }
            if (u % L == 0)
                continue;
            for (uint32_t k = pos[u - 1]; k < pos[u]; ++k) {
                const uint32_t c = idx[k];
                if (stamp[c] == uint32_t(u)) {
                    ent[k].y = where[c];
                    ent[pos[u] + where[c]].x |= 0x80000000u;
                }
            }
        }
        t->d_went.alloc(ent.size());
        UB_CUDA(cudaMemcpy(t->d_went.p, ent.data(), sizeof(uint2) * ent.size(), cudaMemcpyHostToDevice));
    }

    constexpr uint32_t NONE = ~0u;
    const uint32_t views = uint32_t(t->views);
    std::vector<uint32_t> last(t->cells, NONE), first(t->cells, NONE);
    std::vector<uint32_t> run_max[2] = {std::vector<uint32_t>(views, 0), std::vector<uint32_t>(views, 0)};
    std::vector<std::pair<uint32_t, uint32_t>> cand;  // (view, required lines) of one line
    auto condense = [&](int xs, std::vector<uint32_t>& out) {
        // keep, per view, the largest requirement; drop what an earlier line implies
        std::sort(cand.begin(), cand.end());
        for (size_t i = 0; i < cand.size(); ++i) {
            if (i + 1 < cand.size() && cand[i + 1].first == cand[i].first)
                continue;
            const uint32_t w = cand[i].first, need = cand[i].second;
            if (need > run_max[xs][w]) {
                run_max[xs][w] = need;
                out.push_back(w | (uint32_t(xs) << 31));
                out.push_back(need);
            }
        }
        cand.clear();
    };
    std::vector<std::vector<uint32_t>> in_deps(units);
    for (uint64_t u = 0; u < units; ++u) {
        const uint32_t v = uint32_t(u / L);
        if (u % L == 0)
            std::fill(run_max[0].begin(), run_max[0].end(), 0u);
        for (uint32_t k = pos[u]; k < pos[u + 1]; ++k) {
            const uint32_t c = idx[k];
            const uint32_t w = last[c];
            if (w == NONE)
                first[c] = uint32_t(u);
            else if (w / L != v)
                cand.emplace_back(w / L, w % L + 1);
            last[c] = uint32_t(u);
        }
        condense(0, in_deps[u]);
    }
    std::vector<uint32_t> dep_off(units + 1), deps;
    dep_off[0] = 0;
    for (uint64_t u = 0; u < units; ++u) {
        const uint32_t v = uint32_t(u / L);
        if (u % L == 0)
            std::fill(run_max[1].begin(), run_max[1].end(), 0u);
        for (uint32_t k = pos[u]; k < pos[u + 1]; ++k) {
            const uint32_t c = idx[k];
            if (first[c] == uint32_t(u) && last[c] / L != v)
                cand.emplace_back(last[c] / L, last[c] % L + 1);
        }
        deps.insert(deps.end(), in_deps[u].begin(), in_deps[u].end());
        condense(1, deps);
        dep_off[u + 1] = uint32_t(deps.size() / 2);
    }
    upload(t->d_wdep_off, dep_off);
    upload(t->d_wdeps, deps);
    t->wave_deps = deps.size() / 2;
}

void build_wave(uscg_tracer_s* t) {
    if (t->wave_built)
        return;
    const auto h0 = std::chrono::steady_clock::now();
    const uint64_t units = t->units();
    std::vector<uint32_t> pos(units + 1);
    pos[0] = 0;
    for (uint64_t u = 0; u < units; ++u)
        pos[u + 1] = pos[u] + t->h_cells[u];
    const uint64_t total = pos[units];
    upload(t->d_wpos, pos);
    DevBuf<uint32_t> d_idx;
    d_idx.alloc(std::max<uint64_t>(total, 1));
    launch_trace_dump(t->trace_args(), 0, uint32_t(units), t->max_recs, t->max_cells, t->d_wpos.p, d_idx.p, t->st());
    const char* host = std::getenv("USCG_HOST_WAVE");
    if ((host && std::atoi(host)) || !wave_build_supported(uint32_t(t->lines), uint32_t(t->views), t->cells)) {
        build_wave_host(t, pos, d_idx.p);
    } else {
        t->d_went.alloc(std::max<uint64_t>(total, 1));
        std::vector<uint32_t> dep_off, deps;
        gpu_wave_build(t->d_wpos.p, d_idx.p, total, uint32_t(units), uint32_t(t->lines), uint32_t(t->views),
                       t->cells, t->d_went.p, dep_off, deps, t->st());
        upload(t->d_wdep_off, dep_off);
        upload(t->d_wdeps, deps);
        t->wave_deps = deps.size() / 2;
    }
    t->wave_built = true;
    t->wave_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
    if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
        std::fprintf(stderr, "wave schedule: %llu traced entries, %llu requirements, %.3f s\n",
                     (unsigned long long)total, (unsigned long long)t->wave_deps, t->wave_seconds);
}

// The wave entries split by cell index mod `parts` for the clustered wave
// kernel (built on first use per cluster size).
void ensure_split(uscg_tracer_s* t, int parts) {
    if (t->wave_split_parts == parts)
        return;
    const uint64_t units = t->units(), total = t->cells_per_sweep;
    t->d_wsplit.alloc(std::max<uint64_t>(total, 1));
    t->d_wspos.alloc(size_t(parts) * (units + 1));
    t->wave_split_longest = gpu_wave_split(t->d_wpos.p, t->d_went.p, total, uint32_t(units), uint32_t(parts),
                                           t->d_wspos.p, t->d_wsplit.p, t->st());
    t->wave_split_parts = parts;
}

// The flow executor's one-problem lists (USCG_FLOW_LISTS=0 disables): the
// traced index list of every (view, line) in unit order, written by the trace
// kernel in batches of at most 2^27 cells (u32 positions within a batch), so
// the single-warp updaters copy a line instead of tracing it every sweep. Kept
// only when it takes at most half of the free device memory.
void build_lists(uscg_tracer_s* t) {
    if (t->lists_built || t->lists_off)
        return;
    if (const char* e = std::getenv("USCG_FLOW_LISTS"); e && !std::atoi(e)) {
        t->lists_off = true;
        return;
    }
    const auto h0 = std::chrono::steady_clock::now();
    const uint64_t units = t->units(), total = t->cells_per_sweep;
    size_t free_b = 0, total_b = 0;
    UB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (total == 0 || total * 4 + (units + 1) * 8 > free_b / 2) {
        t->lists_off = true;
        return;
    }
    std::vector<unsigned long long> lpos(units + 1);
    lpos[0] = 0;
    for (uint64_t u = 0; u < units; ++u)
        lpos[u + 1] = lpos[u] + t->h_cells[u];
    t->d_lpos.alloc(lpos.size());
    UB_CUDA(cudaMemcpy(t->d_lpos.p, lpos.data(), sizeof(unsigned long long) * lpos.size(), cudaMemcpyHostToDevice));
    t->d_lists.alloc(total);
    constexpr uint64_t kBatch = uint64_t(1) << 27;
    std::vector<uint32_t> pos;
    DevBuf<uint32_t> d_pos;
    uint64_t u0 = 0;
    while (u0 < units) {
        uint64_t u1 = u0 + 1;
        while (u1 < units && lpos[u1 + 1] - lpos[u0] <= kBatch)
            ++u1;
        pos.resize(size_t(u1 - u0) + 1);
        for (uint64_t u = u0; u <= u1; ++u)
            pos[size_t(u - u0)] = uint32_t(lpos[u] - lpos[u0]);
        d_pos.ensure(pos.size());
        UB_CUDA(cudaMemcpyAsync(d_pos.p, pos.data(), sizeof(uint32_t) * pos.size(), cudaMemcpyHostToDevice, t->st()));
        launch_trace_dump(t->trace_args(), uint32_t(u0), uint32_t(u1 - u0), t->max_recs, t->max_cells, d_pos.p,
                          t->d_lists.p + lpos[u0], t->st());
        UB_CUDA(cudaStreamSynchronize(t->st()));  // pos is reused
        u0 = u1;
    }
    t->lists_built = true;
    t->lists_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
    if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
        std::fprintf(stderr, "flow lists: %llu entries, %.3f s\n", (unsigned long long)total, t->lists_seconds);
}

// The level executor's schedule (mart_levels.cu): the line DAG (runs of one
// line) levelled on the device (schedule_gpu.cu); only the level-sorted order
// and the level offsets are kept.
void build_line_levels(uscg_tracer_s* t) {
    if (t->lv_built)
        return;
    const auto h0 = std::chrono::steady_clock::now();
    DevBuf<uint32_t> tmp[7];
    GpuSchedule G;
    G.alloc = [&](GpuSchedule::Array a, size_t n) -> uint32_t* {
        if (a == GpuSchedule::kOrder) {
            t->d_lv_order.alloc(n);
            return t->d_lv_order.p;
        }
        if (a == GpuSchedule::kLevelOff) {
            t->d_lv_off.alloc(n);
            return t->d_lv_off.p;
        }
        tmp[a].alloc(n);
        return tmp[a].p;
    };
    gpu_schedule_build(t->trace_args(), t->views, t->max_recs, t->max_cells, t->cells, t->cells_per_sweep, 1u,
                       uint32_t(t->lines), G, t->st());
    UB_CUDA(cudaStreamSynchronize(t->st()));
    t->lv_off = std::move(G.level_off);
    t->lv_built = true;
    t->lv_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
    if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
        std::fprintf(stderr, "line levels: %zu lines, %zu levels, %.3f s\n", size_t(t->units()),
                     t->lv_off.size() - 1, t->lv_seconds);
}

// The tile executor's schedule (mart_tile.cu): every line's ASAP level within
// a sweep (level = 1 + the largest level of an earlier line sharing a cell),
// lines sorted by level. Geometry only, built once per tracer from the traced
// lists; small problems only (tile_fits).
bool build_tile(uscg_tracer_s* t) {
    if (t->tile_built || t->tile_off)
        return t->tile_built;
    const uint64_t units = t->units(), total = t->cells_per_sweep;
    if (units >= (uint64_t(1) << 24) || total >= (uint64_t(1) << 32) ||
        !tile_fits(t->cells, int(units), 1)) {
        t->tile_off = true;
        return false;
    }
    build_lists(t);
    if (!t->lists_built) {
        t->tile_off = true;
        return false;
    }
    std::vector<unsigned long long> lpos(units + 1);
    std::vector<uint32_t> idx(std::max<uint64_t>(total, 1));
    UB_CUDA(cudaMemcpy(lpos.data(), t->d_lpos.p, sizeof(unsigned long long) * lpos.size(), cudaMemcpyDeviceToHost));
    UB_CUDA(cudaMemcpy(idx.data(), t->d_lists.p, sizeof(uint32_t) * total, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> last(t->cells, 0), level(units);
    uint32_t levels = 0;
    for (uint64_t u = 0; u < units; ++u) {
        uint32_t lev = 0;
        for (uint64_t k = lpos[u]; k < lpos[u + 1]; ++k)
            lev = std::max(lev, last[idx[k]]);
        ++lev;
        for (uint64_t k = lpos[u]; k < lpos[u + 1]; ++k)
            last[idx[k]] = lev;
        level[u] = lev - 1;
        levels = std::max(levels, lev);
    }
    if (!tile_fits(t->cells, int(units), int(levels))) {
        t->tile_off = true;
        return false;
    }
    std::vector<uint32_t> off(levels + 1, 0);
    for (uint64_t u = 0; u < units; ++u)
        ++off[level[u] + 1];
    for (uint32_t l = 0; l < levels; ++l)
        off[l + 1] += off[l];
    std::vector<uint4> meta(units);
    std::vector<uint32_t> fill(off.begin(), off.end() - 1);
    for (uint64_t u = 0; u < units; ++u)
        meta[fill[level[u]]++] = make_uint4(uint32_t(u), uint32_t(lpos[u]), uint32_t(lpos[u + 1] - lpos[u]), 0u);
    upload(t->d_tmeta, meta);
    upload(t->d_tlevel, off);
    t->tile_levels = int(levels);
    t->tile_built = true;
    return true;
}

}  // namespace

extern "C" {

const char* uscg_last_error(void) { return g_last_error.c_str(); }
const char* uscg_version(void) { return "uscg_b200 0.1 (sm_100a)"; }
uint64_t uscg_launch_count(void) { return g_launches.load(); }

int32_t uscg_problem_stride(int32_t problems) { return problems < 1 ? 0 : problem_stride(problems); }

uscg_status uscg_ctx_create(int32_t device, uscg_ctx* out) {
    return guarded([&] {
        need(out != nullptr, "null output");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw NoDevice("no CUDA device: the uscg_b200 path runs on sm_100 only (no CPU fallback)");
        }
        need(device >= 0 && device < n, "device index out of range");
        cudaDeviceProp prop;
        UB_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            throw NoDevice(std::string("device ") + prop.name + " is not sm_100 (Blackwell B200)");
        UB_CUDA(cudaSetDevice(device));
        auto* c = new uscg_ctx_s;
        c->device = device;
        cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            throw CudaError(cudaGetErrorString(e));
        }
        c->stream = c->own;
        *out = c;
    });
}

uscg_status uscg_ctx_destroy(uscg_ctx ctx) {
    return guarded([&] {
        if (!ctx)
            return;
        cudaSetDevice(ctx->device);
        if (ctx->resample || ctx->metrics) {
            cudaDeviceSynchronize();
            delete ctx->resample;
            delete ctx->metrics;
        }
        if (ctx->own)
            cudaStreamDestroy(ctx->own);
        delete ctx;
    });
}

uscg_status uscg_ctx_set_stream(uscg_ctx ctx, void* stream) {
    return guarded([&] {
        need(ctx != nullptr, "null context");
        bind(ctx);
        // work queued on the old stream (e.g. a cached resample map) is complete
        // before anything runs on the new one
        UB_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    });
}

uscg_status uscg_ctx_synchronize(uscg_ctx ctx) {
    return guarded([&] {
        bind(ctx);
        UB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

uscg_status uscg_first_view_rays(const uscg_scan* scan, double* src_out, double* det_out) {
    return guarded([&] {
        validate_scan(scan);
        need(src_out && det_out, "null output");
        first_view_rays(scan, src_out, det_out);
    });
}

uscg_status uscg_tracer_create(uscg_ctx ctx, const uscg_grid* grid, const uscg_scan* scan,
                               int32_t quarter_symmetry, uscg_tracer* out) {
    return guarded([&] {
        bind(ctx);
        need(out != nullptr, "null output");
        validate_scan(scan);
        validate_grid(grid);
        if (quarter_symmetry) {
            // precompute_first_view (tracer.cpp:42-44): the mirrored build is
            // bit-identical to the direct one, so only the validation differs
            const bool ok = scan->det_u % 2 == 1 && scan->det_v % 2 == 1 && scan->source[1] == 0 &&
                            scan->source[2] == 0 && scan->detector_center[1] == 0 &&
                            scan->detector_center[2] == 0;
            need(ok, "quarter symmetry requires odd detector counts with source and detector "
                     "center on the x axis");
        }
        const int lines = scan->det_u * scan->det_v;
        std::vector<double> src(size_t(lines) * 3), det(size_t(lines) * 3);
        first_view_rays(scan, src.data(), det.data());
        *out = build_from_rays(ctx, grid, lines, src.data(), det.data(), scan->views,
                               scan->view_angles_deg);
    });
}

uscg_status uscg_tracer_create_from_rays(uscg_ctx ctx, const uscg_grid* grid, int32_t lines,
                                         const double* src, const double* det, int32_t views,
                                         const double* view_angles_deg, uscg_tracer* out) {
    return guarded([&] {
        bind(ctx);
        need(out != nullptr, "null output");
        *out = build_from_rays(ctx, grid, lines, src, det, views, view_angles_deg);
    });
}

uscg_status uscg_tracer_import_cache(uscg_ctx ctx, const uscg_grid* grid, int32_t lines,
                                     const uint32_t* offsets, uint64_t records,
                                     const double* phi_a, const double* phi_b,
                                     const uint16_t* slice, const uint16_t* ring, int32_t views,
                                     const double* view_angles_deg, uscg_tracer* out) {
    return guarded([&] {
        bind(ctx);
        need(out != nullptr, "null output");
        validate_grid(grid);
        need(lines >= 1 && offsets, "line count must be >= 1");
        need(offsets[0] == 0 && offsets[lines] == records, "offsets do not match the record count");
        for (int l = 0; l < lines; ++l)
            need(offsets[l] <= offsets[l + 1], "offsets must be non-decreasing");
        std::unique_ptr<uscg_tracer_s> t(new uscg_tracer_s);
        t->ctx = ctx;
        t->device = ctx->device;
        fill_grid(t.get(), grid);
        fill_views(t.get(), views, view_angles_deg);
        t->lines = lines;
        t->records = records;
        std::vector<uint32_t> key(std::max<uint64_t>(records, 1));
        for (uint64_t i = 0; i < records; ++i) {
            need(ring[i] >= 1 && ring[i] <= t->n_rings, "record ring out of range");
            need(slice[i] < t->n_slices, "record slice out of range");
            key[i] = uint32_t(ring[i]) | (uint32_t(slice[i]) << kSliceShift);
        }
        std::vector<uint32_t> off(offsets, offsets + lines + 1);
        const size_t R = std::max<size_t>(records, 1);
        t->d_off.alloc(size_t(lines) + 1);
        t->d_pa.alloc(R);
        t->d_pb.alloc(R);
        t->d_key.alloc(R);
        UB_CUDA(cudaMemcpy(t->d_off.p, off.data(), sizeof(uint32_t) * off.size(),
                           cudaMemcpyHostToDevice));
        if (records) {
            UB_CUDA(cudaMemcpy(t->d_pa.p, phi_a, sizeof(double) * records, cudaMemcpyHostToDevice));
            UB_CUDA(cudaMemcpy(t->d_pb.p, phi_b, sizeof(double) * records, cudaMemcpyHostToDevice));
            UB_CUDA(cudaMemcpy(t->d_key.p, key.data(), sizeof(uint32_t) * records,
                               cudaMemcpyHostToDevice));
        }
        finish_tracer(t.get(), off);
        *out = t.release();
    });
}

uscg_status uscg_tracer_copy_cache(uscg_tracer t, uint32_t* offsets, double* phi_a, double* phi_b,
                                   uint32_t* keys, uint32_t flags) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        need(offsets && phi_a && phi_b && keys, "null buffer");
        const cudaMemcpyKind k = (flags & USCG_DEVICE_POINTERS) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        cudaStream_t st = t->st();
        UB_CUDA(cudaMemcpyAsync(offsets, t->d_off.p, sizeof(uint32_t) * (size_t(t->lines) + 1), k, st));
        if (t->records) {
            UB_CUDA(cudaMemcpyAsync(phi_a, t->d_pa.p, sizeof(double) * t->records, k, st));
            UB_CUDA(cudaMemcpyAsync(phi_b, t->d_pb.p, sizeof(double) * t->records, k, st));
            UB_CUDA(cudaMemcpyAsync(keys, t->d_key.p, sizeof(uint32_t) * t->records, k, st));
        }
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

uscg_status uscg_tracer_import_cache_keys(uscg_ctx ctx, const uscg_grid* grid, int32_t lines,
                                          const uint32_t* offsets, uint64_t records, const double* phi_a,
                                          const double* phi_b, const uint32_t* keys, int32_t views,
                                          const double* view_angles_deg, uint32_t flags, uscg_tracer* out) {
    return guarded([&] {
        bind(ctx);
        need(out != nullptr, "null output");
        validate_grid(grid);
        need(lines >= 1 && offsets, "line count must be >= 1");
        need(records < (1ull << 32), "record count must fit in 32 bits");
        const bool dev = flags & USCG_DEVICE_POINTERS;
        const cudaMemcpyKind k = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        std::vector<uint32_t> off(size_t(lines) + 1);
        UB_CUDA(cudaMemcpy(off.data(), offsets, sizeof(uint32_t) * off.size(),
                           dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
        need(off[0] == 0 && off[lines] == records, "offsets do not match the record count");
        for (int l = 0; l < lines; ++l)
            need(off[l] <= off[l + 1], "offsets must be non-decreasing");
        std::unique_ptr<uscg_tracer_s> t(new uscg_tracer_s);
        t->ctx = ctx;
        t->device = ctx->device;
        fill_grid(t.get(), grid);
        fill_views(t.get(), views, view_angles_deg);
        t->lines = lines;
        t->records = records;
        const size_t R = std::max<size_t>(records, 1);
        t->d_off.alloc(size_t(lines) + 1);
        t->d_pa.alloc(R);
        t->d_pb.alloc(R);
        t->d_key.alloc(R);
        UB_CUDA(cudaMemcpy(t->d_off.p, off.data(), sizeof(uint32_t) * off.size(), cudaMemcpyHostToDevice));
        if (records) {
            UB_CUDA(cudaMemcpy(t->d_pa.p, phi_a, sizeof(double) * records, k));
            UB_CUDA(cudaMemcpy(t->d_pb.p, phi_b, sizeof(double) * records, k));
            UB_CUDA(cudaMemcpy(t->d_key.p, keys, sizeof(uint32_t) * records, k));
            launch_clear_flags(t->d_key.p, records, t->st());
        }
        finish_tracer(t.get(), off);  // validates nothing further; annotate sets the dedup flags
        *out = t.release();
    });
}

uscg_status uscg_tracer_destroy(uscg_tracer tracer) {
    return guarded([&] {
        if (!tracer)
            return;
        cudaSetDevice(tracer->device);
        cudaDeviceSynchronize();
        delete tracer;
    });
}

uscg_status uscg_tracer_export_wave(uscg_tracer t, uint64_t* n_entries, uint64_t* n_deps, uint32_t* entries,
                                    uint32_t* dep_off, uint32_t* deps) {
    return guarded([&] {
        need(t && n_entries && n_deps, "null argument");
        bind(t->ctx);
        need(t->wave_built, "the wave executor's arrays are not built (run a 2D stack reconstruction first)");
        const uint64_t ne = t->cells_per_sweep, nd = t->wave_deps;
        *n_entries = ne;
        *n_deps = nd;
        if (entries && ne)
            UB_CUDA(cudaMemcpy(entries, t->d_went.p, sizeof(uint2) * ne, cudaMemcpyDeviceToHost));
        if (dep_off)
            UB_CUDA(cudaMemcpy(dep_off, t->d_wdep_off.p, sizeof(uint32_t) * (t->units() + 1), cudaMemcpyDeviceToHost));
        if (deps && nd)
            UB_CUDA(cudaMemcpy(deps, t->d_wdeps.p, sizeof(uint32_t) * 2 * nd, cudaMemcpyDeviceToHost));
    });
}

uscg_status uscg_tracer_get_info(uscg_tracer t, uscg_tracer_info* info) {
    return guarded([&] {
        need(t && info, "null argument");
        info->lines = t->lines;
        info->views = t->views;
        info->n_rings = t->n_rings;
        info->n_slices = t->n_slices;
        info->records = t->records;
        info->cells_per_slice = t->cps;
        info->cell_count = t->cells;
        info->cache_bytes = t->records * 20 + (uint64_t(t->lines) + 1) * 4;
        info->max_line_records = t->max_recs;
        info->max_line_cells = t->max_cells;
        info->cells_per_sweep = t->cells_per_sweep;
        info->chords_per_sweep = t->records * uint64_t(t->views);
        info->levels = t->executor == 5 && t->lv_built ? int32_t(t->lv_off.size()) - 1
                       : (t->sched_built ? int32_t(t->level_off.size()) - 1 : 0);
        info->generator_ms = t->generator_ms;
        info->executor = t->executor;
        info->wave_requirements = t->wave_deps;
        info->wave_build_s = t->wave_seconds;
        info->wave_ctas = t->wave_ctas;
        info->executor_bytes = t->d_lists.bytes() + t->d_lpos.bytes() + t->d_went.bytes() + t->d_wsplit.bytes() +
                               t->d_wpos.bytes() + t->d_wdep_off.bytes() + t->d_wdeps.bytes() +
                               t->d_order.bytes() + t->d_pred_off.bytes() + t->d_preds.bytes() +
                               t->d_succ_off.bytes() + t->d_succs.bytes() + t->d_npred_x.bytes() +
                               t->d_tmeta.bytes() + t->d_tlevel.bytes() + t->d_lv_order.bytes() + t->d_lv_off.bytes();
    });
}

uscg_status uscg_trace_checksums(uscg_tracer t, int32_t view0, int32_t nviews, uint32_t* counts,
                                 uint64_t* sums, uint32_t flags) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        need(counts && sums, "null buffer");
        need(view0 >= 0 && nviews >= 0 && int64_t(view0) + nviews <= t->views, "view range out of bounds");
        const uint64_t n = uint64_t(nviews) * uint64_t(t->lines);
        if (n == 0)
            return;
        auto* dsum = reinterpret_cast<unsigned long long*>(sums);
        if (flags & USCG_DEVICE_POINTERS) {
            launch_checksums(t->trace_args(), view0, nviews, t->n_rings, t->max_recs, counts, dsum, t->st());
            UB_CUDA(cudaStreamSynchronize(t->st()));
            return;
        }
        DevBuf<uint32_t> dc;
        DevBuf<unsigned long long> ds;
        dc.alloc(n);
        ds.alloc(n);
        launch_checksums(t->trace_args(), view0, nviews, t->n_rings, t->max_recs, dc.p, ds.p, t->st());
        UB_CUDA(cudaMemcpyAsync(counts, dc.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, t->st()));
        UB_CUDA(cudaMemcpyAsync(sums, ds.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, t->st()));
        UB_CUDA(cudaStreamSynchronize(t->st()));
    });
}

uscg_status uscg_tracer_export_cache(uscg_tracer t, uint32_t* offsets, double* phi_a,
                                     double* phi_b, uint16_t* slice, uint16_t* ring) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        std::vector<uint32_t> key(t->records);
        if (offsets)
            UB_CUDA(cudaMemcpy(offsets, t->d_off.p, sizeof(uint32_t) * (t->lines + 1),
                               cudaMemcpyDeviceToHost));
        if (t->records == 0)
            return;
        if (phi_a)
            UB_CUDA(cudaMemcpy(phi_a, t->d_pa.p, sizeof(double) * t->records, cudaMemcpyDeviceToHost));
        if (phi_b)
            UB_CUDA(cudaMemcpy(phi_b, t->d_pb.p, sizeof(double) * t->records, cudaMemcpyDeviceToHost));
        UB_CUDA(cudaMemcpy(key.data(), t->d_key.p, sizeof(uint32_t) * t->records,
                           cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < t->records; ++i) {
            if (ring)
                ring[i] = uint16_t(key[i] & kRingMask);
            if (slice)
                slice[i] = uint16_t((key[i] >> kSliceShift) & kSliceMask);
        }
    });
}

uscg_status uscg_trace_line(uscg_tracer t, int32_t line, double theta_deg, uint32_t* out,
                            int64_t cap, int64_t* count) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        need(line >= 0 && line < t->lines, "line index out of range");
        // rotation changes a chord's sector count by at most one
        const int max_cells = t->max_cells + t->max_recs + 1;
        DevBuf<uint32_t> d_out;
        d_out.alloc(size_t(max_cells) + 1);
        launch_trace_one(t->trace_args(), line, norm360(theta_deg), t->max_recs, max_cells,
                         d_out.p, d_out.p + max_cells, t->st());
        uint32_t n = 0;
        UB_CUDA(cudaMemcpyAsync(&n, d_out.p + max_cells, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                t->st()));
        UB_CUDA(cudaStreamSynchronize(t->st()));
        if (count)
            *count = n;
        const int64_t m = std::min<int64_t>(n, cap);
        if (m > 0 && out)
            UB_CUDA(cudaMemcpy(out, d_out.p, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost));
    });
}

uscg_status uscg_trace_counts(uscg_tracer t, uint32_t* cells_out) {
    return guarded([&] {
        need(t && cells_out, "null argument");
        std::memcpy(cells_out, t->h_cells.data(), sizeof(uint32_t) * t->h_cells.size());
    });
}

uscg_status uscg_tracer_export_schedule(uscg_tracer t, int32_t* run, uint32_t* runs, uint32_t* levels,
                                        uint64_t* n_preds, uint32_t* order, uint32_t* level_off,
                                        uint32_t* pred_off, uint32_t* preds, uint32_t* npred_x) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        build_schedule(t);
        if (run)
            *run = t->run;
        if (runs)
            *runs = uint32_t(t->n_runs);
        if (levels)
            *levels = uint32_t(t->level_off.size()) - 1;
        if (n_preds)
            *n_preds = t->n_preds;
        auto get = [&](uint32_t* dst, const DevBuf<uint32_t>& src, size_t n) {
            if (dst && n)
                UB_CUDA(cudaMemcpy(dst, src.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
        };
        get(order, t->d_order, size_t(t->n_runs));
        get(level_off, t->d_level_off, t->level_off.size());
        get(pred_off, t->d_pred_off, size_t(t->n_runs) + 1);
        get(preds, t->d_preds, t->n_preds);
        get(npred_x, t->d_npred_x, size_t(t->n_runs));
    });
}

uscg_status uscg_tracer_export_successors(uscg_tracer t, uint64_t* n_succs, uint32_t* succ_off, uint32_t* succs) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        build_schedule(t);
        if (n_succs)
            *n_succs = t->n_succs;
        if (succ_off)
            UB_CUDA(cudaMemcpy(succ_off, t->d_succ_off.p, sizeof(uint32_t) * (size_t(t->n_runs) + 1),
                               cudaMemcpyDeviceToHost));
        if (succs && t->n_succs)
            UB_CUDA(cudaMemcpy(succs, t->d_succs.p, sizeof(uint32_t) * t->n_succs, cudaMemcpyDeviceToHost));
    });
}

uscg_status uscg_tracer_build_schedule(uscg_tracer t) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        build_schedule(t);
    });
}

uscg_status uscg_project(uscg_tracer t, const float* field, int32_t problems, float* proj_out,
                         uint32_t flags) {
    return guarded([&] {
        need(t != nullptr, "null tracer");
        bind(t->ctx);
        need(problems >= 1, "problem count must be >= 1");
        need(field && proj_out, "null buffer");
        const int S = problems, Sp = problem_stride(S);
        const bool dev = flags & USCG_DEVICE_POINTERS;
        const bool inter = flags & USCG_LAYOUT_INTERLEAVED;
        const uint64_t units = t->units();
        cudaStream_t st = t->st();
        const float* d_field = nullptr;
        if (dev && (inter || S == 1)) {
            d_field = field;
        } else {
            t->w_field.ensure(t->cells * Sp);
            t->w_stage.ensure(std::max<uint64_t>(units * S, t->cells * S));
            if (inter) {
                UB_CUDA(cudaMemcpyAsync(t->w_field.p, field, sizeof(float) * t->cells * Sp,
                                        cudaMemcpyHostToDevice, st));
            } else if (S == 1) {
                UB_CUDA(cudaMemcpyAsync(t->w_field.p, field, sizeof(float) * t->cells,
                                        dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
            } else {
                const float* src = field;
                if (!dev) {
                    UB_CUDA(cudaMemcpyAsync(t->w_stage.p, field, sizeof(float) * t->cells * S,
                                            cudaMemcpyHostToDevice, st));
                    src = t->w_stage.p;
                }
                launch_to_interleaved(src, t->w_field.p, t->cells, S, Sp, 0.f, st);
            }
            d_field = t->w_field.p;
        }
        float* d_out = nullptr;
        const bool direct_out = dev && (inter || S == 1);
        if (direct_out) {
            d_out = proj_out;
        } else {
            t->w_proj.ensure(units * Sp);
            d_out = t->w_proj.p;
        }
        if (flags & USCG_MODEL_LENGTH) {
            need(t->d_rays.p != nullptr,
                 "the length-weighted model needs the tracer's rays (not available for an imported cache)");
            launch_project_length(t->dev_grid(), t->lines, t->views, t->d_rays.p, t->d_theta.p, d_field, Sp,
                                  d_out, st);
        } else if (Sp == 1 && t->lists_built) {
            // one problem whose traced lists the solver has built (volumes):
            // stream them instead of re-tracing every (view, line)
            launch_project_lists(t->d_lists.p, t->d_lpos.p, units, d_field, d_out, st);
        } else {
            launch_project(t->trace_args(), t->views, d_field, Sp, t->max_recs, t->max_cells, d_out, st);
        }
        if (!direct_out) {
            if (inter || S == 1) {
                UB_CUDA(cudaMemcpyAsync(proj_out, d_out, sizeof(float) * units * Sp,
                                        dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
            } else {
                float* dst = proj_out;
                if (!dev) {
                    t->w_stage.ensure(std::max<uint64_t>(units * S, t->cells * S));
                    dst = t->w_stage.p;
                }
                launch_from_interleaved(d_out, dst, units, S, Sp, st);
                if (!dev)
                    UB_CUDA(cudaMemcpyAsync(proj_out, dst, sizeof(float) * units * S,
                                            cudaMemcpyDeviceToHost, st));
            }
        }
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

// The body of uscg_reconstruct. after_launch (may be null) runs once, right
// after the first MART launch is enqueued: uscg_reconstruct_batch queues the
// previous stack's download there, behind this solve's small host reads.
static void reconstruct_body(uscg_tracer t, const float* proj, int32_t problems, const uscg_solver_config* cfg,
                      float* field_inout, int32_t from_init, uscg_report* reports, uint32_t flags,
                      const std::function<void()>* after_launch, std::function<void()>* finish_out = nullptr) {
    need(t != nullptr, "null tracer");
    bind(t->ctx);
    need(cfg != nullptr, "null config");
    need(proj && field_inout, "null buffer");
    need(problems >= 1, "problem count must be >= 1");
    // validate_config (solver.cpp:55-61)
    need(cfg->beta > 0 && cfg->beta < 2, "relaxation must lie in (0, 2)");
    need(cfg->f_init > 0, "initial field value must be positive");
    need(cfg->max_sweeps >= 1, "sweep budget must be >= 1");
    const int S = problems, Sp = problem_stride(S), P = chunk_width(S);
    const bool dev = flags & USCG_DEVICE_POINTERS;
    const bool inter = flags & USCG_LAYOUT_INTERLEAVED;
    const uint64_t units = t->units();
    const uint64_t cells = t->cells;
    cudaStream_t st = t->st();

    // ---- projections -> device [units][Sp] ----
    const float* d_proj = nullptr;
    if (dev && (inter || S == 1)) {
        d_proj = proj;
    } else {
        t->w_proj.ensure(units * Sp);
        if (inter || S == 1) {
            UB_CUDA(cudaMemcpyAsync(t->w_proj.p, proj, sizeof(float) * units * Sp,
                                    dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        } else {
            const float* src = proj;
            if (!dev) {
                t->w_stage.ensure(std::max<uint64_t>(units * S, cells * S));
                UB_CUDA(cudaMemcpyAsync(t->w_stage.p, proj, sizeof(float) * units * S,
                                        cudaMemcpyHostToDevice, st));
                src = t->w_stage.p;
            }
            launch_to_interleaved(src, t->w_proj.p, units, S, Sp, 0.f, st);
        }
        d_proj = t->w_proj.p;
    }

    // ---- ProjectionSet::validate + auto_p_floor + all-zero check ----
    t->w_stats.ensure(proj_stats_words(S));
    launch_proj_stats(d_proj, int(units), S, Sp, t->w_stats.p, st);
    std::vector<double> stats(size_t(4) * S);
    UB_CUDA(cudaMemcpyAsync(stats.data(), t->w_stats.p, sizeof(double) * 4 * S, cudaMemcpyDeviceToHost, st));

    // ---- field -> device [cells][Sp] ----
    float* d_field = nullptr;
    const bool direct_field = dev && (inter || S == 1);
    if (direct_field) {
        d_field = field_inout;
    } else {
        t->w_field.ensure(cells * Sp);
        d_field = t->w_field.p;
    }
    if (from_init) {
        if (!direct_field) {
            if (inter || S == 1) {
                UB_CUDA(cudaMemcpyAsync(d_field, field_inout, sizeof(float) * cells * Sp,
                                        dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                        st));
            } else {
                const float* src = field_inout;
                if (!dev) {
                    t->w_stage.ensure(std::max<uint64_t>(units * S, cells * S));
                    UB_CUDA(cudaMemcpyAsync(t->w_stage.p, field_inout, sizeof(float) * cells * S,
                                            cudaMemcpyHostToDevice, st));
                    src = t->w_stage.p;
                }
                launch_to_interleaved(src, d_field, cells, S, Sp, 1.f, st);
            }
        }
        t->w_tmp.ensure(1);
        UB_CUDA(cudaMemsetAsync(t->w_tmp.p, 0, sizeof(unsigned long long), st));
        launch_count_nonpositive(d_field, cells * Sp, t->w_tmp.p, st);
        unsigned long long bad = 0;
        UB_CUDA(cudaMemcpyAsync(&bad, t->w_tmp.p, sizeof(bad), cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
        need(bad == 0, "initial field must be strictly positive");
    } else {
        launch_fill(d_field, cells * Sp, float(cfg->f_init), st);
    }
    UB_CUDA(cudaStreamSynchronize(st));
    std::vector<double> p_floor(Sp, 1e-12);
    std::vector<uint8_t> active(Sp, 0);
    std::vector<int> all_zero(S, 0);
    for (int p = 0; p < S; ++p) {
        if (stats[4 * p + 3] > 0)
            throw InvalidArgument("projection data contains a non-finite or negative measurement");
        const double cnt = stats[4 * p + 0], sum = stats[4 * p + 1];
        p_floor[p] = cfg->p_floor > 0 ? cfg->p_floor : (cnt == 0 ? 1e-12 : 1e-12 * (sum / cnt));
        all_zero[p] = stats[4 * p + 2] == 0;
        active[p] = !all_zero[p];
    }

    const bool track = cfg->tolerance > 0;
    if (track || reports)
        ensure_crossed(t);

    // ---- per-problem updates per sweep (U counter) ----
    t->w_updates.ensure(Sp);
    UB_CUDA(cudaMemsetAsync(t->w_updates.p, 0, sizeof(unsigned long long) * Sp, st));
    launch_sweep_updates(d_proj, t->d_cells.p, int(units), S, Sp, t->w_updates.p, st);
    std::vector<unsigned long long> upd(Sp);
    UB_CUDA(cudaMemcpyAsync(upd.data(), t->w_updates.p, sizeof(unsigned long long) * Sp,
                            cudaMemcpyDeviceToHost, st));

    t->w_pfloor.ensure(Sp);
    t->w_active.ensure(Sp);
    t->w_clamps.ensure(Sp);
    UB_CUDA(cudaMemcpyAsync(t->w_pfloor.p, p_floor.data(), sizeof(double) * Sp,
                            cudaMemcpyHostToDevice, st));
    UB_CUDA(cudaMemcpyAsync(t->w_active.p, active.data(), Sp, cudaMemcpyHostToDevice, st));
    UB_CUDA(cudaMemsetAsync(t->w_clamps.p, 0, sizeof(unsigned long long) * Sp, st));

    MartArgs h;
    h.tr = t->trace_args();
    h.field = d_field;
    h.proj = d_proj;
    h.p_floor = t->w_pfloor.p;
    h.active = t->w_active.p;
    h.clamps = t->w_clamps.p;
    h.beta = cfg->beta;
    h.power = (flags & USCG_UPDATE_POWER) ? 1 : 0;
    h.Sp = Sp;
    h.nchunks = Sp / P;
    h.max_recs = t->max_recs;
    h.max_cells = t->max_cells;
    h.run = t->run;
    int exec_mode = mart_mode();
    // auto: the wave executor for stacks (P >= 4); the tile executor for one
    // problem that fits in one CTA's shared memory; else flow
    if ((exec_mode == -1 && P >= 4) || exec_mode == 3)
        exec_mode = wave_fits(t) && wave_supported(h) && wave_fits_smem(h, t->lines) ? 3 : 0;
    else if ((exec_mode == -1 || exec_mode == 4) && Sp == 1)
        // (a field within L2: the level executor's ~3.4 us per line level beats
        // the dataflow executor's ~6.5 us per run level, C3 4.3 vs 5.9 ms; a
        // larger field is bound by its scattered updates, where the dataflow
        // executor's persistent warps do better, C4 86 vs 100 ms)
        exec_mode = build_tile(t) ? 4 : (exec_mode == -1 && cells * sizeof(float) <= (96ull << 20) ? 5 : 0);
    else if (exec_mode == -1 || exec_mode == 4)
        exec_mode = 0;
    if (exec_mode == 5) {
        // the level executor: one problem whose traced lists fit in memory
        if (Sp == 1)
            build_lists(t);
        if (Sp != 1 || !t->lists_built)
            exec_mode = 0;
        else
            build_line_levels(t);
    }
    t->executor = exec_mode;
    if (exec_mode == 3) {
        build_wave(t);
        if (t->wave_chunks != h.nchunks) {
            const uint64_t n = uint64_t(t->views) * uint64_t(h.nchunks);
            // one counter per 128-byte line (kWavePad), per CTA of a
            // cluster (up to 4)
            t->d_wprog.alloc(128 * n);
            t->d_wnext.alloc(1);
            UB_CUDA(cudaMemsetAsync(t->d_wprog.p, 0, sizeof(unsigned) * 128 * n, st));
            t->wave_chunks = h.nchunks;
            t->wave_epoch = 0;
        }
    }
    if (exec_mode == 0) {
        // the run DAG of the dataflow executor (the wave and tile executors
        // build their own schedules)
        build_schedule(t);
        h.run = t->run;
    }
    if (exec_mode == 0 && P == 1)
        build_lists(t);  // once per geometry, outside the timed sweeps
    if (exec_mode == 0 && t->done_chunks != h.nchunks) {
        const uint64_t n = uint64_t(t->n_runs) * uint64_t(h.nchunks);
        t->d_done.alloc(n);
        UB_CUDA(cudaMemsetAsync(t->d_done.p, 0, sizeof(unsigned) * n, st));
        t->done_chunks = h.nchunks;
        t->epoch = 0;
    }
    std::vector<int> sweeps(S, 0), converged(S, 0);
    std::vector<std::vector<double>> resid(S);
    std::vector<uint32_t> lv_live_off;  // level executor: live lines per level of this call
    if (track)
        t->w_prev.ensure(cells * Sp), t->w_resid.ensure(Sp);
    int n_active = 0;
    for (int p = 0; p < S; ++p)
        n_active += active[p];
    cudaEvent_t e0, e1;
    UB_CUDA(cudaEventCreate(&e0));
    UB_CUDA(cudaEventCreate(&e1));
    UB_CUDA(cudaEventRecord(e0, st));
    for (int sweep = 0; sweep < cfg->max_sweeps && n_active > 0; ++sweep) {
        if (track)
            UB_CUDA(cudaMemcpyAsync(t->w_prev.p, d_field, sizeof(float) * cells * Sp,
                                    cudaMemcpyDeviceToDevice, st));
        int n_run = 1;
        if (exec_mode == 3) {
            n_run = track ? 1 : cfg->max_sweeps - sweep;
            WaveSchedule ws;
            ws.pos = t->d_wpos.p;
            ws.ent = t->d_went.p;
            ws.dep_off = t->d_wdep_off.p;
            ws.deps = t->d_wdeps.p;
            ws.parts = wave_cluster_size(h);
            if (ws.parts > 1)
                ensure_split(t, ws.parts);
            ws.spos = ws.parts > 1 && t->wave_split_longest <= 384 ? t->d_wspos.p : nullptr;
            t->wave_ctas = ws.spos && !std::getenv("USCG_SWEEP_PROFILE") ? ws.parts : 1;  // as launch_mart_wave picks
            ws.split = t->d_wsplit.p;
            ws.views = t->views;
            ws.lines = t->lines;
            // USCG_SWEEP_PROFILE=<file>: per task {start, end, ready-wait, gather, reduce, store, cta}
            static const char* prof_path = std::getenv("USCG_SWEEP_PROFILE");
            // then per line {published, requirements held} (single-CTA form)
            const size_t nt = size_t(t->views) * h.nchunks * n_run, rec = 8 + 2 * size_t(t->lines);
            DevBuf<unsigned long long> prof;
            if (prof_path) {
                prof.alloc(nt * rec);
                UB_CUDA(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * nt * rec, st));
            }
            launch_mart_wave(h, ws, t->d_wprog.p, t->d_wnext.p, t->wave_epoch, n_run, st, prof.p);
            t->wave_epoch += unsigned(n_run);
            if (prof_path) {
                std::vector<unsigned long long> hp(nt * rec);
                UB_CUDA(cudaMemcpyAsync(hp.data(), prof.p, sizeof(unsigned long long) * hp.size(),
                                        cudaMemcpyDeviceToHost, st));
                UB_CUDA(cudaStreamSynchronize(st));
                if (FILE* fp = std::fopen(prof_path, "wb")) {
                    std::fwrite(hp.data(), sizeof(unsigned long long), hp.size(), fp);
                    std::fclose(fp);
                }
            }
        } else if (exec_mode == 4) {
            n_run = track ? 1 : cfg->max_sweeps - sweep;
            TileSchedule ts;
            ts.meta = t->d_tmeta.p;
            ts.level_off = t->d_tlevel.p;
            ts.lists = t->d_lists.p;
            ts.units = int(units);
            ts.levels = t->tile_levels;
            launch_mart_tile(h, ts, cells, n_run, st);
        } else if (exec_mode == 5) {
            n_run = track ? 1 : cfg->max_sweeps - sweep;
            const uint32_t nl = uint32_t(t->lv_off.size()) - 1;
            LevelSchedule ls;
            ls.lists = t->d_lists.p;
            ls.lpos = t->d_lpos.p;
            if (sweep == 0) {
                // the lines with a non-zero measurement, level by level
                t->w_lv_flags.ensure(units);
                t->w_lv_pos.ensure(units + 1);
                t->w_lv_live.ensure(units);
                t->w_lv_live_off.ensure(nl + 1);
                launch_live_lines(t->d_lv_order.p, d_proj, uint32_t(units), t->d_lv_off.p, nl, t->w_lv_flags.p,
                                  t->w_lv_pos.p, t->w_lv_live.p, t->w_lv_live_off.p, st);
                lv_live_off.resize(nl + 1);
                UB_CUDA(cudaMemcpyAsync(lv_live_off.data(), t->w_lv_live_off.p, sizeof(uint32_t) * (nl + 1),
                                        cudaMemcpyDeviceToHost, st));
                UB_CUDA(cudaStreamSynchronize(st));
            }
            ls.live = t->w_lv_live.p;
            ls.live_off = lv_live_off;
            launch_mart_levels(h, ls, n_run, st, &t->lv_graph);
        } else if (exec_mode == 0) {
            // without a per-sweep residual every remaining sweep runs in one
            // launch, back to back (cross-sweep dependencies)
            n_run = track ? 1 : cfg->max_sweeps - sweep;
            // USCG_SWEEP_PROFILE=<file>: per-task stamps {grab, traced, ready, published}
            static const char* prof_path = std::getenv("USCG_SWEEP_PROFILE");
            const size_t nt = size_t(t->n_runs) * h.nchunks * n_run;
            DevBuf<unsigned long long> prof;
            if (prof_path)
                prof.alloc(nt * 16);
            if (prof_path)
                UB_CUDA(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * nt * 16, st));
            FlowSlab slab;
            {
                const char* e = std::getenv("USCG_SLAB_Q");
                slab.Q = int(std::min<uint64_t>(units, e ? std::max(64, std::atoi(e)) : 8192));
            }
            // [n][indices][u16 next positions] (mart_sweep.cu, flow_tracer_runs)
            slab.slot_words = (1 + t->max_cells + (t->max_cells + 1) / 2 + 31) & ~31;
            t->w_slab.ensure(size_t(slab.Q) * slab.slot_words);
            t->w_slab_ctl.ensure(size_t(slab.Q) * 2 + 1);
            slab.data = t->w_slab.p;
            slab.ready = t->w_slab_ctl.p;
            slab.used = t->w_slab_ctl.p + slab.Q;
            slab.tnext = t->w_slab_ctl.p + 2 * slab.Q;
            FlowSchedule fs;
            fs.order = t->d_order.p;
            fs.pred_off = t->d_pred_off.p;
            fs.succ_off = t->d_succ_off.p;
            fs.succs = t->d_succs.p;
            fs.npred_x = t->d_npred_x.p;
            fs.n_runs = t->n_runs;
            fs.run = t->run;
            fs.runs_per_view = t->runs_per_view;
            launch_mart_flow(h, fs, t->d_done.p, t->d_bar.p + 1, t->epoch + 1, n_run, t->n_rings,
                             slab, st, prof.p, t->lists_built ? t->d_lists.p : nullptr,
                             t->lists_built ? t->d_lpos.p : nullptr);
            t->epoch += unsigned(n_run);
            if (prof_path) {
                std::vector<unsigned long long> hp(nt * 16);
                UB_CUDA(cudaMemcpyAsync(hp.data(), prof.p, sizeof(unsigned long long) * hp.size(),
                                        cudaMemcpyDeviceToHost, st));
                UB_CUDA(cudaStreamSynchronize(st));
                if (FILE* fp = std::fopen(prof_path, "wb")) {
                    std::fwrite(hp.data(), sizeof(unsigned long long), hp.size(), fp);
                    std::fclose(fp);
                }
            }
        }
        if (after_launch) {
            (*after_launch)();
            after_launch = nullptr;
        }
        for (int p = 0; p < S; ++p)
            sweeps[p] += active[p] * n_run;
        sweep += n_run - 1;
        if (track) {
            UB_CUDA(cudaMemsetAsync(t->w_resid.p, 0, sizeof(unsigned int) * Sp, st));
            launch_residual(d_field, t->w_prev.p, t->d_crossed.p, cells, S, Sp, t->w_resid.p, st);
            std::vector<unsigned int> bits(Sp);
            UB_CUDA(cudaMemcpyAsync(bits.data(), t->w_resid.p, sizeof(unsigned int) * Sp,
                                    cudaMemcpyDeviceToHost, st));
            UB_CUDA(cudaStreamSynchronize(st));
            bool changed = false;
            for (int p = 0; p < S; ++p) {
                if (!active[p])
                    continue;
                float r;
                std::memcpy(&r, &bits[p], sizeof(r));
                resid[p].push_back(double(r));
                if (double(r) <= cfg->tolerance) {
                    converged[p] = 1;
                    active[p] = 0;
                    --n_active;
                    changed = true;
                }
            }
            if (changed)
                UB_CUDA(cudaMemcpyAsync(t->w_active.p, active.data(), Sp, cudaMemcpyHostToDevice,
                                        st));
        }
    }
    UB_CUDA(cudaEventRecord(e1, st));
    if (after_launch)  // no sweep ran
        (*after_launch)();

    // ---- field back ----
    if (!direct_field) {
        if (inter || S == 1) {
            UB_CUDA(cudaMemcpyAsync(field_inout, d_field, sizeof(float) * cells * Sp,
                                    dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        } else {
            float* dst = field_inout;
            if (!dev) {
                t->w_stage.ensure(std::max<uint64_t>(units * S, cells * S));
                dst = t->w_stage.p;
            }
            launch_from_interleaved(d_field, dst, cells, S, Sp, st);
            if (!dev)
                UB_CUDA(cudaMemcpyAsync(field_inout, dst, sizeof(float) * cells * S,
                                        cudaMemcpyDeviceToHost, st));
        }
    }
    // the rest waits for the solve: run now, or later by the caller
    // (uscg_reconstruct_batch starts the next stack's solve first). A copy
    // into pageable memory would block here until the solve ends, so the
    // clamp counters are read after the stream has drained.
    const unsigned long long* d_clamps = t->w_clamps.p;
    auto finish = [=]() {
    UB_CUDA(cudaStreamSynchronize(st));
    std::vector<unsigned long long> clamps(Sp);
    UB_CUDA(cudaMemcpyAsync(clamps.data(), d_clamps, sizeof(unsigned long long) * Sp, cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    UB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);

    if (reports) {
        std::vector<uint8_t> crossed;
        bool need_crossed = false;
        for (int p = 0; p < S; ++p)
            need_crossed |= reports[p].crossed != nullptr;
        if (need_crossed) {
            crossed.resize(cells);
            UB_CUDA(cudaMemcpy(crossed.data(), t->d_crossed.p, cells, cudaMemcpyDeviceToHost));
        }
        for (int p = 0; p < S; ++p) {
            uscg_report& r = reports[p];
            r.sweeps = sweeps[p];
            r.converged = converged[p];
            r.all_zero_data = all_zero[p];
            r.seconds = ms * 1e-3;
            r.factor_clamps = clamps[p];
            r.updates = uint64_t(upd[p]) * uint64_t(sweeps[p]);
            // zero-measurement lines are skipped in every sweep (solver.cpp:119-127)
            r.zero_measurement_skips = uint64_t(double(units) - stats[4 * p + 0]) * uint64_t(sweeps[p]);
            if (r.sweep_residuals)
                for (size_t i = 0; i < resid[p].size(); ++i)
                    r.sweep_residuals[i] = resid[p][i];
            if (r.crossed) {
                if (all_zero[p])
                    std::memset(r.crossed, 0, cells);
                else
                    std::memcpy(r.crossed, crossed.data(), cells);
            }
        }
    }
    };
    if (finish_out)
        *finish_out = finish;
    else
        finish();
}

uscg_status uscg_reconstruct(uscg_tracer t, const float* proj, int32_t problems,
                             const uscg_solver_config* cfg, float* field_inout, int32_t from_init,
                             uscg_report* reports, uint32_t flags) {
    return guarded([&] { reconstruct_body(t, proj, problems, cfg, field_inout, from_init, reports, flags, nullptr); });
}

// Batched reconstruction with copy/compute overlap. Device memory: two
// staging sets (the host layout of one stack: projections and field) and,
// for the [S][n] host layout, one interleaved working set that the solves
// use in turn. Per stack b (set k = b % 2):
//   copy-in stream : [wait: set k free] H2D proj/field -> in[k]      -> ev_in[b]
//   ctx stream     : [wait ev_in[b]] to_interleaved -> work           -> ev_used[b]
//                    uscg_reconstruct(work, device pointers)
//                    [wait: out[k] free] from_interleaved -> out[k]   -> ev_ready[b]
//   copy-out stream: [wait ev_ready[b]] D2H out[k] -> host            -> ev_out[b]
// With the interleaved host layout (or S == 1) the solve runs in place on
// in[k] and downloads from it, so in[k] is free only after ev_out[b].
// uscg_reconstruct_batch overlaps neighbouring stacks' solves when the wave
// executor runs them without residual tracking (USCG_BATCH_OVERLAP=0: one at
// a time)
static bool overlap_solves(uscg_tracer t, int S, const uscg_solver_config* cfg) {
    if (const char* e = std::getenv("USCG_BATCH_OVERLAP"); e && !std::atoi(e))
        return false;
    if (cfg == nullptr || cfg->tolerance > 0)
        return false;
    const int mode = mart_mode(), P = chunk_width(S), Sp = problem_stride(S);
    if (!(mode == 3 || (mode == -1 && P >= 4)))
        return false;
    MartArgs h{};
    h.Sp = Sp;
    h.nchunks = Sp / P;
    h.max_recs = t->max_recs;
    h.max_cells = t->max_cells;
    return wave_fits(t) && wave_supported(h) && wave_fits_smem(h, t->lines);
}

uscg_status uscg_reconstruct_batch(uscg_tracer t, int32_t batch, const float* const* proj, int32_t problems,
                                   const uscg_solver_config* cfg, float* const* field_inout, int32_t from_init,
                                   uscg_report* reports, uint32_t flags) {
    // events of one call (destroyed after both copy streams drained)
    struct Events {
        std::vector<cudaEvent_t> ev;
        cudaStream_t in, out;
        ~Events() {
            if (in)
                cudaStreamSynchronize(in);
            if (out)
                cudaStreamSynchronize(out);
            for (cudaEvent_t e : ev)
                cudaEventDestroy(e);
        }
        cudaEvent_t make() {
            cudaEvent_t e;
            UB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev.push_back(e);
            return e;
        }
    };
    return guarded([&] {
        need(t != nullptr, "null tracer");
        need(batch >= 0, "batch must be >= 0");
        need(batch == 0 || (proj && field_inout), "null buffer");
        need(!(flags & USCG_DEVICE_POINTERS), "uscg_reconstruct_batch takes host buffers");
        need(problems >= 1, "problem count must be >= 1");
        for (int b = 0; b < batch; ++b)
            need(proj[b] && field_inout[b], "null buffer");
        if (batch == 0)
            return;
        bind(t->ctx);
        const int S = problems, Sp = problem_stride(S);
        const bool inter = (flags & USCG_LAYOUT_INTERLEAVED) || S == 1;
        const uint64_t units = t->units(), cells = t->cells;
        const uint64_t pw = inter ? units * Sp : units * S;  // host-layout words per stack
        const uint64_t fw = inter ? cells * Sp : cells * S;
        cudaStream_t st = t->st();
        if (!t->copy_in)
            UB_CUDA(cudaStreamCreateWithFlags(&t->copy_in, cudaStreamNonBlocking));
        if (!t->copy_out)
            UB_CUDA(cudaStreamCreateWithFlags(&t->copy_out, cudaStreamNonBlocking));
        Events E{{}, t->copy_in, t->copy_out};
        DevBuf<float>* in = t->w_bin;
        DevBuf<float>* out = t->w_bout;
        // solve slots (and staging sets) in turn: USCG_BATCH_SLOTS, 2..4
        int NS = 2;
        if (const char* e = std::getenv("USCG_BATCH_SLOTS"))
            NS = std::max(2, std::min(4, std::atoi(e)));
        for (int k = 0; k < NS && k < batch; ++k) {
            in[k].ensure(pw + fw);
            if (!inter)
                out[k].ensure(fw);
        }
        if (!inter) {  // the solves' interleaved working set
            t->w_proj.ensure(units * Sp);
            t->w_field.ensure(cells * Sp);
        }
        std::vector<cudaEvent_t> ev_in(batch), ev_free(batch), ev_ready(batch), ev_out(batch);
        for (int b = 0; b < batch; ++b) {
            ev_in[b] = E.make();
            ev_free[b] = E.make();
            ev_ready[b] = E.make();
            ev_out[b] = E.make();
        }
        // earlier work on the context stream (e.g. the caller's) precedes the uploads
        cudaEvent_t start = E.make();
        UB_CUDA(cudaEventRecord(start, st));
        UB_CUDA(cudaStreamWaitEvent(t->copy_in, start, 0));
        auto upload = [&](int b) {
            const int k = b % NS;
            if (b >= NS)  // in[k] is free once stack b-NS no longer needs it
                UB_CUDA(cudaStreamWaitEvent(t->copy_in, ev_free[b - NS], 0));
            UB_CUDA(cudaMemcpyAsync(in[k].p, proj[b], sizeof(float) * pw, cudaMemcpyHostToDevice, t->copy_in));
            if (from_init)
                UB_CUDA(cudaMemcpyAsync(in[k].p + pw, field_inout[b], sizeof(float) * fw, cudaMemcpyHostToDevice,
                                        t->copy_in));
            UB_CUDA(cudaEventRecord(ev_in[b], t->copy_in));
        };
        // stack b-1's download is queued only once stack b's solve is launched:
        // the solve's small host reads (validation statistics) would otherwise
        // wait behind it on the copy engine, serializing download and solve
        int queued_down = 0;  // stacks [0, queued_down) have their download queued
        auto download = [&](int b) {
            queued_down = b + 1;
            UB_CUDA(cudaStreamWaitEvent(t->copy_out, ev_ready[b], 0));
            const float* src = inter ? in[b % NS].p + pw : out[b % NS].p;
            UB_CUDA(cudaMemcpyAsync(field_inout[b], src, sizeof(float) * fw, cudaMemcpyDeviceToHost,
                                    t->copy_out));
            UB_CUDA(cudaEventRecord(ev_out[b], t->copy_out));
            if (inter)  // the solve ran in place on in[k]: free after the download
                UB_CUDA(cudaEventRecord(ev_free[b], t->copy_out));
        };
        // overlapped solves (wave executor, no residual tracking): stack b+1's
        // solve is launched on the other solve slot before stack b's has
        // drained, so the wave's ramp and drain of neighbouring stacks overlap
        const bool overlap = batch > 1 && overlap_solves(t, S, cfg);
        std::vector<std::function<void()>> fin(batch);
        std::vector<char> fin_done(batch, 0);
        auto finish = [&](int b) {
            if (fin[b] && !fin_done[b]) {
                fin_done[b] = 1;
                fin[b]();
            }
        };
        cudaStream_t orig = t->ctx->stream;
        if (overlap)
            for (auto& sl : t->slots)
                if (!sl.st)
                    UB_CUDA(cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking));
        int failed = batch;  // the stack being solved when an error is thrown
        try {
        upload(0);
        for (int b = 0; b < batch; ++b) {
            failed = b;
            const int k = b % NS;
            if (overlap && b >= NS)
                finish(b - NS);  // stack b-NS (this slot's previous solve) finished

            struct SlotIn {  // the slot's workspaces and stream, swapped in for this solve
                uscg_tracer_s* t;
                uscg_tracer_s::SolveSlot* sl;
                cudaStream_t orig;
                SlotIn(uscg_tracer_s* tt, uscg_tracer_s::SolveSlot* s, cudaStream_t o) : t(tt), sl(s), orig(o) {
                    if (sl) {
                        t->swap_slot(*sl);
                        t->ctx->stream = sl->st;
                    }
                }
                ~SlotIn() {
                    if (sl) {
                        t->swap_slot(*sl);
                        t->ctx->stream = orig;
                    }
                }
            } slot_in(t, overlap ? &t->slots[k] : nullptr, orig);
            const cudaStream_t cur = t->st();
            UB_CUDA(cudaStreamWaitEvent(cur, ev_in[b], 0));
            float* d_proj = in[k].p;
            float* d_field = in[k].p + pw;
            if (!inter) {
                t->w_proj.ensure(units * Sp);
                t->w_field.ensure(cells * Sp);
                launch_to_interleaved(in[k].p, t->w_proj.p, units, S, Sp, 0.f, cur);
                if (from_init)
                    launch_to_interleaved(in[k].p + pw, t->w_field.p, cells, S, Sp, 1.f, cur);
                UB_CUDA(cudaEventRecord(ev_free[b], cur));
                d_proj = t->w_proj.p;
                d_field = t->w_field.p;
            }
            const std::function<void()> hook = [&] {
                if (b >= 1)
                    download(b - 1);
                if (b + 1 < batch)
                    upload(b + 1);  // overlaps this stack's solve
            };
            reconstruct_body(t, d_proj, S, cfg, d_field, from_init, reports ? reports + size_t(b) * S : nullptr,
                             USCG_DEVICE_POINTERS | USCG_LAYOUT_INTERLEAVED, &hook, overlap ? &fin[b] : nullptr);
            if (!inter) {
                if (b >= NS)  // out[k] is free once stack b-NS has been downloaded
                    UB_CUDA(cudaStreamWaitEvent(cur, ev_out[b - NS], 0));
                launch_from_interleaved(t->w_field.p, out[k].p, cells, S, Sp, cur);
            }
            UB_CUDA(cudaEventRecord(ev_ready[b], cur));
        }
        } catch (...) {
            // the stacks solved before the failing one still deliver their
            // fields and reports, and no copy or solve is left in flight
            try {
                for (int b = 0; b < failed; ++b)
                    finish(b);
                for (int b = queued_down; b < failed; ++b)
                    download(b);
                cudaStreamSynchronize(t->copy_out);
                cudaStreamSynchronize(t->copy_in);
                for (auto& sl : t->slots)
                    if (sl.st)
                        cudaStreamSynchronize(sl.st);
                cudaStreamSynchronize(st);
            } catch (...) {
            }
            throw;
        }
        if (overlap)
            for (int b = std::max(0, batch - NS); b < batch; ++b)
                finish(b);
        download(batch - 1);
        // the context stream ends after the last download (callers time on it)
        UB_CUDA(cudaStreamWaitEvent(st, ev_out[batch - 1], 0));
        UB_CUDA(cudaStreamSynchronize(t->copy_out));
        UB_CUDA(cudaStreamSynchronize(t->copy_in));
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

uscg_status uscg_resample(uscg_ctx ctx, const uscg_grid* grid, const float* field,
                          int32_t problems, int32_t npix, float* out, uint32_t flags) {
    return guarded([&] {
        bind(ctx);
        validate_grid(grid);
        need(field && out, "null buffer");
        need(problems >= 1, "problem count must be >= 1");
        need(npix >= 2 && npix % 2 == 0, "image size must be even");
        need(npix <= 65534, "image size must be at most 65534");
        const bool perm = grid->ring_counts == nullptr && npix == 2 * grid->n_rings;
        if (!ctx->resample)
            ctx->resample = new ResampleCache;
        ResampleCache& rc = *ctx->resample;
        if (!rc.matches(grid, npix)) {
            UB_CUDA(cudaStreamSynchronize(ctx->stream));  // the old map may still be in use
            rc.grid.reset(new uscg_tracer_s);
            rc.grid->ctx = ctx;
            fill_grid(rc.grid.get(), grid);
            if (!perm) {
                rc.map.alloc(size_t(npix) * npix);
                launch_bin_map(rc.grid->dev_grid(), npix, rc.map.p, ctx->stream);
            }
            rc.tiled = npix % 32 == 0;
            if (rc.tiled)
                build_resample_plan(rc, perm, npix, ctx->stream);
            rc.n_rings = grid->n_rings;
            rc.n_slices = grid->volume ? grid->n_slices : 1;
            rc.volume = grid->volume ? 1 : 0;
            rc.npix = npix;
            rc.ring_spacing = grid->ring_spacing;
            rc.slice_height = grid->slice_height;
            rc.counts.assign(grid->ring_counts ? grid->ring_counts : nullptr,
                             grid->ring_counts ? grid->ring_counts + grid->n_rings : nullptr);
        }
        const uscg_tracer_s* t = rc.grid.get();
        const int S = problems;
        const bool dev = flags & USCG_DEVICE_POINTERS;
        const bool inter = flags & USCG_LAYOUT_INTERLEAVED;
        const int Sp = inter ? problem_stride(S) : 0;
        const int slices = t->n_slices;
        const uint64_t in_n = t->cells * uint64_t(inter ? Sp : S);
        const uint64_t out_n = uint64_t(npix) * npix * slices * S;
        cudaStream_t st = ctx->stream;
        DevBuf<float> d_in, d_out;
        const float* fin = field;
        if (!dev) {
            d_in.alloc(in_n);
            UB_CUDA(cudaMemcpyAsync(d_in.p, field, sizeof(float) * in_n, cudaMemcpyHostToDevice, st));
            fin = d_in.p;
        }
        float* fout = out;
        if (!dev) {
            d_out.alloc(out_n);
            fout = d_out.p;
        }
        if (rc.tiled)
            launch_tiled_resample(fin, t->cps, slices, S, Sp, rc.toff.p, rc.tcells.p, rc.slot.p, npix, fout, st);
        else if (perm)
            launch_perm_resample(fin, t->cps, slices, S, Sp, npix, fout, st);
        else
            launch_map_resample(fin, t->cps, slices, S, Sp, rc.map.p, npix, fout, st);
        if (!dev)
            UB_CUDA(cudaMemcpyAsync(out, fout, sizeof(float) * out_n, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

uscg_status uscg_cartesian_to_field(uscg_ctx ctx, const uscg_grid* grid, const float* images, int32_t problems,
                                    int32_t npix, float* field_out, uint32_t flags) {
    return guarded([&] {
        bind(ctx);
        validate_grid(grid);  // spec.validate() (phantom.cpp:166)
        need(images && field_out, "null buffer");
        need(problems >= 1, "problem count must be >= 1");
        need(grid->ring_counts == nullptr,
             "cartesian_to_field needs the reference sector law (uspg_to_cg_map is defined for it only)");
        need(npix == 2 * grid->n_rings, "slice shape does not match the grid");  // phantom.cpp:174-175
        uscg_tracer_s g;
        g.ctx = ctx;
        fill_grid(&g, grid);
        const int S = problems;
        const bool dev = flags & USCG_DEVICE_POINTERS;
        const bool inter = flags & USCG_LAYOUT_INTERLEAVED;
        const int Sp = inter ? problem_stride(S) : 0;
        const int slices = g.n_slices;
        const uint64_t in_n = uint64_t(npix) * npix * slices * S;
        const uint64_t out_n = g.cells * uint64_t(inter ? Sp : S);
        cudaStream_t st = ctx->stream;
        DevBuf<float> d_in, d_out;
        const float* in = images;
        if (!dev) {
            d_in.alloc(in_n);
            UB_CUDA(cudaMemcpyAsync(d_in.p, images, sizeof(float) * in_n, cudaMemcpyHostToDevice, st));
            in = d_in.p;
        }
        float* out = field_out;
        if (!dev) {
            d_out.alloc(out_n);
            out = d_out.p;
        }
        if (inter && Sp > S)  // padded problems stay 0 (every cell of a real problem is written)
            UB_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * out_n, st));
        launch_cart_to_field(in, g.cps, slices, S, Sp, npix, out, st);
        if (!dev)
            UB_CUDA(cudaMemcpyAsync(field_out, out, sizeof(float) * out_n, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

uscg_status uscg_image_sharpness(uscg_ctx ctx, const float* image, int32_t slices, int32_t rows, int32_t cols,
                                 double* sharpness_out, uint32_t flags) {
    return guarded([&] {
        bind(ctx);
        need(image && sharpness_out, "null buffer");
        need(slices >= 1, "volume slice counts differ or are empty");
        need(rows >= 2 && cols >= 2, "sharpness needs at least a 2x2 image");  // metrics.cpp:139-140
        const uint64_t px = uint64_t(rows) * uint64_t(cols);
        const uint64_t n = px * uint64_t(slices);
        cudaStream_t st = ctx->stream;
        DevBuf<float> d_img;
        const float* a = image;
        if (!(flags & USCG_DEVICE_POINTERS)) {
            d_img.alloc(n);
            UB_CUDA(cudaMemcpyAsync(d_img.p, image, sizeof(float) * n, cudaMemcpyHostToDevice, st));
            a = d_img.p;
        }
        if (!ctx->metrics)
            ctx->metrics = new MetricsWork;
        MetricsWork& w = *ctx->metrics;
        w.part.ensure(size_t(slices) * size_t(metrics_blocks(px)));
        w.sout.ensure(size_t(slices));
        launch_sharpness(a, slices, rows, cols, w.part.p, w.sout.p, st);
        UB_CUDA(cudaMemcpyAsync(sharpness_out, w.sout.p, sizeof(double) * slices, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

uscg_status uscg_intensity_profile(const float* image, int32_t rows, int32_t cols, int32_t row, double* out) {
    return guarded([&] {
        need(image && out, "null buffer");
        need(rows >= 1 && cols >= 1, "empty image");
        need(row >= 0 && row < rows, "profile row out of range");  // metrics.cpp:155-156
        for (int32_t c = 0; c < cols; ++c)
            out[c] = double(image[size_t(row) * size_t(cols) + size_t(c)]);
    });
}

uscg_status uscg_image_metrics(uscg_ctx ctx, const float* ref, const float* test, int32_t slices,
                               int32_t rows, int32_t cols, int32_t shared_range,
                               double dynamic_range, double* mae_out, double* rmse_out,
                               double* ssim_out, uint32_t flags) {
    return guarded([&] {
        bind(ctx);
        need(ref && test, "null image");
        need(slices >= 1, "volume slice counts differ or are empty");  // metrics.cpp:165
        need(rows >= 1 && cols >= 1, "empty image");                     // metrics.cpp:16
        if (ssim_out)
            need(rows >= 8 && cols >= 8, "image smaller than the 8x8 ssim window");  // metrics.cpp:109
        const uint64_t px = uint64_t(rows) * uint64_t(cols);
        const uint64_t n = px * uint64_t(slices);
        cudaStream_t st = ctx->stream;
        DevBuf<float> d_ref, d_test;
        const float* a = ref;
        const float* b = test;
        if (!(flags & USCG_DEVICE_POINTERS)) {
            d_ref.alloc(n);
            d_test.alloc(n);
            UB_CUDA(cudaMemcpyAsync(d_ref.p, ref, sizeof(float) * n, cudaMemcpyHostToDevice, st));
            UB_CUDA(cudaMemcpyAsync(d_test.p, test, sizeof(float) * n, cudaMemcpyHostToDevice, st));
            a = d_ref.p;
            b = d_test.p;
        }
        if (!ctx->metrics)
            ctx->metrics = new MetricsWork;
        MetricsWork& w = *ctx->metrics;
        w.part.ensure(size_t(slices) * size_t(metrics_blocks(px)) * 4);
        w.mom.ensure(size_t(slices) * 4);
        launch_moments(a, b, slices, px, w.part.p, w.mom.p, st);
        std::vector<double> m(size_t(slices) * 4);
        UB_CUDA(cudaMemcpyAsync(m.data(), w.mom.p, sizeof(double) * m.size(), cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
        for (int s = 0; s < slices; ++s) {
            if (mae_out)
                mae_out[s] = m[4 * s + 2] / double(px);
            if (rmse_out)
                rmse_out[s] = std::sqrt(m[4 * s + 3] / double(px));
        }
        if (!ssim_out)
            return;
        // dynamic range: given, per reference slice, or over the whole stack
        double lo_all = m[0], hi_all = m[1];
        for (int s = 1; s < slices; ++s) {
            lo_all = std::min(lo_all, m[4 * s]);
            hi_all = std::max(hi_all, m[4 * s + 1]);
        }
        std::vector<double> c1c2(size_t(slices) * 2);
        for (int s = 0; s < slices; ++s) {
            double L = dynamic_range;
            if (!(L > 0)) {
                const double r = shared_range ? hi_all - lo_all : m[4 * s + 1] - m[4 * s];
                L = r > 0 ? r : 1.0;
            }
            c1c2[2 * s] = (0.01 * L) * (0.01 * L);
            c1c2[2 * s + 1] = (0.03 * L) * (0.03 * L);
        }
        w.c1c2.ensure(c1c2.size());
        w.spart.ensure(size_t(slices) * size_t(ssim_tiles(rows, cols)));
        w.sout.ensure(size_t(slices));
        UB_CUDA(cudaMemcpyAsync(w.c1c2.p, c1c2.data(), sizeof(double) * c1c2.size(), cudaMemcpyHostToDevice, st));
        launch_ssim(a, b, slices, rows, cols, w.c1c2.p, w.spart.p, w.sout.p, st);
        UB_CUDA(cudaMemcpyAsync(ssim_out, w.sout.p, sizeof(double) * slices, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

// ---- Cartesian comparator ------------------------------------------------------

struct uscg_csystem_s {
    uscg_ctx ctx = nullptr;
    DevCart C{};
    int lines = 0, views = 0, stored = 1;
    uint64_t voxels = 0, entries = 0;
    double precompute_ms = 0;
    DevBuf<double> d_rays, d_theta;
    DevBuf<uint32_t> d_off, d_idx, d_order, w_order;
    DevBuf<float> d_w, w_proj, w_field;
    DevBuf<unsigned long long> w_clamps;
    std::vector<uint32_t> level_off;
};

uscg_status uscg_cartesian_like(const uscg_grid* grid, uscg_cartesian* out) {
    return guarded([&] {
        validate_grid(grid);
        need(out != nullptr, "null output");
        const int n = 2 * grid->n_rings;
        const double radius = 0.5 * n * grid->ring_spacing;
        out->nx = out->ny = n;
        out->voxel = grid->ring_spacing;
        out->origin[0] = out->origin[1] = -radius;
        if (grid->volume) {
            out->nz = grid->n_slices;
            out->origin[2] = -0.5 * grid->n_slices * grid->slice_height;
        } else {
            out->nz = 1;
            out->origin[2] = -0.5 * grid->ring_spacing;
        }
    });
}

uscg_status uscg_csystem_create(uscg_ctx ctx, const uscg_cartesian* cart, const uscg_scan* scan,
                                int32_t stored, uscg_csystem* out) {
    return guarded([&] {
        bind(ctx);
        need(cart && scan && out, "null argument");
        need(cart->nx >= 1 && cart->ny >= 1 && cart->nz >= 1, "voxel counts must be >= 1");  // siddon.cpp:11-16
        need(cart->voxel > 0, "voxel size must be positive");
        validate_scan(scan);
        std::unique_ptr<uscg_csystem_s> s(new uscg_csystem_s);
        s->ctx = ctx;
        s->C = DevCart{cart->nx, cart->ny, cart->nz, cart->voxel, cart->origin[0], cart->origin[1], cart->origin[2]};
        s->voxels = uint64_t(cart->nx) * uint64_t(cart->ny) * uint64_t(cart->nz);
        need(s->voxels < (1ull << 32), "voxel count must fit in 32 bits");
        s->stored = stored ? 1 : 0;
        s->lines = scan->det_u * scan->det_v;
        s->views = scan->views;
        const uint64_t rows = uint64_t(s->lines) * uint64_t(s->views);
        need(rows < (1ull << 31), "views * lines must fit in 31 bits");
        std::vector<double> rays(size_t(s->lines) * 6);
        first_view_rays(scan, rays.data(), rays.data() + 3 * size_t(s->lines));
        std::vector<double> th(size_t(s->views));
        const double step = 360.0 / s->views;
        for (int v = 0; v < s->views; ++v)
            th[v] = norm360(scan->view_angles_deg ? scan->view_angles_deg[v] : v * step);
        cudaStream_t st = ctx->stream;
        s->d_rays.alloc(rays.size());
        s->d_theta.alloc(th.size());
        UB_CUDA(cudaMemcpyAsync(s->d_rays.p, rays.data(), sizeof(double) * rays.size(), cudaMemcpyHostToDevice, st));
        UB_CUDA(cudaMemcpyAsync(s->d_theta.p, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice, st));
        cudaEvent_t e0, e1;
        UB_CUDA(cudaEventCreate(&e0));
        UB_CUDA(cudaEventCreate(&e1));
        UB_CUDA(cudaEventRecord(e0, st));
        DevBuf<uint32_t> cnt;
        cnt.alloc(rows);
        launch_siddon_count(s->C, s->lines, s->views, s->d_rays.p, s->d_theta.p, cnt.p, st);
        s->d_off.alloc(rows + 1);
        launch_exclusive_scan_u32(cnt.p, s->d_off.p, int(rows), st);
        uint32_t total = 0;
        UB_CUDA(cudaMemcpyAsync(&total, s->d_off.p + rows, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
        s->entries = total;
        s->d_idx.alloc(std::max<uint64_t>(total, 1));
        s->d_w.alloc(std::max<uint64_t>(total, 1));
        launch_siddon_write(s->C, s->lines, s->views, s->d_rays.p, s->d_theta.p, s->d_off.p, s->d_idx.p, s->d_w.p, st);
        UB_CUDA(cudaEventRecord(e1, st));
        // the dependency schedule of the supports (host, schedule.h)
        std::vector<uint32_t> off(rows + 1), idx(total);
        UB_CUDA(cudaMemcpyAsync(off.data(), s->d_off.p, sizeof(uint32_t) * off.size(), cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaMemcpyAsync(idx.data(), s->d_idx.p, sizeof(uint32_t) * idx.size(), cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
        float ms = 0;
        UB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        s->precompute_ms = ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        AsapSchedule sched(s->voxels, uint32_t(s->lines), 1);
        sched.add(idx.data(), off.data(), uint32_t(rows));
        sched.done();
        std::vector<uint32_t> order;
        sched.finish(order, s->level_off);
        s->d_order.alloc(order.size());
        UB_CUDA(cudaMemcpyAsync(s->d_order.p, order.data(), sizeof(uint32_t) * order.size(), cudaMemcpyHostToDevice, st));
        UB_CUDA(cudaStreamSynchronize(st));
        if (!s->stored) {  // on the fly: only the schedule is kept
            s->d_idx.release();
            s->d_w.release();
        }
        *out = s.release();
    });
}

// The polar grid's own (voxel, chord length) system: the LengthWeighted
// model's pieces (phantom.cpp:213-269) of every (view, line) as CSR lists, a
// cell's pieces merged at its first position (a line may meet a cell on both
// sides of its closest approach; the binary tracer's stamp dedup,
// tracer.cpp:181-195, handles the same case), with the MART dependency
// schedule of those supports. The returned system runs weighted_update
// (siddon.cpp:141-154) on the USPG / USCG field through
// uscg_csystem_reconstruct, and uscg_csystem_export gives the lists.
uscg_status uscg_tracer_length_system(uscg_tracer t, uscg_csystem* out) {
    return guarded([&] {
        need(t && out, "null argument");
        bind(t->ctx);
        need(t->d_rays.p != nullptr,
             "the length-weighted model needs the tracer's rays (not available for an imported cache)");
        const uint64_t rows = t->units();
        need(rows < (1ull << 31), "views * lines must fit in 31 bits");
        need(t->cells < (1ull << 32), "cell count must fit in 32 bits");
        std::unique_ptr<uscg_csystem_s> s(new uscg_csystem_s);
        s->ctx = t->ctx;
        s->voxels = t->cells;
        s->stored = 1;
        s->lines = t->lines;
        s->views = t->views;
        cudaStream_t st = t->st();
        cudaEvent_t e0, e1;
        UB_CUDA(cudaEventCreate(&e0));
        UB_CUDA(cudaEventCreate(&e1));
        UB_CUDA(cudaEventRecord(e0, st));
        // pieces per line, then the pieces themselves
        DevBuf<uint32_t> cnt, roff, ridx;
        DevBuf<float> rlen;
        cnt.alloc(rows);
        launch_length_lists(t->dev_grid(), t->lines, t->views, t->d_rays.p, t->d_theta.p, nullptr, cnt.p, nullptr,
                            nullptr, st);
        std::vector<uint32_t> hc(rows);
        UB_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, sizeof(uint32_t) * rows, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
        std::vector<uint32_t> raw_off(rows + 1, 0);
        uint64_t raw = 0;
        for (uint64_t r = 0; r < rows; ++r) {
            raw_off[r] = uint32_t(raw);
            raw += hc[r];
            need(raw < (1ull << 32), "the (voxel, length) lists must hold fewer than 2^32 entries");
        }
        raw_off[rows] = uint32_t(raw);
        roff.alloc(rows + 1);
        ridx.alloc(std::max<uint64_t>(raw, 1));
        rlen.alloc(std::max<uint64_t>(raw, 1));
        UB_CUDA(cudaMemcpyAsync(roff.p, raw_off.data(), sizeof(uint32_t) * (rows + 1), cudaMemcpyHostToDevice, st));
        launch_length_lists(t->dev_grid(), t->lines, t->views, t->d_rays.p, t->d_theta.p, roff.p, nullptr, ridx.p,
                            rlen.p, st);
        UB_CUDA(cudaEventRecord(e1, st));
        std::vector<uint32_t> idx(raw);
        std::vector<float> len(raw);
        UB_CUDA(cudaMemcpyAsync(idx.data(), ridx.p, sizeof(uint32_t) * raw, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaMemcpyAsync(len.data(), rlen.p, sizeof(float) * raw, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
        float ms = 0;
        UB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        s->precompute_ms = ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        // a cell's pieces merged at its first position (in place: the merged
        // lists are never longer)
        std::vector<uint32_t> off(rows + 1), mark(t->cells, 0), where(t->cells, 0);
        std::vector<double> acc;
        uint64_t n = 0;
        for (uint64_t r = 0; r < rows; ++r) {
            const uint64_t begin = n;
            off[r] = uint32_t(n);
            acc.clear();
            for (uint64_t k = raw_off[r]; k < raw_off[r + 1]; ++k) {
                const uint32_t c = idx[k];
                if (mark[c] == uint32_t(r) + 1) {
                    acc[where[c]] += double(len[k]);
                    continue;
                }
                mark[c] = uint32_t(r) + 1;
                where[c] = uint32_t(n - begin);
                idx[n++] = c;
                acc.push_back(double(len[k]));
            }
            for (uint64_t k = begin; k < n; ++k)
                len[k] = float(acc[k - begin]);
        }
        off[rows] = uint32_t(n);
        s->entries = n;
        s->d_off.alloc(rows + 1);
        s->d_idx.alloc(std::max<uint64_t>(n, 1));
        s->d_w.alloc(std::max<uint64_t>(n, 1));
        UB_CUDA(cudaMemcpyAsync(s->d_off.p, off.data(), sizeof(uint32_t) * (rows + 1), cudaMemcpyHostToDevice, st));
        UB_CUDA(cudaMemcpyAsync(s->d_idx.p, idx.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
        UB_CUDA(cudaMemcpyAsync(s->d_w.p, len.data(), sizeof(float) * n, cudaMemcpyHostToDevice, st));
        // the dependency schedule of the supports (host, schedule.h)
        AsapSchedule sched(s->voxels, uint32_t(s->lines), 1);
        sched.add(idx.data(), off.data(), uint32_t(rows));
        sched.done();
        std::vector<uint32_t> order;
        sched.finish(order, s->level_off);
        s->d_order.alloc(std::max<size_t>(order.size(), 1));
        UB_CUDA(cudaMemcpyAsync(s->d_order.p, order.data(), sizeof(uint32_t) * order.size(), cudaMemcpyHostToDevice, st));
        UB_CUDA(cudaStreamSynchronize(st));
        *out = s.release();
    });
}

uscg_status uscg_csystem_info(uscg_csystem s, uint64_t* entries, uint64_t* device_bytes, int32_t* levels,
                              double* precompute_ms) {
    return guarded([&] {
        need(s != nullptr, "null system");
        if (entries)
            *entries = s->entries;
        if (device_bytes)  // offsets + (stored) voxel index + length per entry
            *device_bytes = sizeof(uint32_t) * (uint64_t(s->lines) * s->views + 1) +
                            (s->stored ? s->entries * (sizeof(uint32_t) + sizeof(float)) : 0);
        if (levels)
            *levels = int32_t(s->level_off.size()) - 1;
        if (precompute_ms)
            *precompute_ms = s->precompute_ms;
    });
}

uscg_status uscg_csystem_export(uscg_csystem s, uint32_t* offsets, uint32_t* idx, float* weight) {
    return guarded([&] {
        need(s != nullptr, "null system");
        need(s->stored, "an on-the-fly system keeps no coefficients");
        need(offsets && idx && weight, "null buffer");
        bind(s->ctx);
        cudaStream_t st = s->ctx->stream;
        const uint64_t rows = uint64_t(s->lines) * s->views;
        UB_CUDA(cudaMemcpyAsync(offsets, s->d_off.p, sizeof(uint32_t) * (rows + 1), cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaMemcpyAsync(idx, s->d_idx.p, sizeof(uint32_t) * s->entries, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaMemcpyAsync(weight, s->d_w.p, sizeof(float) * s->entries, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
    });
}

uscg_status uscg_csystem_reconstruct(uscg_csystem s, const float* proj, const uscg_solver_config* cfg,
                                     float* field_out, double* seconds, uint32_t flags) {
    return guarded([&] {
        need(s && proj && cfg && field_out, "null argument");
        bind(s->ctx);
        need(cfg->beta > 0 && cfg->beta < 2, "beta must lie in (0, 2)");  // validate_config
        need(cfg->f_init > 0, "f_init must be positive");
        need(cfg->max_sweeps >= 1, "max_sweeps must be >= 1");
        cudaStream_t st = s->ctx->stream;
        const uint64_t rows = uint64_t(s->lines) * s->views;
        const bool dev = flags & USCG_DEVICE_POINTERS;
        // p_floor (auto_p_floor, siddon.cpp:135-145) from the measurements
        std::vector<float> hp;
        const float* pp = proj;
        if (dev) {
            hp.resize(rows);
            UB_CUDA(cudaMemcpyAsync(hp.data(), proj, sizeof(float) * rows, cudaMemcpyDeviceToHost, st));
            UB_CUDA(cudaStreamSynchronize(st));
            pp = hp.data();
        }
        double sum = 0;
        uint64_t count = 0;
        for (uint64_t i = 0; i < rows; ++i) {
            need(std::isfinite(pp[i]) && pp[i] >= 0, "projection data must be finite and non-negative");
            if (pp[i] > 0) {
                sum += pp[i];
                ++count;
            }
        }
        const double p_floor = cfg->p_floor > 0 ? cfg->p_floor : (count == 0 ? 1e-12 : 1e-12 * (sum / count));
        const float* d_proj = proj;
        if (!dev) {
            s->w_proj.ensure(rows);
            UB_CUDA(cudaMemcpyAsync(s->w_proj.p, proj, sizeof(float) * rows, cudaMemcpyHostToDevice, st));
            d_proj = s->w_proj.p;
        }
        float* d_field = field_out;
        if (!dev) {
            s->w_field.ensure(s->voxels);
            d_field = s->w_field.p;
        }
        launch_fill(d_field, s->voxels, float(cfg->f_init), st);
        s->w_clamps.ensure(1);
        UB_CUDA(cudaMemsetAsync(s->w_clamps.p, 0, sizeof(unsigned long long), st));
        cudaEvent_t e0, e1;
        UB_CUDA(cudaEventCreate(&e0));
        UB_CUDA(cudaEventCreate(&e1));
        // the lines with a non-zero measurement, level by level (a zero
        // measurement is skipped, siddon.cpp:143: no block is launched for it)
        int levels = int(s->level_off.size()) - 1;
        std::vector<uint32_t> live_off(1, 0u);
        {
            std::vector<uint32_t> order(rows), live;
            UB_CUDA(cudaMemcpyAsync(order.data(), s->d_order.p, sizeof(uint32_t) * rows, cudaMemcpyDeviceToHost, st));
            UB_CUDA(cudaStreamSynchronize(st));
            live.reserve(rows);
            for (int l = 0; l < levels; ++l) {
                for (uint32_t k = s->level_off[l]; k < s->level_off[l + 1]; ++k)
                    if (pp[order[k]] > 0)
                        live.push_back(order[k]);
                if (live.size() > live_off.back())  // (a level without live lines is dropped)
                    live_off.push_back(uint32_t(live.size()));
            }
            s->w_order.ensure(std::max<size_t>(live.size(), 1));
            UB_CUDA(cudaMemcpyAsync(s->w_order.p, live.data(), sizeof(uint32_t) * live.size(), cudaMemcpyHostToDevice,
                                    st));
            UB_CUDA(cudaStreamSynchronize(st));  // `live` leaves scope
            levels = int(live_off.size()) - 1;
        }
        auto one_sweep = [&] {
            for (int l = 0; l < levels; ++l) {
                const uint32_t* units = s->w_order.p + live_off[l];
                const int n = int(live_off[l + 1] - live_off[l]);
                if (s->stored)
                    launch_csr_level(units, n, s->d_off.p, s->d_idx.p, s->d_w.p, d_proj, d_field, cfg->beta, p_floor,
                                     s->w_clamps.p, st);
                else
                    launch_otf_level(s->C, s->lines, s->d_rays.p, s->d_theta.p, units, n, d_proj, d_field, cfg->beta,
                                     p_floor, s->w_clamps.p, st);
            }
        };
        // a sweep is one launch per dependency level: captured once and
        // replayed per sweep (USCG_CSR_GRAPH=0: plain launches)
        const char* ge = std::getenv("USCG_CSR_GRAPH");
        const bool graph = cfg->max_sweeps >= 2 && levels >= 8 && !(ge && !std::atoi(ge));
        if (graph) {
            cudaGraph_t g = nullptr;
            cudaGraphExec_t exec = nullptr;
            UB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                one_sweep();
            } catch (...) {
                cudaStreamEndCapture(st, &g);
                if (g)
                    cudaGraphDestroy(g);
                throw;
            }
            UB_CUDA(cudaStreamEndCapture(st, &g));
            const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
            if (ie != cudaSuccess) {
                cudaGraphDestroy(g);
                UB_CUDA(ie);
            }
            UB_CUDA(cudaEventRecord(e0, st));  // (the sweeps: capture and instantiation are host-side set-up)
            for (int sweep = 0; sweep < cfg->max_sweeps; ++sweep)
                UB_CUDA(cudaGraphLaunch(exec, st));
            UB_CUDA(cudaEventRecord(e1, st));
            count_launch(uint64_t(levels) * uint64_t(cfg->max_sweeps - 1));  // (the capture counted one sweep)
            UB_CUDA(cudaStreamSynchronize(st));
            cudaGraphExecDestroy(exec);
            cudaGraphDestroy(g);
        } else {
            UB_CUDA(cudaEventRecord(e0, st));
            for (int sweep = 0; sweep < cfg->max_sweeps; ++sweep)
                one_sweep();
            UB_CUDA(cudaEventRecord(e1, st));
        }
        UB_CUDA(cudaGetLastError());
        if (!dev)
            UB_CUDA(cudaMemcpyAsync(field_out, d_field, sizeof(float) * s->voxels, cudaMemcpyDeviceToHost, st));
        UB_CUDA(cudaStreamSynchronize(st));
        float ms = 0;
        UB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (seconds)
            *seconds = ms * 1e-3;
    });
}

uscg_status uscg_csystem_destroy(uscg_csystem s) {
    return guarded([&] {
        if (!s)
            return;
        cudaSetDevice(s->ctx->device);
        cudaDeviceSynchronize();
        delete s;
    });
}

uscg_status uscg_uspg_to_cg_map(uscg_ctx ctx, int32_t n, uint32_t* out) {
    return guarded([&] {
        bind(ctx);
        if (n < 2 || n % 2 != 0)  // grid.cpp:76-77
            throw DomainError("image size must be even, got " + std::to_string(n));
        need(out != nullptr, "null output");
        DevBuf<uint32_t> d;
        d.alloc(size_t(n) * n);
        launch_cg_map(n, d.p, ctx->stream);
        UB_CUDA(cudaMemcpyAsync(out, d.p, sizeof(uint32_t) * n * n, cudaMemcpyDeviceToHost,
                                ctx->stream));
        UB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

uscg_status uscg_diag_math(uscg_ctx ctx, int32_t n, const double* x, const double* y, double* out) {
    return guarded([&] {
        bind(ctx);
        need(n >= 0 && x && y && out, "null buffer");
        if (n == 0)
            return;
        DevBuf<double> d;
        d.alloc(size_t(n) * 6);
        UB_CUDA(cudaMemcpyAsync(d.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        UB_CUDA(cudaMemcpyAsync(d.p + n, y, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        DevBuf<double> o;
        o.alloc(size_t(n) * 5);
        launch_diag_math(n, d.p, d.p + n, o.p, ctx->stream);
        UB_CUDA(cudaMemcpyAsync(out, o.p, sizeof(double) * 5 * n, cudaMemcpyDeviceToHost, ctx->stream));
        UB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"

extern "C" uscg_status uscg_schedule_build(uint32_t units, uint32_t lines_per_view, uint32_t run,
                                           const uint32_t* pos, const uint32_t* idx,
                                           uint64_t cell_count, uint32_t* order,
                                           uint32_t* level_off, uint32_t* levels,
                                           uint32_t* pred_off, uint32_t* preds, uint64_t* n_preds,
                                           uint32_t* npred_x) {
    return guarded([&] {
        need(pos && idx && order && level_off && levels, "null buffer");
        need(lines_per_view >= 1 && run >= 1 && lines_per_view % run == 0 &&
                 units % lines_per_view == 0,
             "runs must tile the views");
        for (uint32_t u = 0; u < units; ++u)
            need(pos[u] <= pos[u + 1], "support offsets must be non-decreasing");
        for (uint32_t i = 0; i < pos[units]; ++i)
            need(idx[i] < cell_count, "support cell out of range");
        AsapSchedule s(cell_count, lines_per_view, run);
        std::vector<uint32_t> rel(pos, pos + units + 1);
        for (auto& p : rel)
            p -= pos[0];
        s.add(idx + pos[0], rel.data(), units);
        s.done();
        std::vector<uint32_t> ord, loff;
        s.finish(ord, loff);
        std::memcpy(order, ord.data(), sizeof(uint32_t) * ord.size());
        std::memcpy(level_off, loff.data(), sizeof(uint32_t) * loff.size());
        *levels = s.levels();
        if (pred_off)
            std::memcpy(pred_off, s.pred_off().data(), sizeof(uint32_t) * s.pred_off().size());
        if (preds)
            std::memcpy(preds, s.preds().data(), sizeof(uint32_t) * s.preds().size());
        if (n_preds)
            *n_preds = s.preds().size();
        if (npred_x) {
            std::vector<uint32_t> nx, so, sa;
            s.cross(nx, so, sa);
            std::memcpy(npred_x, nx.data(), sizeof(uint32_t) * nx.size());
        }
    });
}
