// Host-callable launch wrappers for the uscg_b200 kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <vector>

#include "internal.cuh"

namespace ub {

struct MartArgs {
    TraceArgs tr;
    float* field;                 // [cells][Sp]
    const float* proj;            // [units][Sp]
    const double* p_floor;        // [Sp]
    const uint8_t* active;        // [Sp]
    unsigned long long* clamps;   // [Sp]
    double beta;
    int Sp;
    int nchunks;
    int max_recs;
    int max_cells;
    int run = 1;  // lines per dataflow task: shared memory holds `run` index lists per group
    int power = 0;  // USCG_UPDATE_POWER: multiplicative form (m/p)^beta instead of solver.cpp:41
};

// The line's multiplicative correction from ratio = m / max(p, p_floor).
// Linear (the reference, proj/src/solver.cpp:41): 1 - beta (1 - ratio).
// Power (USCG_UPDATE_POWER; the multiplicative MART form x *= (m/p)^(beta a/max a)
// with binary coefficients, a = max a = 1): ratio^beta; a non-positive ratio
// gives 0, which the callers clamp to p_floor like the reference's
// non-positive linear factor (solver.cpp:42-45).
__device__ __forceinline__ double mart_factor(double ratio, double beta, int power) {
    if (power)
        return ratio > 0 ? pow(ratio, beta) : 0.0;
    return 1.0 - beta * (1.0 - ratio);
}

// problem-chunk width P for S problems (power of two <= 32)
int chunk_limit();
int chunk_width(int problems);
int problem_stride(int problems);
int stride_chunk(int Sp);

// K1: first-view generator. rays: lines*3 src + lines*3 det (device).
void launch_generate_count(const DevGrid& g, int lines, const double* src, const double* det,
                           uint32_t* counts, cudaStream_t st);
void launch_generate_write(const DevGrid& g, int lines, const double* src, const double* det,
                           const uint32_t* off, double* pa, double* pb, uint32_t* key,
                           cudaStream_t st);
// one-pass form: per-ray record bound, bounded slots (true counts, overflow
// flag), compaction into the packed store
void launch_generate_bound(const DevGrid& g, int lines, const double* src, const double* det, uint32_t* bound,
                           cudaStream_t st);
void launch_generate_slots(const DevGrid& g, int lines, const double* src, const double* det, const uint32_t* boff,
                           double* pa, double* pb, uint32_t* key, uint32_t* counts, unsigned* overflow,
                           cudaStream_t st);
void launch_compact_records(int lines, const uint32_t* boff, const uint32_t* off, const double* spa,
                            const double* spb, const uint32_t* skey, double* pa, double* pb, uint32_t* key,
                            cudaStream_t st);
void launch_annotate(int lines, const uint32_t* off, const double* pa, const double* pb,
                     uint32_t* key, const RingRow* rings, cudaStream_t st);
// drop the dedup flags of imported keys (annotate sets them again)
void launch_clear_flags(uint32_t* key, uint64_t n, cudaStream_t st);
void launch_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int n, cudaStream_t st);

// traces
void launch_trace_one(const TraceArgs& A, int line, double theta, int max_recs, int max_cells,
                      uint32_t* out, uint32_t* count, cudaStream_t st);
void launch_trace_counts(const TraceArgs& A, int views, int max_recs, uint32_t* cells,
                         cudaStream_t st);
// rotated reuse: |active| and the u64 sum of the active cells of every line
// of views [view0, view0 + nviews)
void launch_checksums(const TraceArgs& A, int view0, int nviews, int n_rings, int max_recs,
                      uint32_t* counts, unsigned long long* sums, cudaStream_t st);
void launch_trace_dump(const TraceArgs& A, uint32_t unit0, uint32_t units, int max_recs,
                       int max_cells, const uint32_t* pos, uint32_t* out, cudaStream_t st);
void launch_crossed(const TraceArgs& A, int views, int max_recs, int max_cells, uint8_t* crossed,
                    cudaStream_t st);

// K2' length-weighted projector (fp64 geometry and sums): rays = first-view
// [src lines*3][det lines*3] (device), field [cells][Sp], out [views*lines][Sp]
void launch_project_length(const DevGrid& g, int lines, int views, const double* rays,
                           const double* theta, const float* field, int Sp, float* out,
                           cudaStream_t st);

// The LengthWeighted model's pieces per (view, line) as (cell, length) pairs:
// off == nullptr: counts[unit] = pieces of the line; else written at off[unit]
void launch_length_lists(const DevGrid& g, int lines, int views, const double* rays, const double* theta,
                         const uint32_t* off, uint32_t* counts, uint32_t* idx, float* len, cudaStream_t st);

// K2 for one problem from precomputed traced lists (lists[lpos[u], lpos[u+1])): out [units]
void launch_project_lists(const uint32_t* lists, const unsigned long long* lpos, uint64_t units, const float* field,
                          float* out, cudaStream_t st);

// K2 projector: out [units][Sp]
void launch_project(const TraceArgs& A, int views, const float* field, int Sp, int max_recs,
                    int max_cells, float* out, cudaStream_t st);

// K3 for one small problem (mart_tile.cu): one CTA, the field in shared
// memory, the lines of each ASAP level in parallel (one warp per line), a
// block barrier between levels.
struct TileSchedule {
    const uint4* meta;         // [units] in level order: {unit, list offset, cells, 0}
    const uint32_t* level_off; // [levels + 1] slots per level (one sweep)
    const uint32_t* lists;     // traced index lists (offsets below 2^32)
    int units;
    int levels;
};
size_t tile_smem_bytes(uint64_t cells, int units, int levels);
bool tile_fits(uint64_t cells, int units, int levels);
void launch_mart_tile(const MartArgs& h, const TileSchedule& ts, uint64_t cells, int sweeps, cudaStream_t st);

// K3 level executor (mart_levels.cu; one problem): a kernel per ASAP level of
// the line DAG, a 64-thread block per line with a non-zero measurement, levels
// chained by programmatic dependent launch, a sweep replayed from a CUDA graph.
struct LevelSchedule {
    const uint32_t* lists;             // traced index lists
    const unsigned long long* lpos;    // [units + 1]
    const uint32_t* live;              // live lines (non-zero measurement) in level order (device)
    std::vector<uint32_t> live_off;    // [levels + 1] into `live` (host)
};
// order: every line sorted by level (device), level_off_dev [levels + 1];
// writes flags / pos (units + 1) scratch, the compacted `live` lines and
// live_off_dev [levels + 1]
void launch_live_lines(const uint32_t* order, const float* proj, uint32_t units, const uint32_t* level_off_dev,
                       uint32_t levels, uint32_t* flags, uint32_t* pos, uint32_t* live, uint32_t* live_off_dev,
                       cudaStream_t st);
// One sweep's level launches as an instantiated CUDA graph, kept by the tracer
// between calls: replayed while the same buffers, parameters and live lines
// come back (instantiation costs ~5 us a node, so a graph is built for 16
// sweeps or more, or when a call repeats the previous call's key).
struct LevelGraphCache {
    struct Key {
        const void *field = nullptr, *proj = nullptr, *p_floor = nullptr, *clamps = nullptr, *lists = nullptr,
                   *lpos = nullptr, *live = nullptr;
        double beta = 0;
        int power = 0, threads = 0, pdl = 0;
        std::vector<uint32_t> live_off;
        bool operator==(const Key& o) const {
            return field == o.field && proj == o.proj && p_floor == o.p_floor && clamps == o.clamps &&
                   lists == o.lists && lpos == o.lpos && live == o.live && beta == o.beta && power == o.power &&
                   threads == o.threads && pdl == o.pdl && live_off == o.live_off;
        }
    };
    cudaGraphExec_t exec = nullptr;
    Key key;        // of `exec`
    Key seen;       // of the last call that ran without a graph
    bool have_seen = false;
    void reset();   // destroys the graph (the caller has drained the stream)
    ~LevelGraphCache() { reset(); }
};
void launch_mart_levels(const MartArgs& h, const LevelSchedule& ls, int sweeps, cudaStream_t st,
                        LevelGraphCache* cache = nullptr);

// Ring of traced index lists shared by the chunk tasks of a unit:
// slot = [n, idx[0..n)], slot_words >= max_cells + 1.
struct FlowSlab {
    uint32_t* data;     // [Q * slot_words]
    unsigned* ready;    // [Q]
    unsigned* used;     // [Q]
    unsigned* tnext;    // tracer queue head
    int Q;
    int slot_words;
};

// K3 dataflow: tasks wait only on their predecessors (dependency counters)
// The run-granular dependency schedule on the device (schedule.h)
struct FlowSchedule {
    const uint32_t* order;     // runs in topological order
    const uint32_t* pred_off;  // runs + 1
    const uint32_t* succ_off;  // runs + 1 (in- and cross-sweep successors)
    const uint32_t* succs;
    const uint32_t* npred_x;   // runs
    int n_runs;
    int run;                   // lines per run
    int runs_per_view;
};

// Runs `sweeps` sweeps back to back (cross-sweep dependencies, no boundary);
// epoch = global 1-based index of the first of them.
// lists/lpos (optional, one-problem runs): every (view, line)'s traced list
// at lists[lpos[u], lpos[u+1]) instead of tracing each line every sweep
void launch_mart_flow(const MartArgs& h, const FlowSchedule& fs, unsigned* count, unsigned* next,
                      unsigned epoch, int sweeps, int n_rings, const FlowSlab& slab,
                      cudaStream_t st, unsigned long long* prof = nullptr, const uint32_t* lists = nullptr,
                      const unsigned long long* lpos = nullptr);

// K3 wave executor (2D problem stacks, mart_sweep.cu): one task per (sweep,
// view, problem chunk) updates the view's lines in order; other views are
// ordered by per-(view, chunk) progress counters.
struct WaveSchedule {
    const uint32_t* pos;      // [units + 1] offsets into ent
    const uint2* ent;         // every (view, line)'s traced list: {cell | in previous line << 31,
                              //  position in the next line of the view (0xFFFF: none)}
    const uint32_t* dep_off;  // [units + 1]
    const uint32_t* deps;     // pairs {view | cross-sweep << 31, required lines of that view}
    const uint32_t* spos;     // [parts][units + 1]: entries split by cell index mod parts (clustered
    const uint2* split;       //   wave kernel), or null
    int parts;                // CTAs per cluster of the split (2 or 4)
    int views;
    int lines;
};
// entries split by cell index mod parts (clustered wave kernel): spos
// [parts][units + 1] offsets into split; returns the longest per-part line
uint32_t gpu_wave_split(const uint32_t* pos, const uint2* ent, uint64_t total, uint32_t units, uint32_t parts,
                        uint32_t* spos, uint2* split, cudaStream_t st);
// the wave executor's entries and requirements built on the device
// (wave_build.cu) from the traced lists idx[pos[u], pos[u+1]) of every unit
bool wave_build_supported(uint32_t lines, uint32_t views, uint64_t cells);
void gpu_wave_build(const uint32_t* pos, const uint32_t* idx, uint64_t total, uint32_t units, uint32_t lines,
                    uint32_t views, uint64_t cells, uint2* ent, std::vector<uint32_t>& dep_off,
                    std::vector<uint32_t>& deps, cudaStream_t st);
bool wave_supported(const MartArgs& h);
int wave_cluster_size(const MartArgs& h);  // CTAs per view task of the wave executor (1, 2 or 4)
bool wave_fits_smem(const MartArgs& h, int lines);
size_t wave_smem_bytes(const MartArgs& m, int lines);
// prog: [views * nchunks] cumulative line counters; epoch: 0-based global
// index of the launch's first sweep
void launch_mart_wave(const MartArgs& h, const WaveSchedule& ws, unsigned* prog, unsigned* next, unsigned epoch,
                      int sweeps, cudaStream_t st, unsigned long long* prof = nullptr);

// per-problem projection statistics: stats[p*4 + {0: count>0, 1: sum>0, 2: any!=0, 3: invalid}];
// stats must hold proj_stats_words(S) doubles (the tail is block partials)
size_t proj_stats_words(int S);
void launch_proj_stats(const float* proj, int units, int S, int Sp, double* stats, cudaStream_t st);
// per-problem updates per sweep: sum over units with m != 0 of cells[u]
void launch_sweep_updates(const float* proj, const uint32_t* cells, int units, int S, int Sp,
                          unsigned long long* out, cudaStream_t st);
// max relative change over crossed cells, per problem (as uint bits of a float)
void launch_residual(const float* field, const float* prev, const uint8_t* crossed, uint64_t cells,
                     int S, int Sp, unsigned int* out, cudaStream_t st);
// count of field values that are not > 0 (reconstruct_from check)
void launch_count_nonpositive(const float* field, uint64_t n, unsigned long long* out,
                              cudaStream_t st);

// layout transposes: [S][n] <-> [n][Sp]
void launch_to_interleaved(const float* in, float* out, uint64_t n, int S, int Sp, float pad,
                           cudaStream_t st);
void launch_from_interleaved(const float* in, float* out, uint64_t n, int S, int Sp,
                             cudaStream_t st);
void launch_fill(float* p, uint64_t n, float v, cudaStream_t st);

// image-quality metrics (metrics.cu): per slice of `slices` rasters of px pixels
// out[4*s + {0: min ref, 1: max ref, 2: sum |ref-test|, 3: sum (ref-test)^2}];
// part: slices * metrics_blocks(px) * 4 doubles
int metrics_blocks(uint64_t px);
void launch_moments(const float* ref, const float* test, int slices, uint64_t px, double* part,
                    double* out, cudaStream_t st);
// mean gradient magnitude per slice (sharpness); part: slices * metrics_blocks(px) doubles
void launch_sharpness(const float* img, int slices, int rows, int cols, double* part, double* out,
                      cudaStream_t st);
// mean SSIM per slice; c1c2 [slices][2]; part: slices * ssim_tiles(rows, cols) doubles
int ssim_tiles(int rows, int cols);
void launch_ssim(const float* ref, const float* test, int slices, int rows, int cols,
                 const double* c1c2, double* part, double* out, cudaStream_t st);

// Cartesian comparator (cartesian.cu): an axis-aligned voxel grid
// (CartesianSpec, proj/include/uscg/siddon.hpp:11-25)
struct DevCart {
    int nx, ny, nz;
    double voxel;
    double o0, o1, o2;  // minimum corner
};
// Siddon system: counts per (view, line), then CSR lists (u32 voxel, f32 length)
void launch_siddon_count(const DevCart& C, int lines, int views, const double* rays, const double* theta,
                         uint32_t* counts, cudaStream_t st);
void launch_siddon_write(const DevCart& C, int lines, int views, const double* rays, const double* theta,
                         const uint32_t* off, uint32_t* idx, float* w, cudaStream_t st);
// one dependency level of the weighted MART: stored lists or Siddon on the fly
void launch_csr_level(const uint32_t* units, int n, const uint32_t* off, const uint32_t* idx, const float* w,
                      const float* proj, float* f, double beta, double p_floor, unsigned long long* clamps,
                      cudaStream_t st);
void launch_otf_level(const DevCart& C, int lines, const double* rays, const double* theta, const uint32_t* units,
                      int n, const float* proj, float* f, double beta, double p_floor, unsigned long long* clamps,
                      cudaStream_t st);

// The MART run schedule built on the device (schedule_gpu.cu): the same
// structures AsapSchedule produces (schedule.h), written into device arrays
// the caller allocates through `alloc` (which, count) once the sizes are known.
struct GpuSchedule {
    enum Array { kOrder, kLevelOff, kPredOff, kPreds, kNpredX, kSuccOff, kSuccs };
    std::function<uint32_t*(Array, size_t)> alloc;
    std::vector<uint32_t> level_off;  // host copy
    uint64_t n_preds = 0, n_succs = 0;
    double seconds[4] = {0, 0, 0, 0};  // edges, lists, levels, order
};
void gpu_schedule_build(const TraceArgs& A, int views, int max_recs, int max_cells, uint64_t cells, uint64_t visits,
                        uint32_t run, uint32_t runs_per_view, GpuSchedule& out, cudaStream_t st);

// K4 resample
void launch_perm_resample(const float* field, uint64_t cells_per_slice, int slices, int S, int Sp,
                          int n, float* out, cudaStream_t st);
void launch_bin_map(const DevGrid& g, int npix, uint32_t* map, cudaStream_t st);
// pixel -> cell of the reference permutation, npix x npix
void launch_perm_map(int n, uint32_t* map, cudaStream_t st);
// tiled resample (npix % 32 == 0): per 32x32 tile its distinct source cells
// tcells[toff[t], toff[t+1]) and per pixel (tile-major) the cell's slot
// (0xFFFF: outside the disc)
void launch_tiled_resample(const float* field, uint64_t cps, int slices, int S, int Sp, const uint32_t* toff,
                           const uint32_t* tcells, const uint16_t* slot, int n, float* out, cudaStream_t st);
void launch_map_resample(const float* field, uint64_t cells_per_slice, int slices, int S, int Sp,
                         const uint32_t* map, int npix, float* out, cudaStream_t st);
void launch_cg_map(int n, uint32_t* out, cudaStream_t st);
// cartesian_to_field for the reference law (npix = 2 * rings): field cell of
// pixel (row, col) = the inverse permutation; images [S][slices][n][n] ->
// field [S][cells] (Sp <= 0) or [cells][Sp]
void launch_cart_to_field(const float* img, uint64_t cps, int slices, int S, int Sp, int n, float* field,
                          cudaStream_t st);
// out[4*i + {0: atan2_cr, 1: hypot_cr, 2: azimuth_deg, 3: libdevice atan2}]
void launch_diag_math(int n, const double* x, const double* y, double* out, cudaStream_t st);

}  // namespace ub
