/*
 * uscg_b200 — C ABI of the B200-native USPG/USCG MART hot path.
 *
 * This is the drop-in boundary for the reference library's reconstruction
 * path (/root/reference/proj, C++ namespace uscg). Plain pointers and sizes,
 * no C++ or torch types; every entry point names the reference interface it
 * replaces. The C++ mirror of the reference API (include/uscg_b200.hpp) and
 * the Python mirror (paper_2208_12964_b200/uscg.py) sit on top of it.
 *
 * Conventions
 *  - Status codes mirror the reference's exception types:
 *      USCG_ERR_INVALID_ARGUMENT  <-> std::invalid_argument
 *      USCG_ERR_DOMAIN            <-> std::domain_error
 *    uscg_last_error() returns the message of the last failure on this thread.
 *  - All calls are blocking and run on the context's stream (its own, or one
 *    set with uscg_ctx_set_stream). Handles are not thread-safe (as the
 *    reference's TraceScratch).
 *  - The tracer owns its device-resident first-view cache; the caller owns
 *    every buffer passed in. Buffers are host memory unless
 *    USCG_DEVICE_POINTERS is set, in which case they are device memory.
 *  - "problems": S independent reconstructions sharing one tracer (the
 *    BASELINE 2D slice stack). Host-layout fields are problem-major
 *    ([S][cell_count], each the reference flat order); host-layout
 *    projections are [S][views][lines] (reference ProjectionSet order).
 *    USCG_LAYOUT_INTERLEAVED selects the device-native layouts instead:
 *    field [cell_count][S_pad], projections [views*lines][S_pad]
 *    (S_pad from uscg_problem_stride).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    call fails with USCG_ERR_NO_DEVICE.
 */
#ifndef USCG_B200_H
#define USCG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    USCG_OK = 0,
    USCG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    USCG_ERR_DOMAIN = 2,           /* std::domain_error in the reference */
    USCG_ERR_CUDA = 3,
    USCG_ERR_NO_DEVICE = 4,
    USCG_ERR_ALLOC = 5
} uscg_status;

enum {
    USCG_DEVICE_POINTERS = 1u,     /* buffers are device memory */
    USCG_LAYOUT_INTERLEAVED = 2u,  /* device-native problem-minor layouts */
    USCG_MODEL_LENGTH = 4u,        /* uscg_project: ForwardModel::LengthWeighted */
    USCG_UPDATE_POWER = 8u         /* uscg_reconstruct: the multiplicative MART correction
                                      x *= (m/p)^beta (BASELINE north_star's (m/p)^(lambda a/max a)
                                      with binary coefficients) instead of the reference's linear
                                      1 - beta (1 - m/p) (proj/src/solver.cpp:41); an extension
                                      with no reference counterpart, checked against the oracle's
                                      same-named variant only */
};

typedef struct uscg_ctx_s* uscg_ctx;
typedef struct uscg_tracer_s* uscg_tracer;

/* GridSpec (proj/include/uscg/grid.hpp:21-44), generalized at two seams:
 * ring_counts (any sector law; NULL = the reference's 4(2k-1),
 * proj/src/grid.cpp:18-22) and n_slices decoupled from the ring count. */
typedef struct {
    int32_t n_rings;
    double ring_spacing;
    int32_t n_slices;      /* 1 for a 2D grid */
    double slice_height;
    int32_t volume;        /* 0 = GridMode::Slice2D, 1 = GridMode::Volume3D */
    const uint32_t* ring_counts;
} uscg_grid;

typedef enum {
    USCG_DET_FLAT = 0,     /* ScanGeometry flat panel (proj/src/scan.cpp:27-36) */
    USCG_DET_ARC = 1,      /* equiangular arc about the source; spacing_u in degrees */
    USCG_DET_PARALLEL = 2  /* parallel beam: source and detector both shift along u */
} uscg_detector;

/* ScanGeometry (proj/include/uscg/scan.hpp:21-41) plus the detector kind and
 * an optional view-angle list (NULL = view*360/views, proj/src/solver.cpp:101,116). */
typedef struct {
    int32_t detector;
    double source[3];
    double detector_center[3];
    int32_t det_u, det_v;
    double spacing_u, spacing_v;
    int32_t views;
    const double* view_angles_deg;
} uscg_scan;

/* SolverConfig (proj/include/uscg/solver.hpp:34-41) */
typedef struct {
    double beta;        /* in (0, 2) */
    double tolerance;   /* <= 0 runs every sweep */
    int32_t max_sweeps;
    double f_init;
    double p_floor;     /* <= 0: 1e-12 * mean nonzero measurement, per problem */
} uscg_solver_config;

/* ReconReport (proj/include/uscg/solver.hpp:43-52), one per problem.
 * sweep_residuals (max_sweeps doubles) and crossed (cell_count bytes) are
 * caller-owned and optional (NULL skips them). */
typedef struct {
    int32_t sweeps;
    int32_t converged;
    int32_t all_zero_data;
    double seconds;                  /* device time of the sweeps (CUDA events) */
    uint64_t zero_measurement_skips;
    uint64_t factor_clamps;
    uint64_t updates;                /* ray-voxel updates applied (U) */
    double* sweep_residuals;
    uint8_t* crossed;
} uscg_report;

typedef struct {
    int32_t lines, views;
    int32_t n_rings, n_slices;
    uint64_t records;              /* chord records in the first-view cache */
    uint64_t cells_per_slice;
    uint64_t cell_count;
    uint64_t cache_bytes;          /* device bytes of the record store + offsets */
    int32_t max_line_records;
    int32_t max_line_cells;        /* over every (view, line) */
    uint64_t cells_per_sweep;      /* sum of |active| over every (view, line) */
    uint64_t chords_per_sweep;     /* records * views */
    int32_t levels;                /* MART dependency levels per sweep (0 until built) */
    double generator_ms;           /* device time of the first-view generator (count + scan +
                                      write + annotate; 0 for an imported cache) */
    int32_t executor;              /* MART executor of the last reconstruction: -1 none yet,
                                      0 flow, 3 wave, 4 tile, 5 levels (USCG_MART_MODE) */
    uint64_t wave_requirements;    /* wave executor: other-view requirements per sweep (0 until built) */
    double wave_build_s;           /* wave executor: seconds to build its lists and requirements */
    uint64_t executor_bytes;       /* device bytes the MART executors derived from the record store
                                      (traced lists, wave entries/requirements, run schedule) */
    int32_t wave_ctas;             /* wave executor: CTAs per view task of the last solve (1 single,
                                      2 pairs, 4 clusters of four; 0 before any wave solve) */
} uscg_tracer_info;

const char* uscg_last_error(void);
const char* uscg_version(void);
/* number of kernels this library has launched in the process */
uint64_t uscg_launch_count(void);

/* ---- context ----------------------------------------------------------- */
uscg_status uscg_ctx_create(int32_t device, uscg_ctx* out);
uscg_status uscg_ctx_destroy(uscg_ctx ctx);
/* run on an external stream (a cudaStream_t passed as void*); NULL restores
 * the context's own stream */
uscg_status uscg_ctx_set_stream(uscg_ctx ctx, void* stream);
uscg_status uscg_ctx_synchronize(uscg_ctx ctx);

/* ---- rays --------------------------------------------------------------- */
/* First-view line endpoints (ScanGeometry::line_endpoints, proj/src/scan.cpp:38-42):
 * src_out/det_out hold lines*3 doubles, line = iv*det_u + iu. Host only. */
uscg_status uscg_first_view_rays(const uscg_scan* scan, double* src_out, double* det_out);

/* ---- tracer: FirstViewCache + Tracer (proj/include/uscg/tracer.hpp:18-105) */
/* Tracer(geom, spec, quarter_symmetry, threads) (tracer.hpp:87) — the cache is
 * generated on the device (K1). quarter_symmetry is validated like
 * precompute_first_view (tracer.cpp:42-44) and yields the identical cache. */
uscg_status uscg_tracer_create(uscg_ctx ctx, const uscg_grid* grid, const uscg_scan* scan,
                               int32_t quarter_symmetry, uscg_tracer* out);
/* Same, from explicit first-view rays (the ray-generator seam). */
uscg_status uscg_tracer_create_from_rays(uscg_ctx ctx, const uscg_grid* grid, int32_t lines,
                                         const double* src, const double* det, int32_t views,
                                         const double* view_angles_deg, uscg_tracer* out);
/* Adopt an existing FirstViewCache (offsets lines+1, records SoA). */
uscg_status uscg_tracer_import_cache(uscg_ctx ctx, const uscg_grid* grid, int32_t lines,
                                     const uint32_t* offsets, uint64_t records,
                                     const double* phi_a, const double* phi_b,
                                     const uint16_t* slice, const uint16_t* ring, int32_t views,
                                     const double* view_angles_deg, uscg_tracer* out);
/* The record store in its device layout (offsets lines+1 u32; phi_a, phi_b
 * records f64; keys records u32 = ring | slice << 12 | dedup flag << 31) into
 * caller buffers, host or (USCG_DEVICE_POINTERS) device. */
uscg_status uscg_tracer_copy_cache(uscg_tracer tracer, uint32_t* offsets, double* phi_a, double* phi_b,
                                   uint32_t* keys, uint32_t flags);
/* uscg_tracer_import_cache from that layout, host or (USCG_DEVICE_POINTERS)
 * device arrays: the assembly step of the row-sharded multi-GPU generator
 * (dedup flags are recomputed). */
uscg_status uscg_tracer_import_cache_keys(uscg_ctx ctx, const uscg_grid* grid, int32_t lines,
                                          const uint32_t* offsets, uint64_t records, const double* phi_a,
                                          const double* phi_b, const uint32_t* keys, int32_t views,
                                          const double* view_angles_deg, uint32_t flags, uscg_tracer* out);
/* Diagnostics: the wave executor's derived arrays (built by the first 2D
 * stack reconstruction; USCG_HOST_WAVE=1 builds them on the host): entries
 * (2 u32 per traced cell: cell | in-previous-line << 31, position in the next
 * line or 0xFFFF), requirement offsets (units + 1) and requirement pairs
 * ({view | cross-sweep << 31, lines of that view}). NULL arrays: sizes only. */
uscg_status uscg_tracer_export_wave(uscg_tracer tracer, uint64_t* n_entries, uint64_t* n_deps,
                                    uint32_t* entries, uint32_t* dep_off, uint32_t* deps);
uscg_status uscg_tracer_destroy(uscg_tracer tracer);
uscg_status uscg_tracer_get_info(uscg_tracer tracer, uscg_tracer_info* info);
/* FirstViewCache::offsets()/records() (tracer.hpp:28-29) to host arrays */
uscg_status uscg_tracer_export_cache(uscg_tracer tracer, uint32_t* offsets, double* phi_a,
                                     double* phi_b, uint16_t* slice, uint16_t* ring);
/* Tracer::trace_line (tracer.cpp:148-201): deduplicated active cells of one
 * line at theta, in the reference's emission order, computed on the device by
 * the same trace the solver uses. *count receives the full count; at most cap
 * indices are written. */
uscg_status uscg_trace_line(uscg_tracer tracer, int32_t line, double theta_deg, uint32_t* out,
                            int64_t cap, int64_t* count);
/* |active| of every line of every view, views*lines u32 (TraceScratch::cells). */
uscg_status uscg_trace_counts(uscg_tracer tracer, uint32_t* cells_out);
/* Rotated reuse of the record store (the symmetry saving of FirstViewCache,
 * tracer.hpp:18-39, served per view by Tracer::trace_line, tracer.cpp:148-201):
 * for views [view0, view0 + nviews) and every line, |active| (counts,
 * nviews*lines u32) and the sum of the active cell indices (sums, u64,
 * independent of emission order), computed from the records without expanding
 * the index lists. USCG_DEVICE_POINTERS: counts/sums are device buffers. */
uscg_status uscg_trace_checksums(uscg_tracer tracer, int32_t view0, int32_t nviews,
                                 uint32_t* counts, uint64_t* sums, uint32_t flags);
/* Build the MART dependency schedule now (otherwise built on first use). */
uscg_status uscg_tracer_build_schedule(uscg_tracer tracer);
/* The schedule the dataflow executor runs (built if needed): lines per run,
 * runs, levels, the level-sorted run order (runs), level offsets (levels+1),
 * in-sweep predecessors (pred_off runs+1, preds *n_preds) and cross-sweep
 * predecessor counts (runs). Call with null arrays first for the sizes. */
uscg_status uscg_tracer_export_schedule(uscg_tracer tracer, int32_t* run, uint32_t* runs, uint32_t* levels,
                                        uint64_t* n_preds, uint32_t* order, uint32_t* level_off,
                                        uint32_t* pred_off, uint32_t* preds, uint32_t* npred_x);
/* its merged successor lists (in- and cross-sweep, the dependency counters'
 * push targets): succ_off [runs + 1], succs [n_succs]; NULL arrays are skipped */
uscg_status uscg_tracer_export_successors(uscg_tracer tracer, uint64_t* n_succs, uint32_t* succ_off,
                                          uint32_t* succs);
/* stride of the interleaved problem dimension for S problems */
int32_t uscg_problem_stride(int32_t problems);

/* ---- forward model: generate_projections (proj/include/uscg/phantom.hpp:51-52)
 * Binary (proj/src/phantom.cpp:182-211) by default; USCG_MODEL_LENGTH selects
 * LengthWeighted (proj/src/phantom.cpp:213-269): the tracer's rays rotated per
 * view, each chord split at its ring's radial sector boundaries, every piece
 * weighted by its length (fp64 geometry and sums, fp32 output). */
uscg_status uscg_project(uscg_tracer tracer, const float* field, int32_t problems, float* proj_out,
                         uint32_t flags);

/* ---- Sp-MART: reconstruct / reconstruct_from (proj/src/solver.cpp:76-177) -----
 * from_init = 0: field_inout is output only and starts at cfg->f_init
 * (reconstruct); 1: field_inout holds the initial field (reconstruct_from,
 * must be > 0). reports: `problems` entries (may be NULL). */
uscg_status uscg_reconstruct(uscg_tracer tracer, const float* proj, int32_t problems,
                             const uscg_solver_config* cfg, float* field_inout, int32_t from_init,
                             uscg_report* reports, uint32_t flags);
/* uscg_reconstruct over `batch` independent problem stacks in host memory
 * (proj[b], field_inout[b] as in uscg_reconstruct; host layout per
 * USCG_LAYOUT_INTERLEAVED), with the transfers overlapped with the solves:
 * stack b+1 uploads on one copy stream and stack b-1 downloads on another
 * while stack b is solved (double-buffered device staging). Pinned host
 * buffers are needed for the overlap. reports: batch * problems entries, or
 * NULL. The first failing stack's error is returned; later stacks are not run. */
uscg_status uscg_reconstruct_batch(uscg_tracer tracer, int32_t batch, const float* const* proj,
                                   int32_t problems, const uscg_solver_config* cfg, float* const* field_inout,
                                   int32_t from_init, uscg_report* reports, uint32_t flags);

/* ---- resampling: uspg_to_cg_map + field_to_cartesian (proj/src/grid.cpp:75-99,
 * proj/src/phantom.cpp:149-163). Output [S][slices][npix][npix], row 0 at the
 * bottom. Reference law with npix = 2*n_rings: the reference permutation;
 * any other law / size: the bin-point rule of proj/tests/oracles.hpp:36-58 at
 * pixel centres (pixels outside the disc -> 0). */
uscg_status uscg_resample(uscg_ctx ctx, const uscg_grid* grid, const float* field,
                          int32_t problems, int32_t npix, float* out, uint32_t flags);
/* uspg_to_cg_map(n) itself (grid.hpp:84), n*n u32, host output. */
uscg_status uscg_uspg_to_cg_map(uscg_ctx ctx, int32_t n, uint32_t* out);
/* cartesian_to_field (proj/include/uscg/phantom.hpp:59, proj/src/phantom.cpp:165-180):
 * the inverse of uscg_resample for the reference law. images: [S][slices][npix][npix]
 * (row 0 at the bottom, as uscg_resample writes them); field_out: S fields in
 * the host layout [S][cell_count] (or, with USCG_LAYOUT_INTERLEAVED, the
 * device-native [cell_count][S_pad]). Errors as the reference: a grid that
 * fails GridSpec::validate, and npix != 2 * n_rings ("slice shape does not
 * match the grid", invalid argument). Other sector laws have no
 * uspg_to_cg_map (the reference's is for its own law only): invalid argument. */
uscg_status uscg_cartesian_to_field(uscg_ctx ctx, const uscg_grid* grid, const float* images, int32_t problems,
                                    int32_t npix, float* field_out, uint32_t flags);

/* ---- image-quality metrics (proj/src/metrics.cpp) on the device ------------
 * ref, test: `slices` rasters of rows x cols floats each (row-major, row 0 at
 * the bottom, as uscg_resample writes them). Per slice (any output may be
 * NULL): mae / rmse (metrics.cpp:35-60) and ssim (metrics.cpp:105-136: 8x8
 * windows, stride 1, C1 = (0.01 L)^2, C2 = (0.03 L)^2). L is dynamic_range when
 * > 0, else the range (max - min, 1 when constant) of each reference slice
 * (ssim, metrics.cpp:27-31) or, with shared_range = 1, of the whole reference
 * stack (ssim_volume, metrics.cpp:186-199). mae/rmse/ssim_volume are the means
 * of the per-slice values. Errors as the reference: empty images, and images
 * smaller than the 8x8 window when ssim is asked for (invalid argument). */
uscg_status uscg_image_metrics(uscg_ctx ctx, const float* ref, const float* test, int32_t slices,
                               int32_t rows, int32_t cols, int32_t shared_range,
                               double dynamic_range, double* mae_out, double* rmse_out,
                               double* ssim_out, uint32_t flags);
/* sharpness (proj/src/metrics.cpp:138-152) of each of `slices` rows x cols
 * rasters: the mean central-difference gradient magnitude (one-sided at the
 * borders), fp64. Errors as the reference: rows or cols < 2 ("sharpness needs
 * at least a 2x2 image", invalid argument). */
uscg_status uscg_image_sharpness(uscg_ctx ctx, const float* image, int32_t slices, int32_t rows, int32_t cols,
                                 double* sharpness_out, uint32_t flags);
/* intensity_profile (proj/src/metrics.cpp:154-159): row `row` of one rows x
 * cols raster (host memory) as doubles. Errors as the reference: row outside
 * [0, rows) ("profile row out of range", invalid argument). Host only. */
uscg_status uscg_intensity_profile(const float* image, int32_t rows, int32_t cols, int32_t row, double* out);

/* ---- Cartesian comparator (proj/include/uscg/siddon.hpp) ------------------
 * The paper's baseline on the same hardware: MART on an axis-aligned voxel
 * grid with Siddon path-length coefficients for every (view, line) — no
 * symmetry compression, so the stored system grows with the view count. */
typedef struct {
    int32_t nx, ny, nz;
    double voxel;
    double origin[3]; /* minimum corner */
} uscg_cartesian;
typedef struct uscg_csystem_s* uscg_csystem;
/* CartesianSpec::like (siddon.cpp:18-31): n x n (x slices) voxels of the
 * ring spacing covering the grid's square / cube. Host only. */
uscg_status uscg_cartesian_like(const uscg_grid* grid, uscg_cartesian* out);
/* precompute_cartesian_system (siddon.cpp:104-125) on the device, plus the
 * MART dependency schedule of its supports. stored = 0 keeps the schedule only
 * (cartesian_mart_otf: every line re-traced on every pass). */
uscg_status uscg_csystem_create(uscg_ctx ctx, const uscg_cartesian* cart, const uscg_scan* scan,
                                int32_t stored, uscg_csystem* out);
/* The USPG / USCG grid's own (voxel index, chord length) system: the pieces
 * of the LengthWeighted model (proj/src/phantom.cpp:213-269: every chord cut
 * at its ring's radial sector planes, a piece in the sector of its midpoint)
 * of every (view, line) of the tracer's scan, as stored lists with the pieces
 * of one cell merged (voxel indices in the reference's flat cell order), plus
 * the MART dependency schedule of those supports. uscg_csystem_export returns
 * the lists; uscg_csystem_reconstruct runs the reference's length-weighted row
 * action (weighted_update, proj/src/siddon.cpp:141-154) on the polar field
 * (field_out: cell_count values). The reference has no such entry point: its
 * length model only feeds generate_projections, and its weighted update only
 * runs on the Cartesian grid; this composes the two. */
uscg_status uscg_tracer_length_system(uscg_tracer tracer, uscg_csystem* out);
uscg_status uscg_csystem_info(uscg_csystem sys, uint64_t* entries, uint64_t* device_bytes,
                              int32_t* levels, double* precompute_ms);
/* CartesianSystem (offsets views*lines+1, voxel indices, f32 lengths) to host
 * arrays; stored systems only. */
uscg_status uscg_csystem_export(uscg_csystem sys, uint32_t* offsets, uint32_t* idx, float* weight);
/* cartesian_mart_stored / cartesian_mart_otf (siddon.cpp:147-209): exactly
 * cfg->max_sweeps sweeps (the reference's comparator has no stopping test),
 * p_floor = cfg->p_floor when > 0 else 1e-12 x the mean positive measurement,
 * field starts at cfg->f_init. proj [views*lines], field_out voxel_count;
 * *seconds receives the device time of the sweeps. */
uscg_status uscg_csystem_reconstruct(uscg_csystem sys, const float* proj, const uscg_solver_config* cfg,
                                     float* field_out, double* seconds, uint32_t flags);
uscg_status uscg_csystem_destroy(uscg_csystem sys);

/* ---- MART dependency schedule (host only) ---------------------------------
 * The schedule the device executors run, from explicit supports: lines in
 * sweep order, support of line u = idx[pos[u] .. pos[u+1]) (cell indices <
 * cell_count), grouped into runs of `run` consecutive lines of a view
 * (run = 1: the line DAG). Outputs, per run: order (sorted by ASAP level,
 * stable), level_off (levels + 1; caller provides runs + 1), *levels,
 * pred_off (runs + 1), preds (caller provides pos[units] entries;
 * *n_preds receives the count), npred_x (cross-sweep predecessors per run,
 * optional). */
uscg_status uscg_schedule_build(uint32_t units, uint32_t lines_per_view, uint32_t run,
                                const uint32_t* pos, const uint32_t* idx, uint64_t cell_count,
                                uint32_t* order, uint32_t* level_off, uint32_t* levels,
                                uint32_t* pred_off, uint32_t* preds, uint64_t* n_preds,
                                uint32_t* npred_x);

/* ---- diagnostics ---------------------------------------------------------
 * The device math the generator uses, for parity tests against glibc:
 * out[5*i + k], k = 0: the generator's atan2 (quick form with the
 * double-double fallback: correctly rounded), 1: hypot (correctly rounded),
 * 2: azimuth_deg (geometry.cpp:39-46), 3: libdevice atan2, 4: the
 * double-double atan2 alone (correctly rounded). */
uscg_status uscg_diag_math(uscg_ctx ctx, int32_t n, const double* x, const double* y, double* out);

#ifdef __cplusplus
}
#endif
#endif /* USCG_B200_H */
