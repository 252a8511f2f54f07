/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the USPG/USCG MART hot path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj/src,
 * cited per function in uscg_oracle.c), generalized only at the seams the
 * BASELINE configs need:
 *   - ring law: any per-ring sector-count table (M1), reference 4(2k-1) default;
 *   - slice count decoupled from ring count (M3);
 *   - first-view rays given as explicit endpoint pairs (flat panel = reference
 *     ScanGeometry::detector_position; arc M7; parallel M4 generators below);
 *   - view angles given as a list (M5), reference default norm360(v*360/p).
 * With the reference defaults every result is bit-identical to the reference
 * library (pinned by tests/test_oracle.py against oracle/_ref and tests/golden).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this; the product never links it.
 */
#ifndef USCG_ORACLE_H
#define USCG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int n_rings;            /* rings, 1-based k = 1..n_rings */
    double ring_spacing;    /* radial width of every ring */
    int n_slices;           /* 1 in 2D */
    double slice_height;
    int volume;             /* 0: 2D (Slice2D), 1: 3D (Volume3D) */
    const uint32_t* counts; /* n_rings sector counts; NULL -> reference 4(2k-1) */
} orc_grid;

typedef struct {
    double phi_a, phi_b;
    uint16_t slice, ring;
} orc_record;

typedef struct {
    int lines;
    uint32_t* offsets; /* lines + 1 */
    orc_record* records;
    uint64_t n_records;
} orc_cache;

/* ring laws */
void orc_ring_counts_ref(int n_rings, uint32_t* out); /* 4(2k-1) */
void orc_ring_counts_m1(int n_rings, uint32_t* out);  /* round(2*pi*(i+0.5)), i = k-1 */
uint64_t orc_cells_per_slice(const orc_grid* g);

/* ray generators: src_out/det_out are lines*3 doubles, line = iv*det_u + iu */
void orc_rays_flat(const double src[3], const double ctr[3], int det_u, int det_v, double su,
                   double sv, double* src_out, double* det_out);
/* equiangular arc centred on the source through ctr; du_deg = angular pitch */
void orc_rays_arc(const double src[3], const double ctr[3], int det_u, double du_deg,
                  double* src_out, double* det_out);
/* parallel beam along +x in the first view: offsets (iu-(n-1)/2)*su in y,
   from x = -half_len to x = +half_len */
void orc_rays_parallel(int det_u, double su, double half_len, double* src_out, double* det_out);

double orc_norm360(double deg);
double orc_azimuth_deg(double x, double y);

/* first-view cache (precompute_first_view, direct build) */
int orc_cache_build(const orc_grid* g, int lines, const double* src, const double* det,
                    orc_cache* out);
void orc_cache_free(orc_cache* c);

/* trace_chord: no dedup; returns count, writes min(count, cap) */
int64_t orc_trace_chord(const orc_grid* g, const orc_record* rec, double theta_deg, uint32_t* out,
                        int64_t cap);

/* Tracer::trace_line with stamp dedup. stamp: cell_count u32 zeroed by caller,
   *gen carried between calls. Returns count (out must hold it). */
int64_t orc_trace_line(const orc_grid* g, const orc_cache* c, int line, double theta_deg,
                       uint32_t* stamp, uint32_t* gen, uint32_t* out, uint64_t* chords);

/* generate_projections (Binary): field f64 cell_count; out f64 views*lines */
void orc_project(const orc_grid* g, const orc_cache* c, int views, const double* theta_deg,
                 const double* field, double* out);

/* generate_projections (LengthWeighted): per (view, line) rotate the endpoints
   and cut every chord at all radial planes of its ring (phantom.cpp:213-269) */
void orc_project_length(const orc_grid* g, int lines, const double* src, const double* det,
                        int views, const double* theta_deg, const double* field, double* out);

/* The (voxel, chord length) lists of the LengthWeighted model per (view, line),
   the pieces of one cell merged at its first position. offsets: views*lines+1.
   idx / len NULL: count only. Returns the entries, (uint64_t)-1 if cap is short. */
uint64_t orc_length_lists(const orc_grid* g, int lines, const double* src, const double* det, int views,
                          const double* theta_deg, uint64_t* offsets, uint32_t* idx, double* len,
                          uint64_t cap);

/* MART over stored (voxel, length) lists (weighted_update and the loop of
   cartesian_mart_stored, siddon.cpp:141-154, 185-209). Returns the clamp count. */
uint64_t orc_weighted_mart(uint64_t rows, const uint64_t* offsets, const uint32_t* idx, const double* w,
                           const double* proj, double* field, double beta, double p_floor_cfg, int sweeps);

/* reconstruct / reconstruct_from. field: in = initial values, out = result.
   report: [0]=sweeps [1]=converged [2]=all_zero [3]=skips [4]=clamps [5]=U (cells updated)
   residuals: max_sweeps (or NULL), crossed: cell_count (or NULL).
   Returns 0, or 1 for invalid arguments. */
int orc_reconstruct(const orc_grid* g, const orc_cache* c, int views, const double* theta_deg,
                    const double* proj, double* field, double beta, double tolerance,
                    int max_sweeps, double p_floor, double* report, double* residuals,
                    uint8_t* crossed);

/* orc_reconstruct's update: 0 linear (the reference), 1 power (m/p)^beta */
void orc_set_update_power(int on);

/* uspg_to_cg_map (reference law, n = 2*rings) */
int orc_uspg_to_cg_map(int n, uint32_t* out);
/* bin-point map for any law (oracles.hpp:36-58 applied to pixel centres):
   out[pixel] = flat index within a slice, or UINT32_MAX outside the disc */
void orc_bin_map(const orc_grid* g, int npix, uint32_t* out);
/* field_to_cartesian: out slices*npix*npix; reference law uses the
   permutation, any other law the bin-point map (outside -> 0) */
void orc_field_to_cartesian(const orc_grid* g, int npix, const double* field, double* out);

/* glibc atan2 / hypot / azimuth_deg, out[3*i + k] */
void orc_math(size_t n, const double* x, const double* y, double* out);

double orc_rmse(size_t n, const double* a, const double* b);
double orc_ssim(int rows, int cols, const double* a, const double* b, double dynamic_range);
/* cartesian_to_field, reference law only (2 otherwise): field slices*cps */
int orc_cartesian_to_field(const orc_grid* g, int npix, const double* images, double* field);
/* sharpness of one rows x cols image (NAN below 2x2) */
double orc_sharpness(int rows, int cols, const double* img);

#ifdef __cplusplus
}
#endif
#endif
