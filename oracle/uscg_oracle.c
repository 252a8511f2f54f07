/* TEST INFRASTRUCTURE ONLY — see uscg_oracle.h.
 *
 * Plain-C restatement of the reference USPG/USCG path. Each function cites the
 * reference code it follows (paths relative to /root/reference/proj). The
 * expression order of every floating-point statement is kept so that, built
 * with gcc on x86-64 (no FMA contraction on the baseline ISA), the results are
 * bit-identical to the reference library with its default ring law.
 */
#include "uscg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int g_update_power = 0;

static const double kPi = 3.141592653589793238462643383279502884;
#define DEG_PER_RAD (180.0 / 3.141592653589793238462643383279502884)
#define RAD_PER_DEG (3.141592653589793238462643383279502884 / 180.0)

/* ---- grid (src/grid.cpp:18-30,61-73) ---------------------------------- */

void orc_ring_counts_ref(int n_rings, uint32_t* out) {
    for (int k = 1; k <= n_rings; ++k)
        out[k - 1] = (uint32_t)(4 * (2 * k - 1)); /* grid.cpp:16-20 */
}

void orc_ring_counts_m1(int n_rings, uint32_t* out) {
    /* BASELINE.json: ring i (0-based) has round(2*pi*(i+0.5)) sectors (M1) */
    for (int i = 0; i < n_rings; ++i)
        out[i] = (uint32_t)llround(2.0 * kPi * (i + 0.5));
}

static uint32_t ring_count(const orc_grid* g, int k) {
    return g->counts ? g->counts[k - 1] : (uint32_t)(4 * (2 * k - 1));
}

static uint32_t ring_head(const orc_grid* g, int k) {
    if (!g->counts) {
        uint32_t m = (uint32_t)(k - 1); /* grid.cpp:22-28 closed form */
        return 4u * m * m;
    }
    uint32_t h = 0;
    for (int j = 1; j < k; ++j)
        h += g->counts[j - 1];
    return h;
}

uint64_t orc_cells_per_slice(const orc_grid* g) {
    uint64_t s = 0;
    for (int k = 1; k <= g->n_rings; ++k)
        s += ring_count(g, k);
    return s;
}

typedef struct {
    uint32_t count, head;
    double inv_step;
} ring_row;

static ring_row* ring_table(const orc_grid* g) {
    ring_row* t = (ring_row*)malloc(sizeof(ring_row) * (size_t)(g->n_rings + 1));
    for (int k = 1; k <= g->n_rings; ++k) {
        t[k].count = ring_count(g, k);
        t[k].head = ring_head(g, k);
        t[k].inv_step = t[k].count / 360.0; /* grid.cpp:68 */
    }
    return t;
}

/* GridSpec accessors (include/uscg/grid.hpp:29-36): n = 2*rings */
static double g_radius(const orc_grid* g) { return 0.5 * (2 * g->n_rings) * g->ring_spacing; }
static double g_z_extent(const orc_grid* g) {
    return g->volume ? g->n_slices * g->slice_height : g->slice_height;
}
static double g_z_offset(const orc_grid* g) { return 0.5 * g_z_extent(g); }
static double g_eps(const orc_grid* g) { return 1e-9 * g_radius(g); } /* geometry.cpp:29 */

/* ---- rays (src/scan.cpp:27-42) ---------------------------------------- */

void orc_rays_flat(const double src[3], const double ctr[3], int det_u, int det_v, double su,
                   double sv, double* src_out, double* det_out) {
    const double ax = ctr[0] - src[0];
    const double ay = ctr[1] - src[1];
    const double alen = sqrt(ax * ax + ay * ay);
    const double ux = -ay / alen;
    const double uy = ax / alen;
    for (int iv = 0; iv < det_v; ++iv)
        for (int iu = 0; iu < det_u; ++iu) {
            const double du = (iu - 0.5 * (det_u - 1)) * su;
            const double dv = (iv - 0.5 * (det_v - 1)) * sv;
            const size_t l = (size_t)iv * det_u + iu;
            src_out[3 * l + 0] = src[0];
            src_out[3 * l + 1] = src[1];
            src_out[3 * l + 2] = src[2];
            det_out[3 * l + 0] = ctr[0] + du * ux;
            det_out[3 * l + 1] = ctr[1] + du * uy;
            det_out[3 * l + 2] = ctr[2] + dv;
        }
}

void orc_rays_arc(const double src[3], const double ctr[3], int det_u, double du_deg,
                  double* src_out, double* det_out) {
    const double ax = ctr[0] - src[0];
    const double ay = ctr[1] - src[1];
    const double rad = sqrt(ax * ax + ay * ay);
    const double a0 = atan2(ay, ax);
    for (int iu = 0; iu < det_u; ++iu) {
        const double g = a0 + (iu - 0.5 * (det_u - 1)) * du_deg * RAD_PER_DEG;
        src_out[3 * iu + 0] = src[0];
        src_out[3 * iu + 1] = src[1];
        src_out[3 * iu + 2] = src[2];
        det_out[3 * iu + 0] = src[0] + rad * cos(g);
        det_out[3 * iu + 1] = src[1] + rad * sin(g);
        det_out[3 * iu + 2] = ctr[2];
    }
}

void orc_rays_parallel(int det_u, double su, double half_len, double* src_out, double* det_out) {
    for (int iu = 0; iu < det_u; ++iu) {
        const double off = (iu - 0.5 * (det_u - 1)) * su;
        src_out[3 * iu + 0] = -half_len;
        src_out[3 * iu + 1] = off;
        src_out[3 * iu + 2] = 0;
        det_out[3 * iu + 0] = half_len;
        det_out[3 * iu + 1] = off;
        det_out[3 * iu + 2] = 0;
    }
}

/* ---- angles (src/geometry.cpp:39-55) ------------------------------------ */

double orc_azimuth_deg(double x, double y) {
    double deg = atan2(y, x) * DEG_PER_RAD;
    if (deg < 0)
        deg += 360.0;
    if (deg >= 360.0)
        deg = 0.0;
    return deg;
}

double orc_norm360(double deg) {
    deg = fmod(deg, 360.0);
    if (deg < 0)
        deg += 360.0;
    if (deg >= 360.0)
        deg = 0.0;
    return deg;
}

/* ---- crossings (src/geometry.cpp:29-37,72-85,127-198) ------------------ */

static int is_axial(const double s[3], const double d[3]) {
    const double ux = s[0] - d[0], uy = s[1] - d[1];
    const double uxy2 = ux * ux + uy * uy;
    const double dx = d[0] - s[0], dy = d[1] - s[1], dz = d[2] - s[2];
    const double dir2 = dx * dx + dy * dy + dz * dz;
    return dir2 == 0.0 || uxy2 <= 1e-24 * dir2;
}

static int circle_taus(const double s[3], const double d[3], double radius, double* tau0,
                       double* tau1) {
    const double ux = s[0] - d[0], uy = s[1] - d[1];
    const double uxy2 = ux * ux + uy * uy;
    const double t = (s[0] * ux + s[1] * uy) / uxy2;
    const double cross = s[0] * d[1] - s[1] * d[0];
    const double d2 = cross * cross / uxy2;
    const double r2 = radius * radius;
    if (d2 > r2)
        return 0;
    const double k = sqrt((r2 - d2) / uxy2);
    *tau0 = t - k;
    *tau1 = t + k;
    return 2;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Returns the number of points written to pts (3 doubles each). */
static int sorted_points(const orc_grid* g, const double s[3], const double d[3], double* taus,
                         double* pts) {
    const double dir[3] = {d[0] - s[0], d[1] - s[1], d[2] - s[2]};
    const double radius = g_radius(g);
    const double eps = g_eps(g);
    const int volume = g->volume;
    const double zoff = g_z_offset(g);
    int nt = 0;

    if (is_axial(s, d)) {
        if (!volume)
            return 0;
        if (hypot(s[0], s[1]) >= radius)
            return 0;
        const double dz = d[2] - s[2];
        if (dz == 0.0)
            return 0;
        for (int m = 0; m <= g->n_slices; ++m) {
            const double tau = (m * g->slice_height - zoff - s[2]) / dz;
            if (tau >= 0.0 && tau <= 1.0)
                taus[nt++] = tau;
        }
    } else {
        const double zlim = zoff + eps;
        for (int ring = 1; ring <= g->n_rings; ++ring) {
            double tv[2];
            if (circle_taus(s, d, ring * g->ring_spacing, &tv[0], &tv[1]) == 0)
                continue;
            for (int i = 0; i < 2; ++i) {
                const double tau = tv[i];
                if (tau < 0.0 || tau > 1.0)
                    continue;
                if (volume) {
                    const double z = s[2] + tau * dir[2];
                    if (fabs(z) > zlim)
                        continue;
                }
                taus[nt++] = tau;
            }
        }
        if (volume && dir[2] != 0.0) {
            const double lim2 = (radius + eps) * (radius + eps);
            for (int m = 0; m <= g->n_slices; ++m) {
                const double tau = (m * g->slice_height - zoff - s[2]) / dir[2];
                if (tau < 0.0 || tau > 1.0)
                    continue;
                const double x = s[0] + tau * dir[0];
                const double y = s[1] + tau * dir[1];
                if (x * x + y * y <= lim2)
                    taus[nt++] = tau;
            }
        }
    }

    qsort(taus, (size_t)nt, sizeof(double), cmp_double);

    const double len = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    int np = 0;
    double last_tau = 0;
    for (int i = 0; i < nt; ++i) {
        const double tau = taus[i];
        if (np > 0 && (tau - last_tau) * len <= eps)
            continue;
        pts[3 * np + 0] = s[0] + tau * dir[0];
        pts[3 * np + 1] = s[1] + tau * dir[1];
        pts[3 * np + 2] = s[2] + tau * dir[2];
        ++np;
        last_tau = tau;
    }
    return np;
}

/* classify_chord (src/geometry.cpp:200-227); returns 1 when a record is made */
static int classify_chord(const orc_grid* g, const double* pk, const double* pk1, orc_record* rec) {
    const double eps = g_eps(g);
    const double ex = pk[0] - pk1[0], ey = pk[1] - pk1[1], ez = pk[2] - pk1[2];
    if (sqrt(ex * ex + ey * ey + ez * ez) <= eps)
        return 0;
    const double mid[3] = {(pk[0] + pk1[0]) / 2, (pk[1] + pk1[1]) / 2, (pk[2] + pk1[2]) / 2};
    int slice = 0;
    if (g->volume) {
        const double zloc = mid[2] + g_z_offset(g);
        const double sf = floor(zloc / g->slice_height);
        if (sf < 0 || sf >= g->n_slices)
            return 0;
        slice = (int)sf;
    }
    const double dm = hypot(mid[0], mid[1]);
    const int ring = (int)floor(dm / g->ring_spacing) + 1;
    if (ring > g->n_rings)
        return 0;
    rec->phi_a = orc_azimuth_deg(pk[0], pk[1]);
    rec->phi_b = orc_azimuth_deg(pk1[0], pk1[1]);
    rec->slice = (uint16_t)slice;
    rec->ring = (uint16_t)ring;
    return 1;
}

/* ---- first-view cache (src/tracer.cpp:38-102, direct build) ------------ */

int orc_cache_build(const orc_grid* g, int lines, const double* src, const double* det,
                    orc_cache* out) {
    const int max_t = 2 * g->n_rings + g->n_slices + 2;
    double* taus = (double*)malloc(sizeof(double) * (size_t)max_t);
    double* pts = (double*)malloc(sizeof(double) * 3 * (size_t)max_t);
    size_t cap = 1024, n = 0;
    orc_record* recs = (orc_record*)malloc(sizeof(orc_record) * cap);
    uint32_t* off = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(lines + 1));
    off[0] = 0;
    for (int l = 0; l < lines; ++l) {
        const int np = sorted_points(g, src + 3 * (size_t)l, det + 3 * (size_t)l, taus, pts);
        for (int i = 0; i + 1 < np; ++i) {
            orc_record r;
            if (!classify_chord(g, pts + 3 * i, pts + 3 * (i + 1), &r))
                continue;
            if (n == cap) {
                cap *= 2;
                recs = (orc_record*)realloc(recs, sizeof(orc_record) * cap);
            }
            recs[n++] = r;
        }
        off[l + 1] = (uint32_t)n;
    }
    free(taus);
    free(pts);
    out->lines = lines;
    out->offsets = off;
    out->records = recs;
    out->n_records = n;
    return 0;
}

void orc_cache_free(orc_cache* c) {
    free(c->offsets);
    free(c->records);
    c->offsets = NULL;
    c->records = NULL;
}

/* ---- per-view tracing (src/tracer.cpp:104-201) -------------------------- */

typedef struct {
    int lo, hi, seam, ng;
    uint32_t base;
} chord_range;

static chord_range rotate_chord(const orc_grid* g, const ring_row* rt, uint64_t per_slice,
                                const orc_record* rec, double theta) {
    const ring_row* rl = &rt[rec->ring];
    const int ng = (int)rl->count;
    double a = rec->phi_a + theta;
    if (a >= 360.0)
        a -= 360.0;
    double b = rec->phi_b + theta;
    if (b >= 360.0)
        b -= 360.0;
    int ga = (int)(a * rl->inv_step);
    if (ga >= ng)
        ga = ng - 1;
    int gb = (int)(b * rl->inv_step);
    if (gb >= ng)
        gb = ng - 1;
    chord_range r;
    r.base = (uint32_t)(rec->slice * (uint32_t)per_slice + rl->head);
    r.ng = ng;
    r.lo = ga < gb ? ga : gb;
    r.hi = ga < gb ? gb : ga;
    r.seam = !(fabs(a - b) <= 180.0);
    (void)g;
    return r;
}

int64_t orc_trace_chord(const orc_grid* g, const orc_record* rec, double theta_deg, uint32_t* out,
                        int64_t cap) {
    ring_row* rt = ring_table(g);
    const chord_range r = rotate_chord(g, rt, orc_cells_per_slice(g), rec, orc_norm360(theta_deg));
    int64_t n = 0;
    if (!r.seam) {
        for (int q = r.lo; q <= r.hi; ++q, ++n)
            if (n < cap)
                out[n] = r.base + (uint32_t)q;
    } else {
        for (int q = r.hi; q < r.ng; ++q, ++n)
            if (n < cap)
                out[n] = r.base + (uint32_t)q;
        for (int q = 0; q <= r.lo; ++q, ++n)
            if (n < cap)
                out[n] = r.base + (uint32_t)q;
    }
    free(rt);
    return n;
}

static int64_t trace_line_rt(const orc_grid* g, const ring_row* rt, uint64_t per_slice,
                             const orc_cache* c, int line, double theta_deg, uint32_t* stamp,
                             uint32_t* gen, uint32_t* out, uint64_t* chords) {
    if (++*gen == 0) {
        memset(stamp, 0, sizeof(uint32_t) * per_slice * (size_t)(g->volume ? g->n_slices : 1));
        *gen = 1;
    }
    const uint32_t gcur = *gen;
    const double theta = orc_norm360(theta_deg);
    int64_t n = 0;
    for (uint32_t i = c->offsets[line]; i < c->offsets[line + 1]; ++i) {
        const chord_range r = rotate_chord(g, rt, per_slice, &c->records[i], theta);
        if (!r.seam) {
            for (int q = r.lo; q <= r.hi; ++q) {
                const uint32_t idx = r.base + (uint32_t)q;
                if (stamp[idx] != gcur) {
                    stamp[idx] = gcur;
                    out[n++] = idx;
                }
            }
        } else {
            for (int q = r.hi; q < r.ng; ++q) {
                const uint32_t idx = r.base + (uint32_t)q;
                if (stamp[idx] != gcur) {
                    stamp[idx] = gcur;
                    out[n++] = idx;
                }
            }
            for (int q = 0; q <= r.lo; ++q) {
                const uint32_t idx = r.base + (uint32_t)q;
                if (stamp[idx] != gcur) {
                    stamp[idx] = gcur;
                    out[n++] = idx;
                }
            }
        }
        if (chords)
            ++*chords;
    }
    return n;
}

int64_t orc_trace_line(const orc_grid* g, const orc_cache* c, int line, double theta_deg,
                       uint32_t* stamp, uint32_t* gen, uint32_t* out, uint64_t* chords) {
    ring_row* rt = ring_table(g);
    const int64_t n =
        trace_line_rt(g, rt, orc_cells_per_slice(g), c, line, theta_deg, stamp, gen, out, chords);
    free(rt);
    return n;
}

static size_t cell_count(const orc_grid* g) {
    return (size_t)orc_cells_per_slice(g) * (size_t)(g->volume ? g->n_slices : 1);
}

static size_t max_line_cells(const orc_grid* g, const orc_cache* c, const ring_row* rt) {
    /* an upper bound: every chord spans at most its ring's full count */
    size_t best = 0;
    for (int l = 0; l < c->lines; ++l) {
        size_t s = 0;
        for (uint32_t i = c->offsets[l]; i < c->offsets[l + 1]; ++i)
            s += rt[c->records[i].ring].count;
        if (s > best)
            best = s;
    }
    (void)g;
    return best + 1;
}

/* ---- binary forward model (src/phantom.cpp:182-211, solver.cpp:25-31) -- */

void orc_project(const orc_grid* g, const orc_cache* c, int views, const double* theta_deg,
                 const double* field, double* out) {
    ring_row* rt = ring_table(g);
    const uint64_t per_slice = orc_cells_per_slice(g);
    uint32_t* stamp = (uint32_t*)calloc(cell_count(g), sizeof(uint32_t));
    uint32_t gen = 0;
    uint32_t* active = (uint32_t*)malloc(sizeof(uint32_t) * max_line_cells(g, c, rt));
    for (int v = 0; v < views; ++v) {
        const double theta = orc_norm360(theta_deg[v]);
        for (int l = 0; l < c->lines; ++l) {
            const int64_t n = trace_line_rt(g, rt, per_slice, c, l, theta, stamp, &gen, active, NULL);
            double sum = 0;
            for (int64_t i = 0; i < n; ++i)
                sum += field[active[i]];
            out[(size_t)v * c->lines + l] = sum;
        }
    }
    free(active);
    free(stamp);
    free(rt);
}

/* ---- length-weighted forward model (src/phantom.cpp:213-269) ------------ */

static void rotate_z(const double p[3], double deg, double out[3]) {
    const double rad = deg * RAD_PER_DEG; /* scan.cpp:50-54 */
    const double cs = cos(rad), sn = sin(rad);
    out[0] = cs * p[0] - sn * p[1];
    out[1] = sn * p[0] + cs * p[1];
    out[2] = p[2];
}

/* The LengthWeighted model's coefficients (phantom.cpp:213-269): every piece
   (cell, length) of the line through s and d, in the reference's order, handed
   to `emit`. Shared by the projector and the list emitter below. */
typedef void (*piece_fn)(void* ctx, uint32_t cell, double length);

static void length_pieces(const orc_grid* g, const ring_row* rt, uint64_t per_slice, double* taus,
                          double* pts, double* cuts, const double* s, const double* d, piece_fn emit,
                          void* ctx) {
    const int np = sorted_points(g, s, d, taus, pts);
    for (int i = 0; i + 1 < np; ++i) {
        orc_record rec;
        if (!classify_chord(g, pts + 3 * i, pts + 3 * (i + 1), &rec))
            continue;
        const double* a = pts + 3 * i;
        const double u[3] = {pts[3 * (i + 1)] - a[0], pts[3 * (i + 1) + 1] - a[1],
                             pts[3 * (i + 1) + 2] - a[2]};
        const double chord_len = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        const ring_row* rl = &rt[rec.ring];
        const double step_deg = 360.0 / rl->count;
        int nc = 0;
        cuts[nc++] = 0.0;
        cuts[nc++] = 1.0;
        for (uint32_t j = 0; j < rl->count; ++j) {
            const double psi = j * step_deg * (kPi / 180.0);
            const double ex = cos(psi), ey = sin(psi);
            const double g0 = ex * a[1] - ey * a[0];
            const double g1 = ex * u[1] - ey * u[0];
            if (g1 == 0.0)
                continue;
            const double tau = -g0 / g1;
            if (tau > 0.0 && tau < 1.0)
                cuts[nc++] = tau;
        }
        qsort(cuts, (size_t)nc, sizeof(double), cmp_double);
        const uint32_t base = (uint32_t)(rec.slice * (uint32_t)per_slice + rl->head);
        for (int q = 0; q + 1 < nc; ++q) {
            const double piece = (cuts[q + 1] - cuts[q]) * chord_len;
            if (piece <= 0)
                continue;
            const double mid = 0.5 * (cuts[q] + cuts[q + 1]);
            const double phi = orc_azimuth_deg(a[0] + mid * u[0], a[1] + mid * u[1]);
            int sector = (int)(phi * rl->inv_step);
            if (sector >= (int)rl->count)
                sector = (int)rl->count - 1;
            emit(ctx, base + (uint32_t)sector, piece);
        }
    }
}

typedef struct {
    const double* field;
    double total;
} sum_ctx;

static void sum_piece(void* c, uint32_t cell, double length) {
    sum_ctx* k = (sum_ctx*)c;
    k->total += length * k->field[cell];
}

void orc_project_length(const orc_grid* g, int lines, const double* src, const double* det,
                        int views, const double* theta_deg, const double* field, double* out) {
    ring_row* rt = ring_table(g);
    const uint64_t per_slice = orc_cells_per_slice(g);
    const int max_t = 2 * g->n_rings + g->n_slices + 2;
    double* taus = (double*)malloc(sizeof(double) * (size_t)max_t);
    double* pts = (double*)malloc(sizeof(double) * 3 * (size_t)max_t);
    uint32_t maxc = 0;
    for (int k = 1; k <= g->n_rings; ++k)
        if (rt[k].count > maxc)
            maxc = rt[k].count;
    double* cuts = (double*)malloc(sizeof(double) * (size_t)(maxc + 2));
    for (int v = 0; v < views; ++v) {
        const double theta = orc_norm360(theta_deg[v]);
        for (int l = 0; l < lines; ++l) {
            double s[3], d[3];
            rotate_z(src + 3 * (size_t)l, theta, s);
            rotate_z(det + 3 * (size_t)l, theta, d);
            sum_ctx k = {field, 0.0};
            length_pieces(g, rt, per_slice, taus, pts, cuts, s, d, sum_piece, &k);
            out[(size_t)v * lines + l] = k.total;
        }
    }
    free(cuts);
    free(taus);
    free(pts);
    free(rt);
}

/* The (voxel, chord length) lists of the LengthWeighted model, one per (view,
   line): the pieces of phantom.cpp:213-269 with the pieces of one cell merged
   (a line may cross a cell twice, either side of its closest approach; the
   binary tracer's stamp dedup, tracer.cpp:181-195, handles the same case), the
   cell listed where it is first met. offsets: views*lines + 1. idx / len NULL:
   count only. Returns the number of entries, or (uint64_t)-1 when cap is too
   small. */
typedef struct {
    uint32_t* idx;
    double* len;
    uint64_t begin, n, cap;
    uint32_t* stamp; /* cell -> 1 + position within the line, valid if mark[cell] == unit + 1 */
    uint32_t* mark;
    uint32_t unit1;
    int overflow;
} list_ctx;

static void list_piece(void* c, uint32_t cell, double length) {
    list_ctx* k = (list_ctx*)c;
    if (k->mark[cell] == k->unit1) {
        if (k->len)
            k->len[k->begin + k->stamp[cell]] += length;
        return;
    }
    k->mark[cell] = k->unit1;
    k->stamp[cell] = (uint32_t)(k->n - k->begin);
    if (k->idx) {
        if (k->n >= k->cap) {
            k->overflow = 1;
            return;
        }
        k->idx[k->n] = cell;
        k->len[k->n] = length;
    }
    ++k->n;
}

uint64_t orc_length_lists(const orc_grid* g, int lines, const double* src, const double* det, int views,
                          const double* theta_deg, uint64_t* offsets, uint32_t* idx, double* len,
                          uint64_t cap) {
    ring_row* rt = ring_table(g);
    const uint64_t per_slice = orc_cells_per_slice(g);
    const size_t ncell = cell_count(g);
    const int max_t = 2 * g->n_rings + g->n_slices + 2;
    double* taus = (double*)malloc(sizeof(double) * (size_t)max_t);
    double* pts = (double*)malloc(sizeof(double) * 3 * (size_t)max_t);
    uint32_t maxc = 0;
    for (int k = 1; k <= g->n_rings; ++k)
        if (rt[k].count > maxc)
            maxc = rt[k].count;
    double* cuts = (double*)malloc(sizeof(double) * (size_t)(maxc + 2));
    list_ctx k = {idx, len, 0, 0, cap, (uint32_t*)calloc(ncell, sizeof(uint32_t)),
                  (uint32_t*)calloc(ncell, sizeof(uint32_t)), 0, 0};
    for (int v = 0; v < views; ++v) {
        const double theta = orc_norm360(theta_deg[v]);
        for (int l = 0; l < lines; ++l) {
            double s[3], d[3];
            rotate_z(src + 3 * (size_t)l, theta, s);
            rotate_z(det + 3 * (size_t)l, theta, d);
            const size_t unit = (size_t)v * lines + l;
            k.begin = k.n;
            k.unit1 = (uint32_t)unit + 1;
            offsets[unit] = k.n;
            length_pieces(g, rt, per_slice, taus, pts, cuts, s, d, list_piece, &k);
        }
    }
    offsets[(size_t)views * lines] = k.n;
    free(k.stamp);
    free(k.mark);
    free(cuts);
    free(taus);
    free(pts);
    free(rt);
    return k.overflow ? (uint64_t)-1 : k.n;
}

/* MART over stored (voxel, length) lists: weighted_update and the sweep loop of
   cartesian_mart_stored (siddon.cpp:141-154, 185-209) — length-weighted forward
   projection, one multiplicative factor per line, no stopping test; p_floor =
   cfg value when > 0, else auto_p_floor (siddon.cpp:128-139). field: in =
   initial values, out = result. Returns the number of clamped factors. */
uint64_t orc_weighted_mart(uint64_t rows, const uint64_t* offsets, const uint32_t* idx, const double* w,
                           const double* proj, double* field, double beta, double p_floor_cfg, int sweeps) {
    double p_floor = p_floor_cfg;
    if (!(p_floor > 0)) {
        double sum = 0;
        uint64_t count = 0;
        for (uint64_t r = 0; r < rows; ++r)
            if (proj[r] > 0) {
                sum += proj[r];
                ++count;
            }
        p_floor = count == 0 ? 1e-12 : 1e-12 * (sum / count);
    }
    uint64_t clamps = 0;
    for (int s = 0; s < sweeps; ++s)
        for (uint64_t r = 0; r < rows; ++r) {
            const uint64_t b = offsets[r], e = offsets[r + 1];
            if (proj[r] == 0 || b == e)
                continue;
            double p_bar = 0;
            for (uint64_t i = b; i < e; ++i)
                p_bar += w[i] * field[idx[i]];
            const double ratio = proj[r] / (p_bar > p_floor ? p_bar : p_floor);
            double factor = 1.0 - beta * (1.0 - ratio);
            if (factor <= 0) {
                factor = p_floor;
                ++clamps;
            }
            for (uint64_t i = b; i < e; ++i)
                field[idx[i]] *= factor;
        }
    return clamps;
}

/* ---- Sp-MART (src/solver.cpp:33-162) ------------------------------------ */

int orc_reconstruct(const orc_grid* g, const orc_cache* c, int views, const double* theta_deg,
                    const double* proj, double* field, double beta, double tolerance,
                    int max_sweeps, double p_floor_cfg, double* report, double* residuals,
                    uint8_t* crossed_out) {
    if (!(beta > 0 && beta < 2) || max_sweeps < 1)
        return 1; /* validate_config, solver.cpp:55-61 */
    const size_t nd = (size_t)views * (size_t)c->lines;
    for (size_t i = 0; i < nd; ++i)
        if (!isfinite(proj[i]) || proj[i] < 0)
            return 1; /* ProjectionSet::validate, solver.cpp:10-23 */
    const size_t ncell = cell_count(g);
    for (int i = 0; i < 6; ++i)
        report[i] = 0;
    uint8_t* crossed = (uint8_t*)calloc(ncell, 1);

    int any = 0;
    for (size_t i = 0; i < nd; ++i)
        if (proj[i] != 0) {
            any = 1;
            break;
        }
    if (!any) {
        report[2] = 1;
        if (crossed_out)
            memcpy(crossed_out, crossed, ncell);
        free(crossed);
        return 0;
    }

    double p_floor = p_floor_cfg;
    if (!(p_floor > 0)) { /* auto_p_floor, solver.cpp:64-74 */
        double sum = 0;
        size_t cnt = 0;
        for (size_t i = 0; i < nd; ++i)
            if (proj[i] > 0) {
                sum += proj[i];
                ++cnt;
            }
        p_floor = cnt == 0 ? 1e-12 : 1e-12 * (sum / cnt);
    }

    ring_row* rt = ring_table(g);
    const uint64_t per_slice = orc_cells_per_slice(g);
    uint32_t* stamp = (uint32_t*)calloc(ncell, sizeof(uint32_t));
    uint32_t gen = 0;
    uint32_t* active = (uint32_t*)malloc(sizeof(uint32_t) * max_line_cells(g, c, rt));
    const int track = tolerance > 0;
    double* prev = track ? (double*)malloc(sizeof(double) * ncell) : NULL;
    double skips = 0, clamps = 0, updates = 0;
    int sweeps = 0, converged = 0;

    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        if (track)
            memcpy(prev, field, sizeof(double) * ncell);
        for (int v = 0; v < views; ++v) {
            const double theta = orc_norm360(theta_deg[v]);
            for (int l = 0; l < c->lines; ++l) {
                const double m = proj[(size_t)v * c->lines + l];
                if (m == 0) {
                    if (sweep == 0) {
                        const int64_t n =
                            trace_line_rt(g, rt, per_slice, c, l, theta, stamp, &gen, active, NULL);
                        for (int64_t i = 0; i < n; ++i)
                            crossed[active[i]] = 1;
                    }
                    skips += 1;
                    continue;
                }
                const int64_t n =
                    trace_line_rt(g, rt, per_slice, c, l, theta, stamp, &gen, active, NULL);
                if (sweep == 0)
                    for (int64_t i = 0; i < n; ++i)
                        crossed[active[i]] = 1;
                /* mart_update_line, solver.cpp:33-51 */
                double p_bar = 0;
                for (int64_t i = 0; i < n; ++i)
                    p_bar += field[active[i]];
                const double ratio = m / (p_bar > p_floor ? p_bar : p_floor);
                /* linear binary form (solver.cpp:41); or, when selected, the
                   power form (m/p)^beta, the builder's extension (USCG_UPDATE_POWER) */
                double factor = g_update_power ? (ratio > 0 ? pow(ratio, beta) : 0.0) : 1.0 - beta * (1.0 - ratio);
                if (factor <= 0) {
                    factor = p_floor;
                    clamps += 1;
                }
                for (int64_t i = 0; i < n; ++i)
                    field[active[i]] *= factor;
                updates += (double)n;
            }
        }
        ++sweeps;
        if (track) {
            double residual = 0;
            for (size_t i = 0; i < ncell; ++i) {
                if (!crossed[i])
                    continue;
                const double rel = fabs(field[i] - prev[i]) / prev[i];
                if (rel > residual)
                    residual = rel;
            }
            if (residuals)
                residuals[sweep] = residual;
            if (residual <= tolerance) {
                converged = 1;
                break;
            }
        }
    }
    report[0] = sweeps;
    report[1] = converged;
    report[3] = skips;
    report[4] = clamps;
    report[5] = updates;
    if (crossed_out)
        memcpy(crossed_out, crossed, ncell);
    free(prev);
    free(active);
    free(stamp);
    free(rt);
    free(crossed);
    return 0;
}

/* update form of orc_reconstruct: 0 the reference's linear 1 - beta (1 - m/p)
   (solver.cpp:41), 1 the power form (m/p)^beta (no reference counterpart) */
void orc_set_update_power(int on) { g_update_power = on != 0; }

/* ---- polar -> Cartesian (src/grid.cpp:75-99, src/phantom.cpp:149-163) ---- */

int orc_uspg_to_cg_map(int n, uint32_t* map) {
    if (n < 2 || n % 2 != 0)
        return 2;
    const int c = n / 2;
#define PIX(row, col) ((uint32_t)(row) * (uint32_t)n + (uint32_t)(col))
    for (int k = 1; k <= c; ++k) {
        uint32_t flat = 4u * (uint32_t)(k - 1) * (uint32_t)(k - 1);
        for (int t = 0; t < k; ++t)
            map[flat++] = PIX(c + t, c + k - 1);
        for (int t = 0; t < 2 * k - 1; ++t)
            map[flat++] = PIX(c + k - 1, c + k - 2 - t);
        for (int t = 0; t < 2 * k - 1; ++t)
            map[flat++] = PIX(c + k - 2 - t, c - k);
        for (int t = 0; t < 2 * k - 1; ++t)
            map[flat++] = PIX(c - k, c - k + 1 + t);
        for (int t = 0; t < k - 1; ++t)
            map[flat++] = PIX(c - k + 1 + t, c + k - 1);
    }
#undef PIX
    return 0;
}

void orc_bin_map(const orc_grid* g, int npix, uint32_t* out) {
    /* bin_point (tests/oracles.hpp:36-58) at pixel centres; pixel size equals
       the ring spacing scaled so that npix pixels span the disc diameter */
    ring_row* rt = ring_table(g);
    const double radius = g_radius(g);
    const double px = 2.0 * radius / npix;
    for (int row = 0; row < npix; ++row) {
        const double y = (row + 0.5 - npix / 2) * px;
        for (int col = 0; col < npix; ++col) {
            const double x = (col + 0.5 - npix / 2) * px;
            const double rho = hypot(x, y);
            uint32_t v = UINT32_MAX;
            if (rho < radius) {
                const int ring = (int)floor(rho / g->ring_spacing) + 1;
                if (ring <= g->n_rings) {
                    const int ng = (int)rt[ring].count;
                    const double phi = orc_azimuth_deg(x, y);
                    int sector = (int)(phi * (ng / 360.0));
                    if (sector >= ng)
                        sector = ng - 1;
                    v = rt[ring].head + (uint32_t)sector;
                }
            }
            out[(size_t)row * npix + col] = v;
        }
    }
    free(rt);
}

void orc_field_to_cartesian(const orc_grid* g, int npix, const double* field, double* out) {
    const int slices = g->volume ? g->n_slices : 1;
    const uint64_t per_slice = orc_cells_per_slice(g);
    const size_t npx = (size_t)npix * npix;
    if (!g->counts && npix == 2 * g->n_rings) {
        uint32_t* map = (uint32_t*)malloc(sizeof(uint32_t) * npx);
        orc_uspg_to_cg_map(npix, map);
        for (int s = 0; s < slices; ++s)
            for (size_t f = 0; f < npx; ++f)
                out[(size_t)s * npx + map[f]] = field[(size_t)s * per_slice + f];
        free(map);
        return;
    }
    uint32_t* map = (uint32_t*)malloc(sizeof(uint32_t) * npx);
    orc_bin_map(g, npix, map);
    for (int s = 0; s < slices; ++s)
        for (size_t p = 0; p < npx; ++p)
            out[(size_t)s * npx + p] =
                map[p] == UINT32_MAX ? 0.0 : field[(size_t)s * per_slice + map[p]];
    free(map);
}

/* cartesian_to_field (src/phantom.cpp:165-180): dst[flat] = img[map[flat]],
   reference law only (npix = 2*rings); returns 2 otherwise */
int orc_cartesian_to_field(const orc_grid* g, int npix, const double* images, double* field) {
    if (g->counts || npix != 2 * g->n_rings)
        return 2;
    const int slices = g->volume ? g->n_slices : 1;
    const uint64_t per_slice = orc_cells_per_slice(g);
    const size_t npx = (size_t)npix * npix;
    uint32_t* map = (uint32_t*)malloc(sizeof(uint32_t) * npx);
    orc_uspg_to_cg_map(npix, map);
    for (int s = 0; s < slices; ++s)
        for (size_t f = 0; f < npx; ++f)
            field[(size_t)s * per_slice + f] = images[(size_t)s * npx + map[f]];
    free(map);
    return 0;
}

/* ---- metrics (src/metrics.cpp:42-50,105-136) ---------------------------- */

double orc_rmse(size_t n, const double* a, const double* b) {
    double acc = 0;
    for (size_t i = 0; i < n; ++i) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    return sqrt(acc / n);
}

double orc_ssim(int rows, int cols, const double* ref, const double* test, double dynamic_range) {
    double L = dynamic_range;
    if (!(L > 0)) {
        double lo = ref[0], hi = ref[0];
        for (size_t i = 0; i < (size_t)rows * cols; ++i) {
            if (ref[i] < lo)
                lo = ref[i];
            if (ref[i] > hi)
                hi = ref[i];
        }
        L = hi - lo > 0 ? hi - lo : 1.0;
    }
    const double c1 = (0.01 * L) * (0.01 * L);
    const double c2 = (0.03 * L) * (0.03 * L);
    const int W = 8;
    const double inv_n = 1.0 / (W * W);
    double acc = 0;
    for (int r0 = 0; r0 + W <= rows; ++r0)
        for (int c0 = 0; c0 + W <= cols; ++c0) {
            double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
            for (int r = r0; r < r0 + W; ++r) {
                const double* a = ref + (size_t)r * cols + c0;
                const double* b = test + (size_t)r * cols + c0;
                for (int q = 0; q < W; ++q) {
                    sx += a[q];
                    sy += b[q];
                    sxx += a[q] * a[q];
                    syy += b[q] * b[q];
                    sxy += a[q] * b[q];
                }
            }
            const double mx = sx * inv_n, my = sy * inv_n;
            const double vx = sxx * inv_n - mx * mx;
            const double vy = syy * inv_n - my * my;
            const double cov = sxy * inv_n - mx * my;
            acc += ((2 * mx * my + c1) * (2 * cov + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
        }
    const size_t windows = (size_t)(rows - W + 1) * (size_t)(cols - W + 1);
    return acc / windows;
}

/* sharpness (src/metrics.cpp:138-152): mean central-difference gradient
   magnitude, the neighbours clamped to the image and divided by their
   distance; NAN below 2x2 (the reference throws) */
double orc_sharpness(int rows, int cols, const double* img) {
    if (rows < 2 || cols < 2)
        return NAN;
    double acc = 0;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const int cl = c > 0 ? c - 1 : 0, ch = c + 1 < cols ? c + 1 : cols - 1;
            const int rl = r > 0 ? r - 1 : 0, rh = r + 1 < rows ? r + 1 : rows - 1;
            const double gx = (img[(size_t)r * cols + ch] - img[(size_t)r * cols + cl]) / (ch - cl);
            const double gy = (img[(size_t)rh * cols + c] - img[(size_t)rl * cols + c]) / (rh - rl);
            acc += sqrt(gx * gx + gy * gy);
        }
    return acc / ((size_t)rows * cols);
}

/* ---- libm probes for the device-math parity tests ------------------------ */
void orc_math(size_t n, const double* x, const double* y, double* out) {
    for (size_t i = 0; i < n; ++i) {
        out[3 * i + 0] = atan2(y[i], x[i]);
        out[3 * i + 1] = hypot(x[i], y[i]);
        out[3 * i + 2] = orc_azimuth_deg(x[i], y[i]);
    }
}
