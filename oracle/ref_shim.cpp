// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (uscg_core), compiled
// from the sources where they lie under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libuscg_ref.so. Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference leg load it, as the checker or the
// CPU baseline. Every entry point forwards to the reference API it names:
//
//   ref_tracer_create      -> uscg::Tracer::Tracer           proj/include/uscg/tracer.hpp:87
//   ref_cache_*            -> uscg::FirstViewCache           proj/include/uscg/tracer.hpp:18-39
//   ref_trace_line         -> uscg::Tracer::trace_line       proj/src/tracer.cpp:148-201
//   ref_trace_chord        -> uscg::trace_chord              proj/src/tracer.cpp:104-142
//   ref_project_binary     -> uscg::generate_projections     proj/src/phantom.cpp:182-211
//   ref_project_length     -> uscg::generate_projections LW  proj/src/phantom.cpp:213-269
//   ref_reconstruct        -> uscg::reconstruct(_from)       proj/src/solver.cpp:166-177
//   ref_mart_update_line   -> uscg::mart_update_line         proj/src/solver.cpp:33-51
//   ref_uspg_to_cg_map     -> uscg::uspg_to_cg_map           proj/src/grid.cpp:75-99
//   ref_field_to_cartesian -> uscg::field_to_cartesian       proj/src/phantom.cpp:149-163
//   ref_rmse / ref_ssim    -> uscg::rmse / uscg::ssim        proj/src/metrics.cpp:42-50,105-136
//   ref_phantom            -> uscg::generate_phantom         proj/src/phantom.cpp:72-147
//
// Errors: every call returns 0 on success, 1 for std::invalid_argument,
// 2 for std::domain_error, 3 for anything else; ref_last_error() has the text.

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "uscg/grid.hpp"
#include "uscg/io.hpp"
#include "uscg/siddon.hpp"
#include "uscg/metrics.hpp"
#include "uscg/phantom.hpp"
#include "uscg/solver.hpp"
#include "uscg/tracer.hpp"

using namespace uscg;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

GridSpec make_spec(int n, double r, double h, int volume) {
    return GridSpec{n, r, h, volume ? GridMode::Volume3D : GridMode::Slice2D};
}

ScanGeometry make_geom(const double* src, const double* ctr, int det_u, int det_v, double su,
                       double sv, int views) {
    ScanGeometry g;
    g.source = {src[0], src[1], src[2]};
    g.detector_center = {ctr[0], ctr[1], ctr[2]};
    g.det_u = det_u;
    g.det_v = det_v;
    g.spacing_u = su;
    g.spacing_v = sv;
    g.views = views;
    return g;
}

struct RefTracer {
    std::unique_ptr<Tracer> tracer;
    std::unique_ptr<TraceScratch> scratch;
    std::vector<std::uint32_t> active;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_tracer_create(int n, double r, double h, int volume, const double* src, const double* ctr,
                      int det_u, int det_v, double su, double sv, int views, int quarter,
                      int threads, void** out) {
    return guarded([&] {
        auto* t = new RefTracer;
        t->tracer = std::make_unique<Tracer>(make_geom(src, ctr, det_u, det_v, su, sv, views),
                                             make_spec(n, r, h, volume), quarter != 0, threads);
        t->scratch = std::make_unique<TraceScratch>(t->tracer->make_scratch());
        *out = t;
    });
}

void ref_tracer_destroy(void* h) { delete static_cast<RefTracer*>(h); }

std::uint64_t ref_cache_records(void* h) {
    return static_cast<RefTracer*>(h)->tracer->cache().record_count();
}

std::uint64_t ref_cache_bytes(void* h) { return static_cast<RefTracer*>(h)->tracer->cache().byte_size(); }

int ref_cache_lines(void* h) { return static_cast<RefTracer*>(h)->tracer->cache().line_count(); }

// offsets: lines+1 u32; phi_a/phi_b: records f64; slice/ring: records u16
void ref_cache_export(void* h, std::uint32_t* offsets, double* phi_a, double* phi_b,
                      std::uint16_t* slice, std::uint16_t* ring) {
    const FirstViewCache& c = static_cast<RefTracer*>(h)->tracer->cache();
    auto off = c.offsets();
    std::memcpy(offsets, off.data(), off.size() * sizeof(std::uint32_t));
    auto recs = c.records();
    for (std::size_t i = 0; i < recs.size(); ++i) {
        phi_a[i] = recs[i].phi_a;
        phi_b[i] = recs[i].phi_b;
        slice[i] = recs[i].slice;
        ring[i] = recs[i].ring;
    }
}

// Returns the number of active cells; copies min(n, cap) of them to out.
// chords/cells receive the TraceScratch counters accumulated so far.
std::int64_t ref_trace_line(void* h, int line, double theta_deg, std::uint32_t* out, std::int64_t cap,
                            std::uint64_t* chords, std::uint64_t* cells) {
    auto* t = static_cast<RefTracer*>(h);
    t->tracer->trace_line(line, theta_deg, *t->scratch, t->active);
    const std::int64_t n = static_cast<std::int64_t>(t->active.size());
    const std::int64_t m = n < cap ? n : cap;
    if (m > 0)
        std::memcpy(out, t->active.data(), std::size_t(m) * sizeof(std::uint32_t));
    if (chords)
        *chords = t->scratch->chords;
    if (cells)
        *cells = t->scratch->cells;
    return n;
}

std::int64_t ref_trace_chord(int n, double r, double h, int volume, double phi_a, double phi_b,
                             int slice, int ring, double theta_deg, std::uint32_t* out,
                             std::int64_t cap) {
    std::vector<std::uint32_t> v;
    const GridSpec spec = make_spec(n, r, h, volume);
    const RingTable rings(spec);
    trace_chord(SegmentRecord{phi_a, phi_b, static_cast<std::uint16_t>(slice),
                              static_cast<std::uint16_t>(ring)},
                theta_deg, spec, rings, v);
    const std::int64_t k = static_cast<std::int64_t>(v.size());
    for (std::int64_t i = 0; i < k && i < cap; ++i)
        out[i] = v[i];
    return k;
}

// field: cell_count f64; out: views*lines f64
int ref_project_binary(void* h, const double* field, double* out) {
    return guarded([&] {
        auto* t = static_cast<RefTracer*>(h);
        const GridSpec& spec = t->tracer->spec();
        Field f{spec, std::vector<double>(field, field + spec.cell_count())};
        ProjectionSet p = generate_projections(f, t->tracer->geometry(), ForwardModel::Binary,
                                               t->tracer.get());
        std::memcpy(out, p.data.data(), p.data.size() * sizeof(double));
    });
}

int ref_project_length(void* h, const double* field, double* out) {
    return guarded([&] {
        auto* t = static_cast<RefTracer*>(h);
        const GridSpec& spec = t->tracer->spec();
        Field f{spec, std::vector<double>(field, field + spec.cell_count())};
        ProjectionSet p =
            generate_projections(f, t->tracer->geometry(), ForwardModel::LengthWeighted, nullptr);
        std::memcpy(out, p.data.data(), p.data.size() * sizeof(double));
    });
}

// report: [0]=sweeps [1]=converged [2]=all_zero [3]=seconds [4]=skips [5]=clamps
// residuals: max_sweeps f64 (may be null); crossed: cell_count u8 (may be null)
int ref_reconstruct(void* h, const double* proj, const double* init, double beta, double tolerance,
                    int max_sweeps, double f_init, double p_floor, double* field_out,
                    double* report, double* residuals, std::uint8_t* crossed) {
    return guarded([&] {
        auto* t = static_cast<RefTracer*>(h);
        const GridSpec& spec = t->tracer->spec();
        ProjectionSet p;
        p.geometry = t->tracer->geometry();
        p.data.assign(proj, proj + std::size_t(p.geometry.views) * p.geometry.lines());
        SolverConfig cfg;
        cfg.beta = beta;
        cfg.tolerance = tolerance;
        cfg.max_sweeps = max_sweeps;
        cfg.f_init = f_init;
        cfg.p_floor = p_floor;
        ReconResult res;
        if (init) {
            Field f0{spec, std::vector<double>(init, init + spec.cell_count())};
            res = reconstruct_from(p, f0, cfg, *t->tracer);
        } else {
            res = reconstruct(p, spec, cfg, *t->tracer);
        }
        std::memcpy(field_out, res.field.values.data(), res.field.values.size() * sizeof(double));
        report[0] = res.report.sweeps;
        report[1] = res.report.converged;
        report[2] = res.report.all_zero_data;
        report[3] = res.report.seconds;
        report[4] = double(res.report.zero_measurement_skips);
        report[5] = double(res.report.factor_clamps);
        if (residuals)
            for (std::size_t i = 0; i < res.report.sweep_residuals.size(); ++i)
                residuals[i] = res.report.sweep_residuals[i];
        if (crossed)
            std::memcpy(crossed, res.report.crossed.data(), res.report.crossed.size());
    });
}

// returns bit0 = skipped, bit1 = clamped
int ref_mart_update_line(int n, double* field, std::int64_t cells, const std::uint32_t* active,
                         std::int64_t count, double p_meas, double beta, double p_floor) {
    Field f{GridSpec::square_2d(n), std::vector<double>(field, field + cells)};
    UpdateDiag d = mart_update_line(f, std::span<const std::uint32_t>(active, std::size_t(count)),
                                    p_meas, beta, p_floor);
    std::memcpy(field, f.values.data(), std::size_t(cells) * sizeof(double));
    return (d.skipped ? 1 : 0) | (d.clamped ? 2 : 0);
}

int ref_uspg_to_cg_map(int n, std::uint32_t* out) {
    return guarded([&] {
        auto m = uspg_to_cg_map(n);
        std::memcpy(out, m.data(), m.size() * sizeof(std::uint32_t));
    });
}

// field: cell_count f64 -> out: slices*n*n f64 (row 0 at the bottom)
int ref_field_to_cartesian(int n, double r, double h, int volume, const double* field, double* out) {
    return guarded([&] {
        const GridSpec spec = make_spec(n, r, h, volume);
        Field f{spec, std::vector<double>(field, field + spec.cell_count())};
        auto imgs = field_to_cartesian(f);
        for (std::size_t s = 0; s < imgs.size(); ++s)
            std::memcpy(out + s * spec.cells_per_slice(), imgs[s].v.data(),
                        imgs[s].v.size() * sizeof(double));
    });
}

// images: slices*n*n f64 (row 0 at the bottom) -> field cell_count f64
int ref_cartesian_to_field(int n, double r, double h, int volume, int img_n, const double* images,
                           double* field) {
    return guarded([&] {
        const GridSpec spec = make_spec(n, r, h, volume);
        std::vector<Image> slices;
        for (int s = 0; s < spec.slices(); ++s)
            slices.push_back(Image{img_n, img_n,
                                   std::vector<double>(images + std::size_t(s) * img_n * img_n,
                                                       images + std::size_t(s + 1) * img_n * img_n)});
        const Field f = cartesian_to_field(slices, spec);
        std::memcpy(field, f.values.data(), f.values.size() * sizeof(double));
    });
}

// sharpness of one image; *out receives the value (errors: status 1 + message)
int ref_sharpness(int rows, int cols, const double* a, double* out) {
    return guarded([&] {
        Image ia{rows, cols, std::vector<double>(a, a + std::size_t(std::max(rows, 0)) * std::max(cols, 0))};
        *out = sharpness(ia);
    });
}

int ref_intensity_profile(int rows, int cols, const double* a, int row, double* out) {
    return guarded([&] {
        Image ia{rows, cols, std::vector<double>(a, a + std::size_t(rows) * cols)};
        const std::vector<double> p = intensity_profile(ia, row);
        std::memcpy(out, p.data(), p.size() * sizeof(double));
    });
}

double ref_rmse(int rows, int cols, const double* a, const double* b) {
    Image ia{rows, cols, std::vector<double>(a, a + std::size_t(rows) * cols)};
    Image ib{rows, cols, std::vector<double>(b, b + std::size_t(rows) * cols)};
    return rmse(ia, ib);
}

double ref_ssim(int rows, int cols, const double* a, const double* b, double dynamic_range) {
    Image ia{rows, cols, std::vector<double>(a, a + std::size_t(rows) * cols)};
    Image ib{rows, cols, std::vector<double>(b, b + std::size_t(rows) * cols)};
    return ssim(ia, ib, dynamic_range, 1);
}

// kind 0 = Shepp-Logan 2D, 1 = Shepp-Logan 3D; out: cell_count f64
int ref_phantom(int n, double r, double h, int volume, int kind, double* out) {
    return guarded([&] {
        const GridSpec spec = make_spec(n, r, h, volume);
        PhantomSpec ph;
        ph.kind = kind == 1 ? PhantomKind::SheppLogan3D : PhantomKind::SheppLogan2D;
        ph.n = n;
        PhantomResult res = generate_phantom(ph, spec);
        std::memcpy(out, res.field.values.data(), res.field.values.size() * sizeof(double));
    });
}

// ---- file formats (proj/src/io.cpp): the reference's own writers, for the
// byte-for-byte format tests of include/uscg_b200_io.hpp. Sidecar entries come
// in as parallel key / value string arrays.
static Sidecar sidecar_of(const char* const* keys, const char* const* vals, int nkv) {
    Sidecar s;
    for (int i = 0; i < nkv; ++i)
        s.set(keys[i], std::string(vals[i]));
    return s;
}

int ref_write_field(const char* path, int n, double r, double h, int volume, const double* values,
                    const char* const* keys, const char* const* vals, int nkv) {
    return guarded([&] {
        Field f{make_spec(n, r, h, volume), {}};
        f.values.assign(values, values + f.spec.cell_count());
        write_field(path, f, sidecar_of(keys, vals, nkv));
    });
}

int ref_write_projections(const char* path, int views, int det_u, int det_v, double su, double sv,
                          const double* src, const double* ctr, const double* data,
                          const char* const* keys, const char* const* vals, int nkv) {
    return guarded([&] {
        ProjectionSet p;
        p.geometry.views = views;
        p.geometry.det_u = det_u;
        p.geometry.det_v = det_v;
        p.geometry.spacing_u = su;
        p.geometry.spacing_v = sv;
        p.geometry.source = {src[0], src[1], src[2]};
        p.geometry.detector_center = {ctr[0], ctr[1], ctr[2]};
        p.data.assign(data, data + std::size_t(views) * det_u * det_v);
        write_projections(path, p, sidecar_of(keys, vals, nkv));
    });
}

int ref_write_pgm16(const char* path, int rows, int cols, const double* v, double wmin, double wmax,
                    const char* const* keys, const char* const* vals, int nkv) {
    return guarded([&] {
        Image im{rows, cols, std::vector<double>(v, v + std::size_t(rows) * cols)};
        write_pgm16(path, im, wmin, wmax, sidecar_of(keys, vals, nkv));
    });
}

// rows, cols out; values (row 0 at the bottom, through the sidecar window) into out (cap doubles)
int ref_read_pgm16(const char* path, int* rows, int* cols, double* out, long long cap) {
    return guarded([&] {
        auto [im, side] = read_pgm16(path);
        *rows = im.rows;
        *cols = im.cols;
        if (static_cast<long long>(im.v.size()) <= cap)
            std::memcpy(out, im.v.data(), im.v.size() * sizeof(double));
    });
}

// ---- Cartesian comparator (proj/src/siddon.cpp) -------------------------
// CartesianSpec::like(GridSpec(n, r, h, mode)) and a ScanGeometry.
// system: counts (rows), entries out via offsets (rows+1, u64), idx, weight;
// call with idx == nullptr first to get the entry count in *entries.
int ref_cartesian_system(int n, double r, double h, int volume, const double* src, const double* ctr,
                         int det_u, int det_v, double su, double sv, int views, std::uint64_t* offsets,
                         std::uint32_t* idx, double* weight, std::uint64_t* entries) {
    return guarded([&] {
        const CartesianSpec c = CartesianSpec::like(make_spec(n, r, h, volume));
        const CartesianSystem sys = precompute_cartesian_system(make_geom(src, ctr, det_u, det_v, su, sv, views), c);
        *entries = sys.idx.size();
        if (!idx)
            return;
        std::memcpy(offsets, sys.offsets.data(), sys.offsets.size() * sizeof(std::uint64_t));
        std::memcpy(idx, sys.idx.data(), sys.idx.size() * sizeof(std::uint32_t));
        std::memcpy(weight, sys.weight.data(), sys.weight.size() * sizeof(double));
    });
}

// cartesian_mart_stored (stored != 0) or cartesian_mart_otf; out: voxel_count values
int ref_cartesian_mart(int n, double r, double h, int volume, const double* src, const double* ctr,
                       int det_u, int det_v, double su, double sv, int views, const double* proj,
                       double beta, int sweeps, double f_init, int stored, double* out, double* seconds) {
    return guarded([&] {
        const CartesianSpec c = CartesianSpec::like(make_spec(n, r, h, volume));
        ProjectionSet p;
        p.geometry = make_geom(src, ctr, det_u, det_v, su, sv, views);
        p.data.assign(proj, proj + std::size_t(views) * det_u * det_v);
        SolverConfig cfg;
        cfg.beta = beta;
        cfg.max_sweeps = sweeps;
        cfg.f_init = f_init;
        cfg.tolerance = 0;
        CartesianMartResult res = stored ? cartesian_mart_stored(p, c, precompute_cartesian_system(p.geometry, c), cfg)
                                         : cartesian_mart_otf(p, c, cfg);
        std::memcpy(out, res.values.data(), res.values.size() * sizeof(double));
        *seconds = res.seconds;
    });
}

}  // extern "C"
