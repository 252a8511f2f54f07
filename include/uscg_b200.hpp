// uscg_b200.hpp — C++ mirror of the reference library's reconstruction API
// (namespace uscg, /root/reference/proj/include/uscg/{grid,scan,tracer,solver,
// phantom}.hpp) on top of the C ABI in uscg_b200.h. Same type and function
// names, same argument meaning, same exception types (std::invalid_argument,
// std::domain_error), so code written against uscg:: switches by changing the
// namespace. Fields and projections keep the reference's std::vector<double>
// value semantics; the device computes in fp32.
//
//   reference                                   here
//   uscg::GridSpec          grid.hpp:21-44       uscg_b200::GridSpec (+ ring_counts, n_slices)
//   uscg::ScanGeometry      scan.hpp:21-41       uscg_b200::ScanGeometry (+ detector, view_angles)
//   uscg::Tracer            tracer.hpp:85-105    uscg_b200::Tracer (device-resident cache)
//   uscg::reconstruct       solver.hpp:78-79     uscg_b200::reconstruct
//   uscg::reconstruct_from  solver.hpp:82-83     uscg_b200::reconstruct_from
//   uscg::generate_projections phantom.hpp:51-52 uscg_b200::generate_projections (Binary)
//   uscg::field_to_cartesian   phantom.hpp:56    uscg_b200::field_to_cartesian
//   uscg::uspg_to_cg_map       grid.hpp:84       uscg_b200::uspg_to_cg_map
//   uscg::cartesian_to_field   phantom.hpp:59    uscg_b200::cartesian_to_field
//   uscg::Image, mae, rmse, ssim, sharpness, intensity_profile, area_average
//                              metrics.hpp:9-33  uscg_b200:: (same names)
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "uscg_b200.h"

namespace uscg_b200 {

struct NoDevice : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(uscg_status s) {
    switch (s) {
        case USCG_OK: return;
        case USCG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(uscg_last_error());
        case USCG_ERR_DOMAIN: throw std::domain_error(uscg_last_error());
        case USCG_ERR_NO_DEVICE: throw NoDevice(uscg_last_error());
        default: throw std::runtime_error(uscg_last_error());
    }
}

enum class GridMode { Slice2D, Volume3D };

struct GridSpec {
    int n = 0;
    double ring_spacing = 0;
    double slice_height = 0;
    GridMode mode = GridMode::Slice2D;
    std::vector<uint32_t> ring_counts;  // empty: the reference 4(2k-1) law
    int n_slices = 0;                   // 0: n slices in 3D (the reference default)

    static GridSpec square_2d(int n) { return GridSpec{n, 2.0 / n, 2.0 / n, GridMode::Slice2D, {}, 0}; }
    static GridSpec cube_3d(int n) { return GridSpec{n, 2.0 / n, 2.0 / n, GridMode::Volume3D, {}, 0}; }
    int rings() const { return n / 2; }
    int slices() const { return mode == GridMode::Volume3D ? (n_slices ? n_slices : n) : 1; }
    double radius() const { return 0.5 * n * ring_spacing; }
    std::size_t cells_per_slice() const {
        if (ring_counts.empty())
            return std::size_t(n) * std::size_t(n);
        std::size_t s = 0;
        for (uint32_t c : ring_counts)
            s += c;
        return s;
    }
    std::size_t cell_count() const { return cells_per_slice() * std::size_t(slices()); }
    uscg_grid c_grid() const {
        return uscg_grid{rings(), ring_spacing, slices(), slice_height,
                         mode == GridMode::Volume3D ? 1 : 0,
                         ring_counts.empty() ? nullptr : ring_counts.data()};
    }
};

struct Point3 {
    double x = 0, y = 0, z = 0;
};

enum class Detector { Flat = USCG_DET_FLAT, Arc = USCG_DET_ARC, Parallel = USCG_DET_PARALLEL };

struct ScanGeometry {
    Point3 source;
    Point3 detector_center;
    int det_u = 1;
    int det_v = 1;
    double spacing_u = 0;
    double spacing_v = 0;
    int views = 1;
    Detector detector = Detector::Flat;
    std::vector<double> view_angles;  // empty: view * 360 / views

    double step_deg() const { return 360.0 / views; }
    int lines() const { return det_u * det_v; }
    uscg_scan c_scan() const {
        uscg_scan s{};
        s.detector = int32_t(detector);
        s.source[0] = source.x;
        s.source[1] = source.y;
        s.source[2] = source.z;
        s.detector_center[0] = detector_center.x;
        s.detector_center[1] = detector_center.y;
        s.detector_center[2] = detector_center.z;
        s.det_u = det_u;
        s.det_v = det_v;
        s.spacing_u = spacing_u;
        s.spacing_v = spacing_v;
        s.views = views;
        s.view_angles_deg = view_angles.empty() ? nullptr : view_angles.data();
        return s;
    }
};

class Context {
public:
    explicit Context(int device = 0) { check(uscg_ctx_create(device, &h_)); }
    ~Context() { uscg_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    uscg_ctx get() const { return h_; }
    static Context& shared() {
        static Context c(0);
        return c;
    }

private:
    uscg_ctx h_ = nullptr;
};

class Tracer {
public:
    Tracer(const ScanGeometry& geom, const GridSpec& spec, bool quarter_symmetry, int threads = 1,
           Context& ctx = Context::shared())
        : geom_(geom), spec_(spec) {
        (void)threads;  // the device generator has no host thread pool
        const uscg_grid g = spec_.c_grid();
        const uscg_scan s = geom_.c_scan();
        uscg_tracer t = nullptr;
        check(uscg_tracer_create(ctx.get(), &g, &s, quarter_symmetry ? 1 : 0, &t));
        h_.reset(t);
    }
    const ScanGeometry& geometry() const { return geom_; }
    const GridSpec& spec() const { return spec_; }
    uscg_tracer get() const { return h_.get(); }

    /// Tracer::trace_line (tracer.hpp:97-98); the scratch is on the device.
    void trace_line(int line, double theta_deg, std::vector<uint32_t>& out) const {
        uscg_tracer_info info{};
        check(uscg_tracer_get_info(h_.get(), &info));
        out.resize(std::size_t(info.max_line_cells + info.max_line_records + 1));
        int64_t n = 0;
        check(uscg_trace_line(h_.get(), line, theta_deg, out.data(), int64_t(out.size()), &n));
        out.resize(std::size_t(n));
    }

    /// Rotated reuse: |active| and the index sum of every line of every view
    /// ([view][line]), without materialising the index lists.
    void trace_checksums(std::vector<uint32_t>& counts, std::vector<uint64_t>& sums) const {
        uscg_tracer_info info{};
        check(uscg_tracer_get_info(h_.get(), &info));
        const std::size_t n = std::size_t(info.views) * std::size_t(info.lines);
        counts.resize(n);
        sums.resize(n);
        check(uscg_trace_checksums(h_.get(), 0, info.views, counts.data(), sums.data(), 0));
    }

private:
    struct Del {
        void operator()(uscg_tracer t) const { uscg_tracer_destroy(t); }
    };
    ScanGeometry geom_;
    GridSpec spec_;
    std::unique_ptr<uscg_tracer_s, Del> h_;
};

struct Field {
    GridSpec spec;
    std::vector<double> values;
    static Field constant(const GridSpec& spec, double v) { return {spec, std::vector<double>(spec.cell_count(), v)}; }
};

struct ProjectionSet {
    ScanGeometry geometry;
    std::vector<double> data;  // view-major, then line
    double at(int view, int line) const { return data[std::size_t(view) * geometry.lines() + line]; }
};

/// Update form: Linear is the reference's 1 - beta (1 - m/p) (solver.cpp:41);
/// Power the multiplicative (m/p)^beta (USCG_UPDATE_POWER, an extension)
enum class UpdateForm { Linear, Power };

struct SolverConfig {
    double beta = 0.4;
    double tolerance = 1e-6;
    int max_sweeps = 100;
    double f_init = 1.0;
    double p_floor = 0;
    UpdateForm update = UpdateForm::Linear;
};

struct ReconReport {
    std::vector<double> sweep_residuals;
    int sweeps = 0;
    bool converged = false;
    bool all_zero_data = false;
    double seconds = 0;
    uint64_t zero_measurement_skips = 0;
    uint64_t factor_clamps = 0;
    uint64_t updates = 0;
    std::vector<uint8_t> crossed;
};

struct ReconResult {
    Field field;
    ReconReport report;
};

namespace detail {
inline ReconResult run(const ProjectionSet& proj, const GridSpec& spec, const SolverConfig& cfg,
                       const Tracer& tracer, const std::vector<double>* init) {
    const std::size_t cells = spec.cell_count();
    std::vector<float> p(proj.data.begin(), proj.data.end());
    std::vector<float> f(cells);
    if (init)
        f.assign(init->begin(), init->end());
    ReconResult r;
    r.report.sweep_residuals.assign(std::size_t(cfg.max_sweeps > 0 ? cfg.max_sweeps : 1), 0.0);
    r.report.crossed.assign(cells, 0);
    uscg_report rep{};
    rep.sweep_residuals = r.report.sweep_residuals.data();
    rep.crossed = r.report.crossed.data();
    const uscg_solver_config c{cfg.beta, cfg.tolerance, cfg.max_sweeps, cfg.f_init, cfg.p_floor};
    check(uscg_reconstruct(tracer.get(), p.data(), 1, &c, f.data(), init ? 1 : 0, &rep,
                           cfg.update == UpdateForm::Power ? uint32_t(USCG_UPDATE_POWER) : 0u));
    r.field = Field{spec, std::vector<double>(f.begin(), f.end())};
    r.report.sweeps = rep.sweeps;
    r.report.converged = rep.converged != 0;
    r.report.all_zero_data = rep.all_zero_data != 0;
    r.report.seconds = rep.seconds;
    r.report.zero_measurement_skips = rep.zero_measurement_skips;
    r.report.factor_clamps = rep.factor_clamps;
    r.report.updates = rep.updates;
    r.report.sweep_residuals.resize(cfg.tolerance > 0 ? std::size_t(rep.sweeps) : 0);
    return r;
}
}  // namespace detail

/// reconstruct (solver.cpp:166-169)
inline ReconResult reconstruct(const ProjectionSet& proj, const GridSpec& spec, const SolverConfig& cfg,
                               const Tracer& tracer) {
    return detail::run(proj, spec, cfg, tracer, nullptr);
}

/// reconstruct_from (solver.cpp:171-177)
inline ReconResult reconstruct_from(const ProjectionSet& proj, const Field& init, const SolverConfig& cfg,
                                    const Tracer& tracer) {
    for (double v : init.values)
        if (!(v > 0))
            throw std::invalid_argument("initial field must be strictly positive");
    return detail::run(proj, init.spec, cfg, tracer, &init.values);
}

/// generate_projections, Binary model (phantom.cpp:182-211)
inline ProjectionSet generate_projections(const Field& field, const ScanGeometry& geom, const Tracer& tracer) {
    std::vector<float> f(field.values.begin(), field.values.end());
    std::vector<float> out(std::size_t(geom.views) * geom.lines());
    check(uscg_project(tracer.get(), f.data(), 1, out.data(), 0));
    return ProjectionSet{geom, std::vector<double>(out.begin(), out.end())};
}

/// Image (metrics.hpp:9-16): rows x cols, row-major, row 0 at the bottom
struct Image {
    int rows = 0;
    int cols = 0;
    std::vector<double> v;

    double at(int row, int col) const { return v[std::size_t(row) * cols + col]; }
    double& at(int row, int col) { return v[std::size_t(row) * cols + col]; }
};

/// field_to_cartesian (phantom.cpp:149-163): one n x n Image per slice
inline std::vector<Image> field_to_cartesian(const Field& field, Context& ctx = Context::shared()) {
    const GridSpec& s = field.spec;
    const int npix = s.n;
    std::vector<float> f(field.values.begin(), field.values.end());
    std::vector<float> out(std::size_t(s.slices()) * npix * npix);
    const uscg_grid g = s.c_grid();
    check(uscg_resample(ctx.get(), &g, f.data(), 1, npix, out.data(), 0));
    std::vector<Image> imgs(std::size_t(s.slices()));
    for (int k = 0; k < s.slices(); ++k)
        imgs[k] = Image{npix, npix,
                        std::vector<double>(out.begin() + std::size_t(k) * npix * npix,
                                            out.begin() + std::size_t(k + 1) * npix * npix)};
    return imgs;
}

/// cartesian_to_field (phantom.cpp:165-180): the inverse permutation, on the device
inline Field cartesian_to_field(const std::vector<Image>& slices, const GridSpec& spec,
                                Context& ctx = Context::shared()) {
    if (int(slices.size()) != spec.slices())
        throw std::invalid_argument("slice count does not match the grid");
    const int npix = slices.empty() ? 0 : slices[0].rows;
    std::vector<float> in;
    in.reserve(std::size_t(spec.slices()) * npix * npix);
    for (const Image& img : slices) {
        if (img.rows != npix || img.cols != npix || img.v.size() != std::size_t(npix) * npix)
            throw std::invalid_argument("slice shape does not match the grid");
        in.insert(in.end(), img.v.begin(), img.v.end());
    }
    std::vector<float> out(spec.cell_count());
    const uscg_grid g = spec.c_grid();
    check(uscg_cartesian_to_field(ctx.get(), &g, in.data(), 1, npix, out.data(), 0));
    return Field{spec, std::vector<double>(out.begin(), out.end())};
}

namespace detail {
inline void metrics_of(const Image& ref, const Image& test, double* mae_o, double* rmse_o, double* ssim_o,
                       double dynamic_range, Context& ctx) {
    if (ref.rows != test.rows || ref.cols != test.cols || ref.v.size() != test.v.size())
        throw std::invalid_argument("image shapes differ");
    std::vector<float> a(ref.v.begin(), ref.v.end()), b(test.v.begin(), test.v.end());
    check(uscg_image_metrics(ctx.get(), a.data(), b.data(), 1, ref.rows, ref.cols, 0, dynamic_range, mae_o, rmse_o,
                             ssim_o, 0));
}
}  // namespace detail

/// mae / rmse / ssim (metrics.cpp:35-60,105-136) on the device
inline double mae(const Image& ref, const Image& test, Context& ctx = Context::shared()) {
    double m = 0;
    detail::metrics_of(ref, test, &m, nullptr, nullptr, -1, ctx);
    return m;
}
inline double rmse(const Image& ref, const Image& test, Context& ctx = Context::shared()) {
    double r = 0;
    detail::metrics_of(ref, test, nullptr, &r, nullptr, -1, ctx);
    return r;
}
inline double ssim(const Image& ref, const Image& test, double dynamic_range = -1, Context& ctx = Context::shared()) {
    double v = 0;
    detail::metrics_of(ref, test, nullptr, nullptr, &v, dynamic_range, ctx);
    return v;
}
/// area_average (metrics.cpp:62-69), host
inline double area_average(const Image& image) {
    if (image.v.empty())
        throw std::invalid_argument("empty image");
    double acc = 0;
    for (double x : image.v)
        acc += x;
    return acc / double(image.v.size());
}
/// sharpness (metrics.cpp:138-152) on the device
inline double sharpness(const Image& image, Context& ctx = Context::shared()) {
    if (image.v.size() != std::size_t(image.rows) * std::size_t(image.cols > 0 ? image.cols : 0))
        throw std::invalid_argument("image size does not match rows x cols");
    std::vector<float> a(image.v.begin(), image.v.end());
    double out = 0;
    check(uscg_image_sharpness(ctx.get(), a.data(), 1, image.rows, image.cols, &out, 0));
    return out;
}
/// intensity_profile (metrics.cpp:154-159)
inline std::vector<double> intensity_profile(const Image& image, int row) {
    if (row < 0 || row >= image.rows)
        throw std::invalid_argument("profile row out of range");
    return {image.v.begin() + std::size_t(row) * image.cols, image.v.begin() + std::size_t(row + 1) * image.cols};
}

/// uspg_to_cg_map (grid.hpp:84)
inline std::vector<uint32_t> uspg_to_cg_map(int n, Context& ctx = Context::shared()) {
    std::vector<uint32_t> m(n > 0 ? std::size_t(n) * n : 0);
    check(uscg_uspg_to_cg_map(ctx.get(), n, m.data()));
    return m;
}

}  // namespace uscg_b200
