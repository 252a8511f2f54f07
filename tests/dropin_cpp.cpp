// The INTEGRATION.md §2 caller, verbatim in shape: the reference's
// Tracer -> reconstruct -> field_to_cartesian sequence (proj/src/cli.cpp:235-311)
// with namespace uscg switched to uscg_b200. Used by tests/test_dropin_cpp.py,
// which compares its outputs with the unmodified reference library.
//
//   dropin_cpp <out prefix> <sweeps>
// writes <prefix>.proj (f64 views x lines), <prefix>.field (f64 cells),
// <prefix>.img (f64 slices x n x n) and <prefix>.rep (sweeps updates skips clamps).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "uscg_b200.hpp"

namespace U = uscg_b200;

static void dump(const std::string& path, const std::vector<double>& v) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f || std::fwrite(v.data(), sizeof(double), v.size(), f) != v.size())
        std::exit(3);
    std::fclose(f);
}

int main(int argc, char** argv) {
    if (argc < 3)
        return 2;
    const std::string out = argv[1];
    const int sweeps = std::atoi(argv[2]);

    U::GridSpec spec = U::GridSpec::cube_3d(64);
    U::ScanGeometry geom;
    geom.source = {-3, 0, 0};
    geom.detector_center = {10, 0, 0};
    geom.det_u = geom.det_v = 101;
    geom.spacing_u = 0.092;
    geom.spacing_v = 0.13;
    geom.views = 70;
    U::Tracer tracer(geom, spec, /*quarter_symmetry=*/true);

    // a smooth positive phantom sampled per cell (flat index order)
    U::Field truth = U::Field::constant(spec, 0.0);
    for (std::size_t i = 0; i < truth.values.size(); ++i)
        truth.values[i] = 0.5 + 0.4 * std::sin(0.001 * double(i)) * std::cos(0.00037 * double(i));
    U::ProjectionSet proj = U::generate_projections(truth, geom, tracer);

    U::SolverConfig cfg;
    cfg.beta = 0.4;
    cfg.tolerance = 0;
    cfg.max_sweeps = sweeps;
    U::ReconResult r = U::reconstruct(proj, spec, cfg, tracer);
    auto images = U::field_to_cartesian(r.field);

    bool threw = false;  // the reference's exception type for invalid input
    try {
        U::SolverConfig bad = cfg;
        bad.beta = 2.5;
        U::reconstruct(proj, spec, bad, tracer);
    } catch (const std::invalid_argument&) {
        threw = true;
    }

    std::vector<double> img;
    for (const auto& s : images)
        img.insert(img.end(), s.v.begin(), s.v.end());

    // the metrics.hpp / phantom.hpp names on the rasters: cartesian_to_field
    // (the inverse permutation), sharpness, intensity_profile, rmse, ssim
    const U::Field back = U::cartesian_to_field(images, spec);
    const std::vector<double> prof = U::intensity_profile(images[32], 10);
    std::vector<double> extra = {U::sharpness(images[32]), U::rmse(images[31], images[32]),
                                 U::ssim(images[31], images[32]), U::mae(images[31], images[32]),
                                 U::area_average(images[32])};
    extra.insert(extra.end(), prof.begin(), prof.end());
    dump(out + ".back", back.values);
    dump(out + ".extra", extra);
    dump(out + ".proj", proj.data);
    dump(out + ".field", r.field.values);
    dump(out + ".img", img);
    FILE* f = std::fopen((out + ".rep").c_str(), "w");
    std::fprintf(f, "%d %llu %llu %llu %d %zu\n", r.report.sweeps, (unsigned long long)r.report.updates,
                 (unsigned long long)r.report.zero_measurement_skips, (unsigned long long)r.report.factor_clamps,
                 threw ? 1 : 0, images.size());
    std::fclose(f);
    return 0;
}
