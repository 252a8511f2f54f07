// uscg_b200: the reference's CLI pipeline (proj/src/cli.cpp) on the device path.
//
//   uscg_b200 phantom     --kind raw-volume|shepp-logan-2d|shepp-logan-3d --n N --out F.fld
//                         [--r R --h H --table T --raw RAW --raw-mode 2d|3d --cg P --pixel-raster P --no-cg]
//   uscg_b200 project     --field F.fld --out D.prj [--views --det-u --det-v --spacing-u --spacing-v
//                         --source x,y[,z] --center x,y[,z] --model binary|length]
//   uscg_b200 reconstruct --proj D.prj --out F.fld [--n --r --h --mode 2d|3d|auto --beta --tol
//                         --sweeps --f-init --quarter on|off|auto --report R]
//   uscg_b200 map         --field F.fld --out P.pgm [--window-min --window-max]
//   uscg_b200 metrics     --ref A.pgm --test B.pgm [--out R --profile-row K]
//   global: --threads N --seed S (recorded in the sidecars)
//
// Same subcommands, options, defaults, sidecar keys, file formats
// (include/uscg_b200_io.hpp) and exit codes (1: argument / I/O / domain
// error, 2: numerical or device error) as the reference, so its pipeline
// (proj/tests/test_io_cli.cpp:163-231) runs unchanged against this binary.
// Every compute step goes through the C ABI (include/uscg_b200.h): the
// generator, the projector, Sp-MART, the resampling and the image metrics run
// on the GPU. The built-in Shepp-Logan tables are not bundled: pass the
// reference's parameter files with --table.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "uscg_b200.h"
#include "uscg_b200_io.hpp"

namespace io = uscg_b200::io;

namespace {

struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct UsageError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

// status -> the reference's exception types
void check(uscg_status s) {
    if (s == USCG_OK)
        return;
    const std::string msg = uscg_last_error();
    if (s == USCG_ERR_INVALID_ARGUMENT)
        throw std::invalid_argument(msg);
    if (s == USCG_ERR_DOMAIN)
        throw std::domain_error(msg);
    throw DeviceError(msg);
}

uscg_ctx context() {
    static uscg_ctx ctx = [] {
        uscg_ctx c = nullptr;
        check(uscg_ctx_create(0, &c));
        return c;
    }();
    return ctx;
}

// ---- options ------------------------------------------------------------

struct Args {
    std::map<std::string, std::string> kv;
    std::vector<std::string> flags;
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    std::string req(const std::string& k) const {
        if (!has(k))
            throw UsageError(k + " is required");
        return kv.at(k);
    }
    double num(const std::string& k, double def) const {
        if (!has(k))
            return def;
        try {
            std::size_t used = 0;
            const double v = std::stod(kv.at(k), &used);
            if (used != kv.at(k).size())
                throw std::invalid_argument("");
            return v;
        } catch (const std::exception&) {
            throw UsageError(k + ": not a number: " + kv.at(k));
        }
    }
    int integer(const std::string& k, int def) const {
        const double v = num(k, def);
        if (v != std::floor(v))
            throw UsageError(k + ": not an integer: " + kv.at(k));
        return int(v);
    }
    bool flag(const std::string& f) const { return std::find(flags.begin(), flags.end(), f) != flags.end(); }
};

struct Globals {
    int threads = 1;
    std::int64_t seed = 0;
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& known,
           const std::vector<std::string>& known_flags, Globals& g) {
    Args a;
    for (int i = first; i < argc; ++i) {
        const std::string k = argv[i];
        if (std::find(known_flags.begin(), known_flags.end(), k) != known_flags.end()) {
            a.flags.push_back(k);
            continue;
        }
        const bool global = k == "--threads" || k == "--seed";
        if (!global && std::find(known.begin(), known.end(), k) == known.end())
            throw UsageError("unknown option " + k);
        if (i + 1 >= argc)
            throw UsageError(k + " needs a value");
        const std::string v = argv[++i];
        if (k == "--threads")
            g.threads = std::stoi(v);
        else if (k == "--seed")
            g.seed = std::stoll(v);
        else
            a.kv[k] = v;
    }
    return a;
}

std::vector<double> parse_point(const std::string& s, const std::string& name) {
    std::vector<double> v;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ','))
        v.push_back(std::stod(tok));
    if (v.size() == 2)
        v.push_back(0.0);
    if (v.size() != 3)
        throw UsageError(name + " needs 2 or 3 comma-separated coordinates");
    return v;
}

// ---- grid / geometry ------------------------------------------------------

struct Grid {
    int n = 0;
    double r = 0, h = 0;
    bool volume = false;
    int slices() const { return volume ? n : 1; }
    uscg_grid c() const { return uscg_grid{n / 2, r, slices(), h, volume ? 1 : 0, nullptr}; }
    std::size_t cells() const { return std::size_t(slices()) * n * n; }
    double radius() const { return 0.5 * n * r; }
};

// make_grid (cli.cpp) + GridSpec::validate (grid.cpp:9-16)
Grid make_grid(int n, double r, double h, bool volume) {
    if (n < 2 || n % 2 != 0)
        throw std::invalid_argument("grid size must be an even integer >= 2, got " + std::to_string(n));
    Grid g{n, r > 0 ? r : 2.0 / n, h > 0 ? h : 2.0 / n, volume};
    return g;
}

Grid grid_of(const io::FieldFile& f) { return Grid{f.n, f.ring_spacing, f.slice_height, f.mode == "3d"}; }

uscg_scan scan_of(const io::ProjFile& p) {
    uscg_scan s{};
    s.detector = USCG_DET_FLAT;
    for (int i = 0; i < 3; ++i) {
        s.source[i] = p.source[i];
        s.detector_center[i] = p.center[i];
    }
    s.det_u = p.det_u;
    s.det_v = p.det_v;
    s.spacing_u = p.spacing_u;
    s.spacing_v = p.spacing_v;
    s.views = p.views;
    s.view_angles_deg = nullptr;
    return s;
}

// ScanGeometry::quarter_symmetric (scan.cpp:44-48)
bool quarter_symmetric(const io::ProjFile& p) {
    if (p.det_u % 2 == 0 || p.det_v % 2 == 0)
        return false;
    return p.source[1] == 0 && p.source[2] == 0 && p.center[1] == 0 && p.center[2] == 0;
}

struct Tracer {
    uscg_tracer h = nullptr;
    Tracer(const Grid& g, const io::ProjFile& p, bool quarter) {
        const uscg_grid gc = g.c();
        const uscg_scan sc = scan_of(p);
        check(uscg_tracer_create(context(), &gc, &sc, quarter ? 1 : 0, &h));
    }
    ~Tracer() {
        if (h)
            uscg_tracer_destroy(h);
    }
    uscg_tracer_info info() const {
        uscg_tracer_info i{};
        check(uscg_tracer_get_info(h, &i));
        return i;
    }
};

// ---- rasters -----------------------------------------------------------

// field_to_cartesian (phantom.cpp:149-163) on the device
std::vector<io::Raster> to_cartesian(const Grid& g, const std::vector<double>& values) {
    std::vector<float> f(values.begin(), values.end());
    std::vector<float> img(std::size_t(g.slices()) * g.n * g.n);
    const uscg_grid gc = g.c();
    check(uscg_resample(context(), &gc, f.data(), 1, g.n, img.data(), 0));
    std::vector<io::Raster> out(g.slices());
    for (int s = 0; s < g.slices(); ++s) {
        out[s].rows = out[s].cols = g.n;
        out[s].v.assign(img.begin() + std::size_t(s) * g.n * g.n, img.begin() + std::size_t(s + 1) * g.n * g.n);
    }
    return out;
}

std::pair<double, double> value_range(const std::vector<double>& v) {
    const auto mm = std::minmax_element(v.begin(), v.end());
    double lo = *mm.first, hi = *mm.second;
    if (!(hi > lo))
        hi = lo + 1;
    return {lo, hi};
}

std::filesystem::path slice_path(const std::filesystem::path& base, int slice, int slices) {
    if (slices == 1)
        return base;
    char suffix[16];
    std::snprintf(suffix, sizeof suffix, "_s%03d", slice);
    std::filesystem::path p = base;
    const std::string ext = p.extension().string();
    p.replace_extension();
    return p.string() + suffix + ext;
}

void write_slices(const std::filesystem::path& base, const std::vector<io::Raster>& slices, double lo,
                  double hi, const io::Sidecar& echo) {
    for (std::size_t s = 0; s < slices.size(); ++s) {
        io::Sidecar side = echo;
        side.set("slice", std::int64_t(s));
        side.set("slices", std::int64_t(slices.size()));
        io::write_pgm16(slice_path(base, int(s), int(slices.size())), slices[s], lo, hi, side);
    }
}

// ---- phantom --------------------------------------------------------------

struct Ellipsoid {
    double intensity, ax, ay, az, cx, cy, cz, angle_deg;
};

// read_phantom_table (io.cpp:392-425)
std::pair<std::string, std::vector<Ellipsoid>> read_table(const std::string& path) {
    std::ifstream in(path);
    if (!in)
        throw io::IoError("cannot open " + path);
    std::string line;
    if (!std::getline(in, line) || line != "uscg-phantom-table v1")
        throw io::IoError(path + ": missing 'uscg-phantom-table v1' header line");
    std::string mode;
    std::vector<Ellipsoid> t;
    while (std::getline(in, line)) {
        if (line.empty() || line[0] == '#')
            continue;
        if (line.rfind("mode", 0) == 0) {
            const std::size_t eq = line.find('=');
            if (eq == std::string::npos)
                throw io::IoError(path + ": malformed mode line");
            mode = line.substr(eq + 1);
            mode.erase(std::remove(mode.begin(), mode.end(), ' '), mode.end());
            if (mode != "2d" && mode != "3d")
                throw io::IoError("unknown grid mode '" + mode + "'");
            continue;
        }
        std::istringstream row(line);
        Ellipsoid e;
        if (!(row >> e.intensity >> e.ax >> e.ay >> e.az >> e.cx >> e.cy >> e.cz >> e.angle_deg))
            throw io::IoError(path + ": malformed table row: " + line);
        t.push_back(e);
    }
    if (mode.empty())
        throw io::IoError(path + ": missing mode line");
    return {mode, t};
}

// phantom_value (phantom.cpp:45-66)
double phantom_value(const std::vector<Ellipsoid>& t, bool volume, double x, double y, double z) {
    const double k = 3.141592653589793238462643383279502884 / 180.0;
    double v = 0;
    for (const Ellipsoid& e : t) {
        const double px = x - e.cx, py = y - e.cy;
        const double c = std::cos(e.angle_deg * k), s = std::sin(e.angle_deg * k);
        const double qx = c * px + s * py, qy = -s * px + c * py;
        double q = (qx / e.ax) * (qx / e.ax) + (qy / e.ay) * (qy / e.ay);
        if (volume) {
            const double qz = (z - e.cz) / e.az;
            q += qz * qz;
        }
        if (q < 1.0)
            v += e.intensity;
    }
    return v;
}

int run_phantom(const Args& a, const Globals& g) {
    const std::string kind = a.str("--kind", "shepp-logan-2d");
    bool volume;
    if (kind == "shepp-logan-2d")
        volume = false;
    else if (kind == "shepp-logan-3d")
        volume = true;
    else if (kind == "raw-volume")
        volume = a.str("--raw-mode", "2d") == "3d";
    else
        throw std::invalid_argument("unknown phantom kind '" + kind + "'");
    std::vector<Ellipsoid> table;
    if (a.has("--table")) {
        auto mt = read_table(a.str("--table"));
        volume = mt.first == "3d";
        table = std::move(mt.second);
    } else if (kind != "raw-volume") {
        throw std::invalid_argument("the built-in Shepp-Logan tables are not bundled: pass --table "
                                    "(e.g. proj/data/shepp_logan_2d.params)");
    }
    const Grid gr = make_grid(a.integer("--n", 128), a.num("--r", 0), a.num("--h", 0), volume);
    const int n = gr.n, slices = gr.slices();
    io::FieldFile f;
    f.mode = volume ? "3d" : "2d";
    f.n = n;
    f.slices = slices;
    f.ring_spacing = gr.r;
    f.slice_height = gr.h;
    f.values.assign(gr.cells(), 0.0);
    std::vector<io::Raster> pixel(slices);
    bool clipped = false;
    if (kind == "raw-volume") {
        if (!a.has("--raw"))
            throw std::invalid_argument("raw-volume needs --raw with float32 data in Cartesian order");
        const std::vector<double> raw = io::read_raw_f32(a.str("--raw"), gr.cells());
        // cartesian_to_field (phantom.cpp:165-180): field[flat] = image[map[flat]]
        std::vector<uint32_t> map(std::size_t(n) * n);
        check(uscg_uspg_to_cg_map(context(), n, map.data()));
        for (int s = 0; s < slices; ++s) {
            const std::size_t o = std::size_t(s) * n * n;
            for (std::size_t k = 0; k < map.size(); ++k)
                f.values[o + k] = raw[o + map[k]];
            pixel[s].rows = pixel[s].cols = n;
            pixel[s].v.assign(raw.begin() + o, raw.begin() + o + std::size_t(n) * n);
        }
    } else {
        // cell-centroid samples (phantom.cpp:95-128), pixel-centre samples
        const double scale = gr.radius(), zoff = 0.5 * (volume ? n * gr.h : gr.h);
        auto sample = [&](double x, double y, double z) {
            double v = phantom_value(table, volume, x / scale, y / scale, z / scale);
            if (v < 0) {
                v = 0;
                clipped = true;
            }
            return v;
        };
        const double k = 3.141592653589793238462643383279502884 / 180.0;
        std::size_t flat = 0;
        for (int s = 0; s < slices; ++s) {
            const double z = volume ? (s + 0.5) * gr.h - zoff : 0.0;
            for (int ring = 1; ring <= n / 2; ++ring) {
                const int cnt = 4 * (2 * ring - 1);
                const double step = 360.0 / cnt, radius = (ring - 0.5) * gr.r;
                for (int j = 0; j < cnt; ++j) {
                    const double ang = (j + 0.5) * step * k;
                    f.values[flat++] = sample(radius * std::cos(ang), radius * std::sin(ang), z);
                }
            }
            pixel[s].rows = pixel[s].cols = n;
            pixel[s].v.resize(std::size_t(n) * n);
            for (int row = 0; row < n; ++row)
                for (int col = 0; col < n; ++col)
                    pixel[s].v[std::size_t(row) * n + col] =
                        sample((col + 0.5 - n / 2) * gr.r, (row + 0.5 - n / 2) * gr.r, z);
        }
    }
    io::Sidecar echo;
    echo.set("provenance", "phantom " + kind);
    echo.set("config.kind", kind);
    echo.set("config.n", std::int64_t(n));
    echo.set("config.ring_spacing", gr.r);
    echo.set("config.slice_height", gr.h);
    if (a.has("--table"))
        echo.set("config.table", a.str("--table"));
    if (a.has("--raw"))
        echo.set("config.raw", a.str("--raw"));
    echo.set("config.threads", std::int64_t(g.threads));
    echo.set("config.seed", g.seed);
    echo.set("clipped_negative", clipped ? "true" : "false");
    const std::string out = a.req("--out");
    io::write_field(out, f, echo);
    const auto w = value_range(f.values);
    if (!a.flag("--no-cg")) {
        const std::filesystem::path cg =
            a.has("--cg") ? std::filesystem::path(a.str("--cg"))
                          : std::filesystem::path(out).replace_extension(".cg.pgm");
        write_slices(cg, to_cartesian(gr, f.values), w.first, w.second, echo);
    }
    if (a.has("--pixel-raster"))
        write_slices(a.str("--pixel-raster"), pixel, w.first, w.second, echo);
    return 0;
}

// ---- project --------------------------------------------------------------

int run_project(const Args& a, const Globals& g) {
    const io::FieldFile f = io::read_field(a.req("--field"));
    const Grid gr = grid_of(f);
    io::ProjFile p;
    const std::vector<double> src = parse_point(a.str("--source", "-8,0,0"), "--source");
    const std::vector<double> ctr = parse_point(a.str("--center", "8,0,0"), "--center");
    for (int i = 0; i < 3; ++i) {
        p.source[i] = src[i];
        p.center[i] = ctr[i];
    }
    p.views = a.integer("--views", 50);
    p.det_u = a.integer("--det-u", 101);
    p.det_v = a.integer("--det-v", 1);
    p.spacing_u = a.num("--spacing-u", 0.05);
    p.spacing_v = a.num("--spacing-v", 0) > 0 ? a.num("--spacing-v", 0) : p.spacing_u;
    const std::string model = a.str("--model", "binary");
    if (model != "binary" && model != "length")
        throw std::invalid_argument("unknown forward model '" + model + "'");
    Tracer tr(gr, p, quarter_symmetric(p));
    const uscg_tracer_info inf = tr.info();
    std::vector<float> fv(f.values.begin(), f.values.end());
    std::vector<float> out(std::size_t(p.views) * p.det_u * p.det_v);
    check(uscg_project(tr.h, fv.data(), 1, out.data(), model == "length" ? USCG_MODEL_LENGTH : 0));
    p.data.assign(out.begin(), out.end());
    io::Sidecar echo;
    echo.set("provenance", "project " + model + " from " + a.req("--field"));
    echo.set("grid_mode", f.mode);
    echo.set("grid_n", std::int64_t(f.n));
    echo.set("grid_ring_spacing", f.ring_spacing);
    echo.set("grid_slice_height", f.slice_height);
    echo.set("config.model", model);
    echo.set("config.views", std::int64_t(p.views));
    echo.set("config.threads", std::int64_t(g.threads));
    echo.set("config.seed", g.seed);
    if (model == "binary")
        echo.set("cache_bytes", std::int64_t(inf.cache_bytes));
    io::write_projections(a.req("--out"), p, echo);
    return 0;
}

// ---- reconstruct ----------------------------------------------------------

int run_reconstruct(const Args& a, const Globals& g) {
    const std::string proj_path = a.req("--proj");
    const io::ProjFile p = io::read_projections(proj_path);
    const std::string mode = a.str("--mode", "auto");
    bool volume;
    if (mode == "2d")
        volume = false;
    else if (mode == "3d")
        volume = true;
    else if (mode == "auto")
        volume = p.det_v > 1;
    else
        throw std::invalid_argument("unknown mode '" + mode + "'");
    int n = a.integer("--n", 0);
    if (n == 0 && p.side.find("grid_n"))
        n = int(p.side.get_int("grid_n"));
    if (n == 0)
        throw std::invalid_argument("--n is required when the projection sidecar has no grid_n");
    const Grid gr = make_grid(n, a.num("--r", 0), a.num("--h", 0), volume);
    const std::string q = a.str("--quarter", "auto");
    bool quarter;
    if (q == "on")
        quarter = true;
    else if (q == "off")
        quarter = false;
    else if (q == "auto")
        quarter = quarter_symmetric(p);
    else
        throw std::invalid_argument("--quarter must be on, off or auto");
    const double beta = a.num("--beta", 0.4), tol = a.num("--tol", 1e-6), f_init = a.num("--f-init", 1.0);
    const int sweeps = a.integer("--sweeps", 100);
    Tracer tr(gr, p, quarter);
    const uscg_tracer_info inf = tr.info();
    const uscg_solver_config cfg{beta, tol, sweeps, f_init, 0.0};
    std::vector<float> proj(p.data.begin(), p.data.end());
    std::vector<float> field(gr.cells());
    std::vector<double> resid(std::size_t(std::max(sweeps, 1)));
    std::vector<uint8_t> crossed(gr.cells());
    uscg_report rep{};
    rep.sweep_residuals = resid.data();
    rep.crossed = crossed.data();
    check(uscg_reconstruct(tr.h, proj.data(), 1, &cfg, field.data(), 0, &rep, 0));
    for (float v : field)
        if (!std::isfinite(v))
            throw NumericalError("reconstructed field contains non-finite values");
    io::Sidecar echo;
    echo.set("provenance", "reconstruct from " + proj_path);
    echo.set("config.beta", beta);
    echo.set("config.tolerance", tol);
    echo.set("config.max_sweeps", std::int64_t(sweeps));
    echo.set("config.f_init", f_init);
    echo.set("config.quarter_symmetry", quarter ? "on" : "off");
    echo.set("config.threads", std::int64_t(g.threads));
    echo.set("config.seed", g.seed);
    echo.set("cache_bytes", std::int64_t(inf.cache_bytes));
    echo.set("cache_records", std::int64_t(inf.records));
    echo.set("sweeps", std::int64_t(rep.sweeps));
    echo.set("converged", rep.converged ? "true" : "false");
    echo.set("seconds", rep.seconds);
    io::FieldFile f;
    f.mode = volume ? "3d" : "2d";
    f.n = gr.n;
    f.slices = gr.slices();
    f.ring_spacing = gr.r;
    f.slice_height = gr.h;
    f.values.assign(field.begin(), field.end());
    const std::string out = a.req("--out");
    io::write_field(out, f, echo);
    io::Sidecar report = echo;
    report.set("all_zero_data", rep.all_zero_data ? "true" : "false");
    report.set("zero_measurement_skips", std::int64_t(rep.zero_measurement_skips));
    report.set("factor_clamps", std::int64_t(rep.factor_clamps));
    std::int64_t nc = 0;
    for (uint8_t c : crossed)
        nc += c;
    report.set("crossed_cells", nc);
    for (int i = 0; i < rep.sweeps; ++i)
        report.set("sweep." + std::to_string(i + 1) + ".residual", resid[i]);
    const std::filesystem::path rpath = a.has("--report")
                                            ? std::filesystem::path(a.str("--report"))
                                            : std::filesystem::path(out).replace_extension(".report.txt");
    io::write_report(rpath, report);
    if (rep.all_zero_data)
        std::cerr << "warning: all measurements are zero; returning the initial field\n";
    return 0;
}

// ---- map ------------------------------------------------------------------

int run_map(const Args& a, const Globals& g) {
    const std::string fp = a.req("--field");
    const io::FieldFile f = io::read_field(fp);
    if (a.has("--window-max") && !a.has("--window-min"))
        throw UsageError("--window-max requires --window-min");
    std::pair<double, double> w;
    if (a.has("--window-min")) {
        w = {a.num("--window-min", 0), a.num("--window-max", 0)};
        if (!(w.second > w.first))
            throw std::invalid_argument("--window-max must exceed --window-min");
    } else {
        w = value_range(f.values);
    }
    io::Sidecar echo;
    echo.set("provenance", "map from " + fp);
    echo.set("config.threads", std::int64_t(g.threads));
    echo.set("config.seed", g.seed);
    write_slices(a.req("--out"), to_cartesian(grid_of(f), f.values), w.first, w.second, echo);
    return 0;
}

// ---- metrics --------------------------------------------------------------

// area_average, sharpness (metrics.cpp:62-69,138-153) on the host
double area_average(const io::Raster& im) {
    double acc = 0;
    for (double x : im.v)
        acc += x;
    return acc / double(im.v.size());
}

double sharpness(const io::Raster& im) {
    if (im.rows < 2 || im.cols < 2)
        throw std::invalid_argument("sharpness needs at least a 2x2 image");
    auto at = [&](int r, int c) { return im.v[std::size_t(r) * im.cols + c]; };
    double acc = 0;
    for (int r = 0; r < im.rows; ++r)
        for (int c = 0; c < im.cols; ++c) {
            const int cl = std::max(c - 1, 0), ch = std::min(c + 1, im.cols - 1);
            const int rl = std::max(r - 1, 0), rh = std::min(r + 1, im.rows - 1);
            const double gx = (at(r, ch) - at(r, cl)) / (ch - cl);
            const double gy = (at(rh, c) - at(rl, c)) / (rh - rl);
            acc += std::sqrt(gx * gx + gy * gy);
        }
    return acc / (double(im.rows) * im.cols);
}

int run_metrics(const Args& a, const Globals&) {
    const std::string rp = a.req("--ref"), tp = a.req("--test");
    const io::Raster ref = io::read_pgm16(rp), test = io::read_pgm16(tp);
    if (ref.rows != test.rows || ref.cols != test.cols)
        throw std::invalid_argument("image shapes differ");
    std::vector<float> ra(ref.v.begin(), ref.v.end()), ta(test.v.begin(), test.v.end());
    double mae = 0, rmse = 0, ssim = 0;
    check(uscg_image_metrics(context(), ra.data(), ta.data(), 1, ref.rows, ref.cols, 0, -1.0, &mae, &rmse, &ssim, 0));
    io::Sidecar report;
    report.set("ref", rp);
    report.set("test", tp);
    report.set("mae", mae);
    report.set("rmse", rmse);
    report.set("ssim", ssim);
    report.set("area_average.ref", area_average(ref));
    report.set("area_average.test", area_average(test));
    report.set("sharpness.ref", sharpness(ref));
    report.set("sharpness.test", sharpness(test));
    const int row = a.integer("--profile-row", -1);
    if (row >= 0) {
        if (row >= ref.rows)
            throw std::invalid_argument("profile row out of range");
        auto join = [&](const io::Raster& im) {
            std::string s;
            for (int c = 0; c < im.cols; ++c)
                s += (c ? " " : "") + std::to_string(im.v[std::size_t(row) * im.cols + c]);
            return s;
        };
        report.set("profile.row", std::int64_t(row));
        report.set("profile.ref", join(ref));
        report.set("profile.test", join(test));
    }
    std::cout << report.text();
    if (a.has("--out"))
        io::write_report(a.str("--out"), report);
    return 0;
}

int usage() {
    std::cerr << "usage: uscg_b200 <phantom|project|reconstruct|map|metrics> [options]\n";
    return 1;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2)
        return usage();
    const std::string cmd = argv[1];
    Globals g;
    try {
        if (cmd == "phantom")
            return run_phantom(parse(argc, argv, 2,
                                     {"--kind", "--n", "--r", "--h", "--table", "--raw", "--raw-mode", "--out",
                                      "--cg", "--pixel-raster"},
                                     {"--no-cg"}, g),
                               g);
        if (cmd == "project")
            return run_project(parse(argc, argv, 2,
                                     {"--field", "--views", "--det-u", "--det-v", "--spacing-u", "--spacing-v",
                                      "--source", "--center", "--model", "--out"},
                                     {}, g),
                               g);
        if (cmd == "reconstruct")
            return run_reconstruct(parse(argc, argv, 2,
                                         {"--proj", "--n", "--r", "--h", "--mode", "--beta", "--tol", "--sweeps",
                                          "--f-init", "--quarter", "--out", "--report"},
                                         {}, g),
                                   g);
        if (cmd == "map")
            return run_map(parse(argc, argv, 2, {"--field", "--out", "--window-min", "--window-max"}, {}, g), g);
        if (cmd == "metrics")
            return run_metrics(parse(argc, argv, 2, {"--ref", "--test", "--out", "--profile-row"}, {}, g), g);
        return usage();
    } catch (const NumericalError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const DeviceError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const io::IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::domain_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
