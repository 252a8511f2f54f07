// Test harness: include/uscg_b200_io.hpp behind a C ABI, so tests/test_io.py
// can write and read files with it and compare them byte for byte with the
// reference's own writers (oracle/_ref). Built by the test with g++.
#include <cstring>
#include <exception>
#include <string>

#include "uscg_b200_io.hpp"

namespace io = uscg_b200::io;

namespace {
io::Sidecar sidecar_of(const char* const* keys, const char* const* vals, int nkv) {
    io::Sidecar s;
    for (int i = 0; i < nkv; ++i)
        s.set(keys[i], std::string(vals[i]));
    return s;
}

template <class F>
int guarded(char* err, int errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const io::IoError& e) {
        std::snprintf(err, std::size_t(errlen), "IoError: %s", e.what());
        return 1;
    } catch (const std::invalid_argument& e) {
        std::snprintf(err, std::size_t(errlen), "invalid_argument: %s", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::snprintf(err, std::size_t(errlen), "error: %s", e.what());
        return 3;
    }
}
}  // namespace

extern "C" {

int io_write_field(const char* path, int n, double r, double h, int volume, const double* values,
                   const char* const* keys, const char* const* vals, int nkv, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        io::FieldFile f;
        f.mode = volume ? "3d" : "2d";
        f.n = n;
        f.slices = volume ? n : 1;
        f.ring_spacing = r;
        f.slice_height = h;
        f.values.assign(values, values + std::size_t(f.slices) * n * n);
        io::write_field(path, f, sidecar_of(keys, vals, nkv));
    });
}

int io_read_field(const char* path, int* n, int* slices, double* values, long long cap, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const io::FieldFile f = io::read_field(path);
        *n = f.n;
        *slices = f.slices;
        if ((long long)f.values.size() <= cap)
            std::memcpy(values, f.values.data(), f.values.size() * sizeof(double));
    });
}

int io_write_projections(const char* path, int views, int det_u, int det_v, double su, double sv,
                         const double* src, const double* ctr, const double* data, const char* const* keys,
                         const char* const* vals, int nkv, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        io::ProjFile p;
        p.views = views;
        p.det_u = det_u;
        p.det_v = det_v;
        p.spacing_u = su;
        p.spacing_v = sv;
        for (int i = 0; i < 3; ++i) {
            p.source[i] = src[i];
            p.center[i] = ctr[i];
        }
        p.data.assign(data, data + std::size_t(views) * det_u * det_v);
        io::write_projections(path, p, sidecar_of(keys, vals, nkv));
    });
}

int io_read_projections(const char* path, int* dims, double* geom, double* data, long long cap, char* err,
                        int errlen) {
    return guarded(err, errlen, [&] {
        const io::ProjFile p = io::read_projections(path);
        dims[0] = p.views;
        dims[1] = p.det_u;
        dims[2] = p.det_v;
        const double g[8] = {p.spacing_u, p.spacing_v, p.source[0], p.source[1], p.source[2], p.center[0],
                             p.center[1], p.center[2]};
        std::memcpy(geom, g, sizeof g);
        if ((long long)p.data.size() <= cap)
            std::memcpy(data, p.data.data(), p.data.size() * sizeof(double));
    });
}

int io_write_pgm16(const char* path, int rows, int cols, const double* v, double wmin, double wmax,
                   const char* const* keys, const char* const* vals, int nkv, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        io::Raster im;
        im.rows = rows;
        im.cols = cols;
        im.v.assign(v, v + std::size_t(rows) * cols);
        io::write_pgm16(path, im, wmin, wmax, sidecar_of(keys, vals, nkv));
    });
}

int io_read_pgm16(const char* path, int* rows, int* cols, double* out, long long cap, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const io::Raster im = io::read_pgm16(path);
        *rows = im.rows;
        *cols = im.cols;
        if ((long long)im.v.size() <= cap)
            std::memcpy(out, im.v.data(), im.v.size() * sizeof(double));
    });
}

// the sidecar text of one double entry ("k = <17 significant digits>\n")
int io_sidecar_double(double v, char* out, int cap) {
    io::Sidecar s;
    s.set("k", v);
    const std::string t = s.text();
    std::snprintf(out, std::size_t(cap), "%s", t.c_str());
    return 0;
}
}
