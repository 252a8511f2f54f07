// uscg_b200 kernels for sm_100a. Built with --fmad=false: every fp64
// statement that mirrors the reference must round exactly like g++ on x86-64.
//
//   K1 generate_*   first-view coefficient generator (tracer.cpp:38-102,
//                   geometry.cpp:127-227)
//   K2 project      binary forward projector (phantom.cpp:182-211)
//   K3 mart_level   one dependency level of the Sp-MART row action
//                   (solver.cpp:33-51,111-136)
//   K4 *_resample   USPG -> Cartesian (grid.cpp:75-99, phantom.cpp:149-163)
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "ddmath.cuh"
#include "kernels.h"

namespace ub {

namespace {
constexpr double kDegPerRad = 180.0 / 3.141592653589793238462643383279502884;

inline int cdiv(long long a, long long b) { return int((a + b - 1) / b); }

void check_launch() {
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw CudaError(std::string("kernel launch: ") + cudaGetErrorString(e));
}
}  // namespace

int chunk_limit() {
    // 32: the wave executor's best on the c2 stack (a cell's 32 problems are
    // one 128-byte segment); the flow executor's best is 8
    const char* e = std::getenv("USCG_CHUNK_WIDTH");
    const int v = e ? std::atoi(e) : 32;
    int p = 1;
    while (p * 2 <= v && p < 32)
        p <<= 1;
    return p;
}

// Problems per MART task: the widest chunk (<= the limit) that pads the
// problem stride by at most 1/8, else the smallest power of two covering the
// problems up to 8. Wide chunks move more bytes per scattered access; up to
// 64 problems the clustered wave's chains run faster on 16-problem chunks
// than on fewer 32-problem ones while the pairs of all chunks still find SMs
// (C2 geometry, ms per iteration: 32 problems 2.25 vs 3.10, 64: 2.84 vs 3.07;
// 96: 4.58 vs 3.26), so 16 is the default limit there.
int chunk_width(int problems) {
    const int limit = std::getenv("USCG_CHUNK_WIDTH") || problems > 64 ? chunk_limit() : std::min(16, chunk_limit());
    int p = 1;
    while (p < problems && p < std::min(8, limit))
        p <<= 1;
    for (int q = limit; q > p; q >>= 1) {
        const long long padded = (static_cast<long long>(problems) + q - 1) / q * q;
        if (padded * 8 <= static_cast<long long>(problems) * 9)
            return q;
    }
    return p;
}

int problem_stride(int problems) {
    const int p = chunk_width(problems);
    return ((problems + p - 1) / p) * p;
}

// chunk width used for an interleaved stride Sp (largest power of two <=
// the chunk limit that divides Sp)
int stride_chunk(int Sp) {
    int p = 1;
    while (p < chunk_limit() && Sp % (p * 2) == 0)
        p <<= 1;
    return p;
}

// =============================================================================
// K1: first-view coefficient generator, one thread per ray.
// =============================================================================

// azimuth_deg (geometry.cpp:39-46)
__device__ __forceinline__ double azimuth_deg(double x, double y) {
    double deg = atan2_gen(y, x) * kDegPerRad;
    if (deg < 0)
        deg += 360.0;
    if (deg >= 360.0)
        deg = 0.0;
    return deg;
}

// floor(a / b) as the reference evaluates it (the correctly rounded quotient,
// floored) from a * inv_b, inv_b = RN(1/b): the product is within 2.5 ulp
// of the rounded quotient, so when q (1 ± 2^-50) spans no integer both
// floor alike; otherwise the division.
__device__ __forceinline__ double floor_quot(double a, double b, double inv_b) {
    const double q = a * inv_b;
    const double d = fabs(q) * 0x1p-50;
    const double f = floor(q - d);
    return f == floor(q + d) ? f : floor(a / b);
}

// floor(hypot(x, y) / b), hypot correctly rounded (geometry.cpp:216-217):
// sqrt(x^2 + y^2) is within 1.75 ulp of hypot_cr and the product with inv_b
// within 4.5 ulp of the reference's quotient (< 2^-50 relative), so the same
// interval test decides it; otherwise hypot_cr and the division.
__device__ __forceinline__ double floor_hypot_quot(double x, double y, double b, double inv_b) {
    const double q = sqrt(x * x + y * y) * inv_b;
    const double d = q * 0x1p-50;
    const double f = floor(q - d);
    return f == floor(q + d) ? f : floor(hypot_cr(x, y) / b);
}

// The sorted crossing list of build_sorted_intersections (geometry.cpp:127-198)
// is the merge of three monotone sequences: entry-side ring roots t - k_k
// (non-increasing in ring k), exit-side roots t + k_k (non-decreasing in k) and
// z-plane roots (monotone in m). Every rounding step is monotone, so merging
// the filtered sequences yields exactly std::sort's output; no sort is needed.
struct RaySources {
    const DevGrid* g;
    double s0, s1, s2, dir0, dir1, dir2;
    double t, d2, uxy2, zlim, lim2;
    bool volume, axial, planes;
    int kA, kB, kmin, m, mstep, mend;

    __device__ double ring_k(int ring) const {
        const double radius = ring * g->ring_spacing;
        const double r2 = radius * radius;
        return sqrt((r2 - d2) / uxy2);
    }
    __device__ bool z_ok(double tau) const {
        if (!volume)
            return true;
        const double z = s2 + tau * dir2;
        return !(fabs(z) > zlim);
    }
    __device__ double nextA() {  // entry roots, ring descending
        while (kA >= kmin) {
            const double tau = t - ring_k(kA);
            --kA;
            if (tau < 0.0 || tau > 1.0)
                continue;
            if (!z_ok(tau))
                continue;
            return tau;
        }
        return DBL_MAX;
    }
    __device__ double nextB() {  // exit roots, ring ascending
        while (kB <= g->n_rings) {
            const double tau = t + ring_k(kB);
            ++kB;
            if (tau < 0.0 || tau > 1.0)
                continue;
            if (!z_ok(tau))
                continue;
            return tau;
        }
        return DBL_MAX;
    }
    __device__ double nextC() {  // slice planes
        while (planes && m != mend) {
            const int mm = m;
            m += mstep;
            const double tau = (mm * g->slice_height - g->zoff - s2) / dir2;
            if (tau < 0.0 || tau > 1.0)
                continue;
            if (!axial) {
                const double x = s0 + tau * dir0;
                const double y = s1 + tau * dir1;
                if (!(x * x + y * y <= lim2))
                    continue;
            }
            return tau;
        }
        return DBL_MAX;
    }
};

// Walk one ray through the grid: the sorted, eps-merged crossings of
// build_sorted_intersections and classify_chord (geometry.cpp:127-227); every
// kept chord (p, q, slice, ring) goes to on_chord, every rejected one to
// on_reject. Returns the number of kept chords.
template <class OnChord, class OnReject>
__device__ uint32_t walk_ray(const DevGrid& g, const double* s, const double* d, OnChord&& on_chord,
                             OnReject&& on_reject) {
    RaySources R;
    R.g = &g;
    R.s0 = s[0];
    R.s1 = s[1];
    R.s2 = s[2];
    R.dir0 = d[0] - s[0];
    R.dir1 = d[1] - s[1];
    R.dir2 = d[2] - s[2];
    R.volume = g.volume != 0;
    // is_axial (geometry.cpp:31-37)
    const double ux = s[0] - d[0], uy = s[1] - d[1];
    R.uxy2 = ux * ux + uy * uy;
    const double dd2 = R.dir0 * R.dir0 + R.dir1 * R.dir1 + R.dir2 * R.dir2;
    R.axial = dd2 == 0.0 || R.uxy2 <= 1e-24 * dd2;
    R.kA = 0;
    R.kmin = 1;
    R.kB = g.n_rings + 1;
    R.planes = false;
    R.m = 0;
    R.mend = 0;
    R.mstep = 1;
    R.zlim = g.zoff + g.eps;
    R.lim2 = (g.radius + g.eps) * (g.radius + g.eps);
    R.t = 0;
    R.d2 = 0;
    if (R.axial) {
        if (!R.volume)
            return 0;
        if (hypot_cr(s[0], s[1]) >= g.radius)
            return 0;
        if (R.dir2 == 0.0)
            return 0;
        R.planes = true;
    } else {
        // circle_taus (geometry.cpp:72-85), per-ray invariants
        R.t = (s[0] * ux + s[1] * uy) / R.uxy2;
        const double cross = s[0] * d[1] - s[1] * d[0];
        R.d2 = cross * cross / R.uxy2;
        int kmin = 1;
        while (kmin <= g.n_rings) {
            const double radius = kmin * g.ring_spacing;
            if (!(R.d2 > radius * radius))
                break;
            ++kmin;
        }
        R.kmin = kmin;
        R.kA = g.n_rings;
        R.kB = kmin;
        R.planes = R.volume && R.dir2 != 0.0;
    }
    if (R.planes) {
        if (R.dir2 > 0) {
            R.m = 0;
            R.mend = g.n_slices + 1;
            R.mstep = 1;
        } else {
            R.m = g.n_slices;
            R.mend = -1;
            R.mstep = -1;
        }
    }

    const double len = sqrt(dd2);  // norm(dir)
    const double inv_rs = 1.0 / g.ring_spacing, inv_h = 1.0 / g.slice_height;
    // sqrt(e) <= eps decided on e where it is certain (e within a factor
    // 1 ± 2^-48 of eps^2 takes the square root)
    const double eps2 = g.eps * g.eps;
    const double eps2_lo = eps2 * (1.0 - 0x1p-48), eps2_hi = eps2 * (1.0 + 0x1p-48);
    double ta = R.axial ? DBL_MAX : R.nextA();
    double tb = R.axial ? DBL_MAX : R.nextB();
    double tc = R.nextC();
    int np = 0;
    double last_tau = 0;
    double p0 = 0, p1 = 0, p2 = 0;
    uint32_t nrec = 0;
    while (true) {
        double tau;
        if (ta <= tb && ta <= tc) {
            tau = ta;
            if (tau == DBL_MAX)
                break;
            ta = R.nextA();
        } else if (tb <= tc) {
            tau = tb;
            tb = R.nextB();
        } else {
            tau = tc;
            tc = R.nextC();
        }
        // eps-merge of near-coincident crossings (geometry.cpp:188-196)
        if (np > 0 && (tau - last_tau) * len <= g.eps)
            continue;
        const double q0 = R.s0 + tau * R.dir0;
        const double q1 = R.s1 + tau * R.dir1;
        const double q2 = R.s2 + tau * R.dir2;
        if (np > 0) {
            // classify_chord (geometry.cpp:200-227)
            const double e0 = p0 - q0, e1 = p1 - q1, e2 = p2 - q2;
            const double e = e0 * e0 + e1 * e1 + e2 * e2;
            bool keep = e > eps2_hi || (e >= eps2_lo && !(sqrt(e) <= g.eps));
            int slice = 0, ring = 0;
            if (keep) {
                const double m0 = (p0 + q0) / 2, m1 = (p1 + q1) / 2, m2 = (p2 + q2) / 2;
                if (g.volume) {
                    const double zloc = m2 + g.zoff;
                    const double sf = floor_quot(zloc, g.slice_height, inv_h);
                    if (sf < 0 || sf >= g.n_slices)
                        keep = false;
                    else
                        slice = int(sf);
                }
                if (keep) {
                    ring = int(floor_hypot_quot(m0, m1, g.ring_spacing, inv_rs)) + 1;
                    if (ring > g.n_rings)
                        keep = false;
                }
            }
            if (keep) {
                on_chord(p0, p1, p2, q0, q1, q2, slice, ring);
                ++nrec;
            } else {
                on_reject();
            }
        }
        p0 = q0;
        p1 = q1;
        p2 = q2;
        last_tau = tau;
        ++np;
    }
    return nrec;
}

// records of one first-view ray (precompute_first_view, tracer.cpp:38-102):
// consecutive kept chords share their azimuth at the common point
template <bool WRITE>
__device__ uint32_t generate_ray(const DevGrid& g, const double* s, const double* d, double* pa,
                                 double* pb, uint32_t* key, uint32_t cap = 0xFFFFFFFFu) {
    double phi_prev = -1.0;
    uint32_t k = 0;
    return walk_ray(
        g, s, d,
        [&](double p0, double p1, double, double q0, double q1, double, int slice, int ring) {
            if (WRITE) {
                if (phi_prev < 0)
                    phi_prev = azimuth_deg(p0, p1);
                const double phi_q = azimuth_deg(q0, q1);
                if (k < cap) {
                    pa[k] = phi_prev;
                    pb[k] = phi_q;
                    key[k] = uint32_t(ring) | (uint32_t(slice) << kSliceShift);
                }
                phi_prev = phi_q;
                ++k;
            }
        },
        [&]() {
            if (WRITE)
                phi_prev = -1.0;
        });
}

__global__ void generate_count_kernel(DevGrid g, int lines, const double* __restrict__ src,
                                      const double* __restrict__ det, uint32_t* counts) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lines)
        return;
    counts[l] = generate_ray<false>(g, src + 3 * size_t(l), det + 3 * size_t(l), nullptr, nullptr,
                                    nullptr);
}

__global__ void generate_write_kernel(DevGrid g, int lines, const double* __restrict__ src,
                                      const double* __restrict__ det,
                                      const uint32_t* __restrict__ off, double* pa, double* pb,
                                      uint32_t* key) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lines)
        return;
    const uint32_t o = off[l];
    generate_ray<true>(g, src + 3 * size_t(l), det + 3 * size_t(l), pa + o, pb + o, key + o);
}

// One-pass generator. A ray's records are at most its crossings (a kept chord
// joins two consecutive crossings): the ring circles it reaches, twice each,
// and the z-planes its segment spans. bound_kernel over-estimates that count
// without walking the ray; the write pass fills each ray's bounded slot,
// records its true count and flags any ray whose slot was too small (the
// caller then falls back to the exact count pass); compaction packs the slots.
__global__ void generate_bound_kernel(DevGrid g, int lines, const double* __restrict__ src,
                                      const double* __restrict__ det, uint32_t* __restrict__ bound) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lines)
        return;
    const double* s = src + 3 * size_t(l);
    const double* d = det + 3 * size_t(l);
    const double dir0 = d[0] - s[0], dir1 = d[1] - s[1], dir2 = d[2] - s[2];
    const double ux = s[0] - d[0], uy = s[1] - d[1];
    const double uxy2 = ux * ux + uy * uy;
    const double dd2 = dir0 * dir0 + dir1 * dir1 + dir2 * dir2;
    const bool axial = dd2 == 0.0 || uxy2 <= 1e-24 * dd2;
    uint32_t b = 2;
    if (!axial) {
        const double cross = s[0] * d[1] - s[1] * d[0];
        const double dist = sqrt(cross * cross / uxy2);
        const int k0 = max(1, int(floor(dist / g.ring_spacing)) - 1);
        if (k0 <= g.n_rings)
            b += 2u * uint32_t(g.n_rings - k0 + 1);
    }
    if (g.volume && dir2 != 0.0) {
        const double za = fmin(s[2], d[2]) + g.zoff, zb = fmax(s[2], d[2]) + g.zoff;
        const int lo = max(0, int(ceil(za / g.slice_height)) - 1);
        const int hi = min(g.n_slices, int(floor(zb / g.slice_height)) + 1);
        if (hi >= lo)
            b += uint32_t(hi - lo + 1);
    }
    bound[l] = b;
}

__global__ void generate_slot_kernel(DevGrid g, int lines, const double* __restrict__ src,
                                     const double* __restrict__ det, const uint32_t* __restrict__ boff,
                                     double* pa, double* pb, uint32_t* key, uint32_t* __restrict__ counts,
                                     unsigned* overflow) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lines)
        return;
    const uint32_t o = boff[l], cap = boff[l + 1] - o;
    const uint32_t n = generate_ray<true>(g, src + 3 * size_t(l), det + 3 * size_t(l), pa + o, pb + o, key + o,
                                          cap);
    counts[l] = n;
    if (n > cap)
        atomicOr(overflow, 1u);
}

// warp per ray: its records from the bounded slot to the packed store
__global__ void compact_records_kernel(int lines, const uint32_t* __restrict__ boff,
                                       const uint32_t* __restrict__ off, const double* __restrict__ spa,
                                       const double* __restrict__ spb, const uint32_t* __restrict__ skey,
                                       double* __restrict__ pa, double* __restrict__ pb, uint32_t* __restrict__ key) {
    const int l = int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (l >= lines)
        return;
    const uint32_t from = boff[l], to = off[l], n = off[l + 1] - to;
    for (uint32_t i = lane; i < n; i += 32) {
        pa[to + i] = spa[from + i];
        pb[to + i] = spb[from + i];
        key[to + i] = skey[from + i];
    }
}

void launch_generate_bound(const DevGrid& g, int lines, const double* src, const double* det, uint32_t* bound,
                           cudaStream_t st) {
    generate_bound_kernel<<<cdiv(lines, 128), 128, 0, st>>>(g, lines, src, det, bound);
    check_launch();
}

void launch_generate_slots(const DevGrid& g, int lines, const double* src, const double* det, const uint32_t* boff,
                           double* pa, double* pb, uint32_t* key, uint32_t* counts, unsigned* overflow,
                           cudaStream_t st) {
    generate_slot_kernel<<<cdiv(lines, 64), 64, 0, st>>>(g, lines, src, det, boff, pa, pb, key, counts, overflow);
    check_launch();
}

void launch_compact_records(int lines, const uint32_t* boff, const uint32_t* off, const double* spa,
                            const double* spb, const uint32_t* skey, double* pa, double* pb, uint32_t* key,
                            cudaStream_t st) {
    compact_records_kernel<<<cdiv(lines, 8), 256, 0, st>>>(lines, boff, off, spa, spb, skey, pa, pb, key);
    check_launch();
}

// =============================================================================
// K2' length-weighted projector (generate_projections LengthWeighted,
// phantom.cpp:213-269): per (view, line) the first-view ray rotated by theta
// (rotate_z_deg, scan.cpp:50-54) is walked through the grid; every chord is
// cut where it crosses a radial sector boundary of its ring and each piece
// contributes length x field of the sector of its midpoint. The reference
// tests every boundary of the ring (O(sectors) per chord); azimuth is monotone
// along a chord that misses the origin, so only the boundaries between the
// sectors of its end points (one extra on each side) can cut it, and they are
// met in order. Rings of at most 16 sectors (where a chord may pass through
// the origin) test every boundary, as the reference does. fp64 throughout.
// =============================================================================
constexpr double kRadPerDeg = 3.141592653589793238462643383279502884 / 180.0;

template <int P>
struct LengthAcc {
    const float* field;  // [cells][Sp], this thread's chunk at column col
    uint32_t Sp, col;
    double acc[P];

    __device__ void piece(double len, uint32_t cell) {
        const float* f = field + size_t(cell) * Sp + col;
#pragma unroll
        for (int p = 0; p < P; ++p)
            acc[p] += len * double(__ldg(f + p));
    }
};

// counts a line's pieces / writes them as (cell, length) pairs: the
// (voxel, chord length) lists of the same walk (launch_length_lists)
struct LengthCount {
    uint32_t n = 0;
    __device__ void piece(double, uint32_t) { ++n; }
};
struct LengthWrite {
    uint32_t* idx;
    float* len;
    uint32_t k;
    __device__ void piece(double l, uint32_t cell) {
        idx[k] = cell;
        len[k] = float(l);
        ++k;
    }
};

template <class Sink>
__device__ void length_chord(const DevGrid& g, double a0, double a1, double a2, double b0, double b1,
                             double b2, int slice, int ring, Sink& A) {
    const double u0 = b0 - a0, u1 = b1 - a1, u2 = b2 - a2;
    const double chord_len = sqrt(u0 * u0 + u1 * u1 + u2 * u2);
    const RingRow rr = g.rings[ring];
    const int ng = int(rr.count);
    const double step_deg = 360.0 / ng;  // RingLayout::step_deg (grid.cpp:69)
    const uint32_t base = uint32_t(slice) * g.cells_per_slice + rr.head;
    auto tau_of = [&](int j, double& tau) {
        const double psi = j * step_deg * kRadPerDeg;
        const double ex = cos(psi), ey = sin(psi);
        const double g0 = ex * a1 - ey * a0;
        const double g1 = ex * u1 - ey * u0;
        if (g1 == 0.0)
            return false;
        tau = -g0 / g1;
        return tau > 0.0 && tau < 1.0;
    };
    double prev = 0.0;
    auto emit = [&](double t1) {
        const double piece = (t1 - prev) * chord_len;
        if (piece > 0) {
            const double mid = 0.5 * (prev + t1);
            const double phi = azimuth_deg(a0 + mid * u0, a1 + mid * u1);
            int sector = int(phi * rr.inv_step);
            if (sector >= ng)
                sector = ng - 1;
            A.piece(piece, base + uint32_t(sector));
        }
        prev = t1;
    };
    if (ng <= 16) {
        double cuts[18];
        int nc = 0;
        for (int j = 0; j < ng; ++j) {
            double tau;
            if (tau_of(j, tau)) {
                int k = nc++;
                while (k > 0 && cuts[k - 1] > tau) {
                    cuts[k] = cuts[k - 1];
                    --k;
                }
                cuts[k] = tau;
            }
        }
        for (int k = 0; k < nc; ++k)
            emit(cuts[k]);
        emit(1.0);
        return;
    }
    int ga = int(azimuth_deg(a0, a1) * rr.inv_step);
    if (ga >= ng)
        ga = ng - 1;
    int gb = int(azimuth_deg(b0, b1) * rr.inv_step);
    if (gb >= ng)
        gb = ng - 1;
    // > 0: azimuth increases along the chord. A radial chord (on a line through
    // the origin) keeps one azimuth: one piece, in its midpoint's sector (the
    // reference's cut there is -g0/g1 of two rounding residues, an arbitrary
    // split of the same length between two sectors)
    const double cross = a0 * u1 - a1 * u0;
    if (fabs(cross) <= 1e-12 * sqrt(a0 * a0 + a1 * a1) * sqrt(u0 * u0 + u1 * u1)) {
        emit(1.0);
        return;
    }
    if (cross > 0) {
        const int nb = ((gb - ga) % ng + ng) % ng + 2;  // boundaries ga .. gb+1
        for (int k = 0; k < nb; ++k) {
            double tau;
            if (tau_of((ga + k) % ng, tau) && tau > prev)
                emit(tau);
        }
    } else if (cross < 0) {
        const int nb = ((ga - gb) % ng + ng) % ng + 2;  // boundaries ga+1 down to gb
        for (int k = 0; k < nb; ++k) {
            double tau;
            if (tau_of(((ga + 1 - k) % ng + ng) % ng, tau) && tau > prev)
                emit(tau);
        }
    }
    emit(1.0);
}

template <int P>
__global__ void __launch_bounds__(128) project_length_kernel(DevGrid g, int lines, int views,
                                                             const double* __restrict__ rays,
                                                             const double* __restrict__ theta,
                                                             const float* __restrict__ field, int Sp,
                                                             float* __restrict__ out) {
    const long long unit = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (unit >= (long long)lines * views)
        return;
    const int v = int(unit / lines), l = int(unit % lines);
    const int chunk = int(blockIdx.y);
    // rotate_z_deg (scan.cpp:50-54)
    const double rad = theta[v] * kRadPerDeg;
    const double c = cos(rad), sn = sin(rad);
    const double* s0 = rays + 3 * size_t(l);
    const double* d0 = rays + 3 * (size_t(lines) + l);
    const double s[3] = {c * s0[0] - sn * s0[1], sn * s0[0] + c * s0[1], s0[2]};
    const double d[3] = {c * d0[0] - sn * d0[1], sn * d0[0] + c * d0[1], d0[2]};
    LengthAcc<P> A{field, uint32_t(Sp), uint32_t(chunk * P), {}};
#pragma unroll
    for (int p = 0; p < P; ++p)
        A.acc[p] = 0.0;
    walk_ray(
        g, s, d,
        [&](double p0, double p1, double p2, double q0, double q1, double q2, int slice, int ring) {
            length_chord(g, p0, p1, p2, q0, q1, q2, slice, ring, A);
        },
        [] {});
    float* o = out + size_t(unit) * Sp + size_t(chunk) * P;
#pragma unroll
    for (int p = 0; p < P; ++p)
        o[p] = float(A.acc[p]);
}

// The (voxel, chord length) lists of every (view, line): a thread per line
// walks it as the projector does; off == nullptr counts the pieces into
// counts[unit], else writes them at off[unit].
__global__ void __launch_bounds__(128) length_lists_kernel(DevGrid g, int lines, int views,
                                                           const double* __restrict__ rays,
                                                           const double* __restrict__ theta,
                                                           const uint32_t* __restrict__ off,
                                                           uint32_t* __restrict__ counts,
                                                           uint32_t* __restrict__ idx, float* __restrict__ len) {
    const long long unit = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (unit >= (long long)lines * views)
        return;
    const int v = int(unit / lines), l = int(unit % lines);
    const double rad = theta[v] * kRadPerDeg;  // rotate_z_deg (scan.cpp:50-54)
    const double c = cos(rad), sn = sin(rad);
    const double* s0 = rays + 3 * size_t(l);
    const double* d0 = rays + 3 * (size_t(lines) + l);
    const double s[3] = {c * s0[0] - sn * s0[1], sn * s0[0] + c * s0[1], s0[2]};
    const double d[3] = {c * d0[0] - sn * d0[1], sn * d0[0] + c * d0[1], d0[2]};
    if (off == nullptr) {
        LengthCount A;
        walk_ray(
            g, s, d,
            [&](double p0, double p1, double p2, double q0, double q1, double q2, int slice, int ring) {
                length_chord(g, p0, p1, p2, q0, q1, q2, slice, ring, A);
            },
            [] {});
        counts[unit] = A.n;
    } else {
        LengthWrite A{idx, len, off[unit]};
        walk_ray(
            g, s, d,
            [&](double p0, double p1, double p2, double q0, double q1, double q2, int slice, int ring) {
                length_chord(g, p0, p1, p2, q0, q1, q2, slice, ring, A);
            },
            [] {});
    }
}

void launch_length_lists(const DevGrid& g, int lines, int views, const double* rays, const double* theta,
                         const uint32_t* off, uint32_t* counts, uint32_t* idx, float* len, cudaStream_t st) {
    const long long units = (long long)lines * views;
    if (units <= 0)
        return;
    length_lists_kernel<<<unsigned((units + 127) / 128), 128, 0, st>>>(g, lines, views, rays, theta, off, counts, idx,
                                                                      len);
    check_launch();
}

void launch_project_length(const DevGrid& g, int lines, int views, const double* rays,
                           const double* theta, const float* field, int Sp, float* out,
                           cudaStream_t st) {
    const long long units = (long long)lines * views;
    if (units <= 0)
        return;
    const int P = stride_chunk(Sp) > 8 ? 8 : stride_chunk(Sp);
    const dim3 grid(unsigned((units + 127) / 128), unsigned(Sp / P));
    switch (P) {
        case 1: project_length_kernel<1><<<grid, 128, 0, st>>>(g, lines, views, rays, theta, field, Sp, out); break;
        case 2: project_length_kernel<2><<<grid, 128, 0, st>>>(g, lines, views, rays, theta, field, Sp, out); break;
        case 4: project_length_kernel<4><<<grid, 128, 0, st>>>(g, lines, views, rays, theta, field, Sp, out); break;
        default: project_length_kernel<8><<<grid, 128, 0, st>>>(g, lines, views, rays, theta, field, Sp, out); break;
    }
    check_launch();
}

void launch_generate_count(const DevGrid& g, int lines, const double* src, const double* det,
                           uint32_t* counts, cudaStream_t st) {
    if (lines <= 0)
        return;
    generate_count_kernel<<<cdiv(lines, 64), 64, 0, st>>>(g, lines, src, det, counts);
    check_launch();
}

void launch_generate_write(const DevGrid& g, int lines, const double* src, const double* det,
                           const uint32_t* off, double* pa, double* pb, uint32_t* key,
                           cudaStream_t st) {
    if (lines <= 0)
        return;
    generate_write_kernel<<<cdiv(lines, 64), 64, 0, st>>>(g, lines, src, det, off, pa, pb, key);
    check_launch();
}

// ---- dedup annotation --------------------------------------------------------
// Two chords of one line can share a cell only if they lie in the same
// (slice, ring) and their short arcs are within one sector of each other (the
// rotation shifts both by the same angle). Such records get the flag bit and
// the trace applies the stamp dedup to them; every other record expands
// without any check.
__device__ __forceinline__ void short_arc(double a, double b, double& st, double& ln) {
    const double lo = a < b ? a : b, hi = a < b ? b : a;
    if (hi - lo <= 180.0) {
        st = lo;
        ln = hi - lo;
    } else {
        st = hi;
        ln = 360.0 - (hi - lo);
    }
}

__device__ __forceinline__ double wrap360(double x) { return x - 360.0 * floor(x / 360.0); }

__device__ bool arcs_near(double a0, double b0, double a1, double b1, double step) {
    double s0, l0, s1, l1;
    short_arc(a0, b0, s0, l0);
    short_arc(a1, b1, s1, l1);
    if (l0 >= 179.0 || l1 >= 179.0)
        return true;
    const double d01 = wrap360(s1 - (s0 + l0));
    const double d10 = wrap360(s0 - (s1 + l1));
    if (fabs(d01 + d10 + l0 + l1 - 360.0) > 1e-6)
        return true;  // overlapping
    return fmin(d01, d10) <= 1.5 * step + 1e-9;
}

__global__ void annotate_kernel(int lines, const uint32_t* __restrict__ off,
                                const double* __restrict__ pa, const double* __restrict__ pb,
                                uint32_t* key, const RingRow* __restrict__ rings) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= lines)
        return;
    const uint32_t r0 = off[warp], r1 = off[warp + 1];
    for (uint32_t i = r0 + 1 + lane; i < r1; i += 32) {
        const uint32_t ki = key[i] & ~kFlagBit;
        const uint32_t ring = ki & kRingMask;
        const double step = 360.0 / rings[ring].count;
        for (uint32_t j = i; j-- > r0;) {
            const uint32_t kj = key[j] & ~kFlagBit;
            if ((kj >> kSliceShift) != (ki >> kSliceShift))
                break;  // records of one slice are contiguous along the ray
            if (kj != ki)
                continue;
            if (arcs_near(pa[i], pb[i], pa[j], pb[j], step)) {
                atomicOr(key + i, kFlagBit);
                break;
            }
        }
    }
}

__global__ void clear_flags_kernel(uint32_t* key, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        key[i] &= ~kFlagBit;
}

void launch_clear_flags(uint32_t* key, uint64_t n, cudaStream_t st) {
    if (n == 0)
        return;
    clear_flags_kernel<<<unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(key, n);
    check_launch();
}

void launch_annotate(int lines, const uint32_t* off, const double* pa, const double* pb,
                     uint32_t* key, const RingRow* rings, cudaStream_t st) {
    if (lines <= 0)
        return;
    annotate_kernel<<<cdiv(lines, 8), 256, 0, st>>>(lines, off, pa, pb, key, rings);
    check_launch();
}


// =============================================================================
// traces
// =============================================================================

template <int NT>
__global__ void __launch_bounds__(NT) trace_one_kernel(TraceArgs A, int line, double theta,
                                                       int max_recs, uint32_t* out,
                                                       uint32_t* count) {
    extern __shared__ uint32_t smem[];
    const TraceSmem S = carve_trace_smem<NT>(smem, max_recs);
    const int n = block_trace<NT>(A, line, theta, S, true);
    for (int i = threadIdx.x; i < n; i += NT)
        out[i] = S.idx[i];
    if (threadIdx.x == 0)
        *count = uint32_t(n);
}

void launch_trace_one(const TraceArgs& A, int line, double theta, int max_recs, int max_cells,
                      uint32_t* out, uint32_t* count, cudaStream_t st) {
    const size_t sm = trace_smem_bytes(256, max_recs, max_cells);
    UB_CUDA(cudaFuncSetAttribute(trace_one_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(sm)));
    trace_one_kernel<256><<<1, 256, sm, st>>>(A, line, theta, max_recs, out, count);
    check_launch();
}

template <int NT>
__global__ void __launch_bounds__(NT) trace_counts_kernel(TraceArgs A, int max_recs,
                                                          uint32_t* cells) {
    extern __shared__ uint32_t smem[];
    const TraceSmem S = carve_trace_smem<NT>(smem, max_recs);
    const int unit = blockIdx.x;
    const int v = unit / A.lines, line = unit % A.lines;
    const int n = block_trace<NT>(A, line, A.theta[v], S, false);
    if (threadIdx.x == 0)
        cells[unit] = uint32_t(n);
}

void launch_trace_counts(const TraceArgs& A, int views, int max_recs, uint32_t* cells,
                         cudaStream_t st) {
    const long long units = (long long)views * A.lines;
    if (units <= 0)
        return;
    const size_t sm = trace_smem_bytes(128, max_recs, 0);
    UB_CUDA(cudaFuncSetAttribute(trace_counts_kernel<128>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    trace_counts_kernel<128><<<unsigned(units), 128, sm, st>>>(A, max_recs, cells);
    check_launch();
}

// rotated reuse (C5): per (view, line) |active| and the sum of its cells. One
// warp per line serves every requested view: the line's records come from
// HBM once and from L1 for the other views (the one-view store serving all
// views, on chip). Each record is rotated in registers and its sector range
// summed arithmetically. Dedup-flagged records (tracer.cpp:181-195 only bites
// between chords of one (slice, ring) whose arcs nearly meet) drop the sectors
// an earlier chord of the same (slice, ring) covers; their partners are found
// once per line (they depend on the keys, not the view) and re-rotated per
// view. Lines beyond the caps scan for partners per view.
constexpr int kSumWarps = 4;
constexpr int kSumFlagged = 128;  // flagged records cached per line
constexpr int kSumPartners = 4;

struct RecRot {
    long long b;
    int lo, hi, ng;
    bool seam;
};

__device__ __forceinline__ RecRot rot_record(const TraceArgs& A, const RingRow* rings, uint32_t r,
                                             double theta) {
    const uint32_t key = __ldg(A.key + r);
    const RingRow rr = rings[key & kRingMask];
    RecRot o;
    rotate_chord(__ldg(A.pa + r), __ldg(A.pb + r), theta, rr.count, rr.inv_step, o.lo, o.hi, o.seam);
    o.b = ((key >> kSliceShift) & kSliceMask) * (long long)A.cells_per_slice + rr.head;
    o.ng = int(rr.count);
    return o;
}

// sectors of flagged record r0+i not covered by the listed earlier partners
// (np < 0: scan every earlier record of the same (slice, ring))
__device__ void flagged_count_sum(const TraceArgs& A, const RingRow* rings, uint32_t r0, int i,
                                  double theta, const uint16_t* partners, int np,
                                  unsigned long long& c, unsigned long long& s) {
    const RecRot me = rot_record(A, rings, r0 + i, theta);
    RecRot p[kSumPartners];
    if (np >= 0)
        for (int k = 0; k < np; ++k)
            p[k] = rot_record(A, rings, r0 + partners[k], theta);
    const uint32_t base_key = __ldg(A.key + r0 + i) & ((kSliceMask << kSliceShift) | kRingMask);
    auto covered = [&](int q) {
        if (np >= 0) {
            for (int k = 0; k < np; ++k)
                if (range_has(q, p[k].lo, p[k].hi, p[k].seam))
                    return true;
            return false;
        }
        for (int j = i - 1; j >= 0; --j) {
            if ((__ldg(A.key + r0 + j) & ((kSliceMask << kSliceShift) | kRingMask)) != base_key)
                continue;
            const RecRot o = rot_record(A, rings, r0 + j, theta);
            if (range_has(q, o.lo, o.hi, o.seam))
                return true;
        }
        return false;
    };
    auto take = [&](int q) {
        if (!covered(q)) {
            ++c;
            s += static_cast<unsigned long long>(me.b + q);
        }
    };
    if (!me.seam) {
        for (int q = me.lo; q <= me.hi; ++q)
            take(q);
    } else {
        for (int q = me.hi; q < me.ng; ++q)
            take(q);
        for (int q = 0; q <= me.lo; ++q)
            take(q);
    }
}

__global__ void __launch_bounds__(32 * kSumWarps) checksum_kernel(TraceArgs A, int view0, int nviews,
                                                                  int n_rings, uint32_t* counts,
                                                                  unsigned long long* sums) {
    extern __shared__ __align__(16) uint32_t smem[];
    RingRow* s_rings = reinterpret_cast<RingRow*>(smem);
    for (int k = threadIdx.x; k <= n_rings; k += blockDim.x)
        s_rings[k] = A.rings[k];
    __shared__ uint16_t s_fl[kSumWarps][kSumFlagged];
    __shared__ uint16_t s_fp[kSumWarps][kSumFlagged][kSumPartners];
    __shared__ int8_t s_np[kSumWarps][kSumFlagged];
    __syncthreads();
    const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
    const int line = int(blockIdx.x) * kSumWarps + warp;
    if (line >= A.lines)
        return;
    const uint32_t r0 = __ldg(A.off + line), r1 = __ldg(A.off + line + 1);
    const int n = int(r1 - r0);
    const uint32_t kmask = (kSliceMask << kSliceShift) | kRingMask;
    // the line's flagged records, in record order
    int nfl = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const bool f = i < n && (__ldg(A.key + r0 + i) & kFlagBit) != 0;
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, f);
        const int at = nfl + __popc(bal & ((1u << lane) - 1u));
        if (f && at < kSumFlagged)
            s_fl[warp][at] = uint16_t(i);
        nfl += __popc(bal);
    }
    const bool cached = nfl <= kSumFlagged;
    if (cached) {
        for (int k = lane; k < nfl; k += 32) {
            const int i = s_fl[warp][k];
            const uint32_t bk = __ldg(A.key + r0 + i) & kmask;
            int np = 0;
            for (int j = i - 1; j >= 0 && np <= kSumPartners; --j)
                if ((__ldg(A.key + r0 + j) & kmask) == bk) {
                    if (np < kSumPartners)
                        s_fp[warp][k][np] = uint16_t(j);
                    ++np;
                }
            s_np[warp][k] = int8_t(np > kSumPartners ? -1 : np);
        }
    }
    __syncwarp();
    for (int j = 0; j < nviews; ++j) {
        const double theta = __ldg(A.theta + view0 + j);
        unsigned long long c = 0, s = 0;
        for (int i = lane; i < n; i += 32) {
            if (__ldg(A.key + r0 + i) & kFlagBit) {
                if (!cached)
                    flagged_count_sum(A, s_rings, r0, i, theta, nullptr, -1, c, s);
                continue;
            }
            const RecRot o = rot_record(A, s_rings, r0 + i, theta);
            range_count_sum(o.b, o.lo, o.hi, o.seam, o.ng, c, s);
        }
        if (cached)
            for (int k = lane; k < nfl; k += 32)
                flagged_count_sum(A, s_rings, r0, s_fl[warp][k], theta, s_fp[warp][k], s_np[warp][k], c, s);
        for (int o = 16; o > 0; o >>= 1) {
            c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
            s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        }
        if (lane == 0) {
            const size_t k = size_t(j) * A.lines + line;
            counts[k] = uint32_t(c);
            sums[k] = s;
        }
    }
}

void launch_checksums(const TraceArgs& A, int view0, int nviews, int n_rings, int max_recs,
                      uint32_t* counts, unsigned long long* sums, cudaStream_t st) {
    if (nviews <= 0 || A.lines <= 0)
        return;
    (void)max_recs;
    const size_t sm = sizeof(RingRow) * size_t(n_rings + 1);
    UB_CUDA(cudaFuncSetAttribute(checksum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    checksum_kernel<<<unsigned((A.lines + kSumWarps - 1) / kSumWarps), 32 * kSumWarps, sm, st>>>(
        A, view0, nviews, n_rings, counts, sums);
    check_launch();
}

template <int NT>
__global__ void __launch_bounds__(NT) trace_dump_kernel(TraceArgs A, uint32_t unit0, int max_recs,
                                                        const uint32_t* __restrict__ pos,
                                                        uint32_t* out) {
    extern __shared__ uint32_t smem[];
    const TraceSmem S = carve_trace_smem<NT>(smem, max_recs);
    const uint32_t unit = unit0 + blockIdx.x;
    const int v = unit / A.lines, line = unit % A.lines;
    const int n = block_trace<NT>(A, line, A.theta[v], S, true);
    uint32_t* o = out + (pos[blockIdx.x] - pos[0]);
    for (int i = threadIdx.x; i < n; i += NT)
        o[i] = S.idx[i];
}

void launch_trace_dump(const TraceArgs& A, uint32_t unit0, uint32_t units, int max_recs,
                       int max_cells, const uint32_t* pos, uint32_t* out, cudaStream_t st) {
    if (units == 0)
        return;
    const size_t sm = trace_smem_bytes(128, max_recs, max_cells);
    UB_CUDA(cudaFuncSetAttribute(trace_dump_kernel<128>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    trace_dump_kernel<128><<<units, 128, sm, st>>>(A, unit0, max_recs, pos, out);
    check_launch();
}

template <int NT>
__global__ void __launch_bounds__(NT) crossed_kernel(TraceArgs A, int max_recs, uint8_t* crossed) {
    extern __shared__ uint32_t smem[];
    const TraceSmem S = carve_trace_smem<NT>(smem, max_recs);
    const int unit = blockIdx.x;
    const int v = unit / A.lines, line = unit % A.lines;
    const int n = block_trace<NT>(A, line, A.theta[v], S, true);
    for (int i = threadIdx.x; i < n; i += NT)
        crossed[S.idx[i]] = 1;
}

void launch_crossed(const TraceArgs& A, int views, int max_recs, int max_cells, uint8_t* crossed,
                    cudaStream_t st) {
    const long long units = (long long)views * A.lines;
    if (units <= 0)
        return;
    const size_t sm = trace_smem_bytes(128, max_recs, max_cells);
    UB_CUDA(cudaFuncSetAttribute(crossed_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(sm)));
    crossed_kernel<128><<<unsigned(units), 128, sm, st>>>(A, max_recs, crossed);
    check_launch();
}

// =============================================================================
// Gather/scatter shape per problem-chunk width P (problems per block):
//   NT threads, NCL = NT / P cell lanes, each lane holds up to KR of the
//   line's cells in registers so that all its loads are in flight at once and
//   the scatter needs no reload. Lines longer than NCL * KR spill the tail to a
//   re-read loop.
// =============================================================================
template <int P> struct Shape;
template <> struct Shape<1> { static constexpr int NT = 128, KR = 8; };
template <> struct Shape<2> { static constexpr int NT = 256, KR = 8; };
template <> struct Shape<4> { static constexpr int NT = 256, KR = 12; };
template <> struct Shape<8> { static constexpr int NT = 512, KR = 12; };
template <> struct Shape<16> { static constexpr int NT = 1024, KR = 12; };
template <> struct Shape<32> { static constexpr int NT = 1024, KR = 16; };

#define UB_DISPATCH_P(P_, CALL)                      \
    switch (P_) {                                    \
        case 1: { constexpr int PP = 1; CALL; } break;   \
        case 2: { constexpr int PP = 2; CALL; } break;   \
        case 4: { constexpr int PP = 4; CALL; } break;   \
        case 8: { constexpr int PP = 8; CALL; } break;   \
        case 16: { constexpr int PP = 16; CALL; } break; \
        default: { constexpr int PP = 32; CALL; } break; \
    }

// Sum over lanes with the same problem (lane % P) and over warps; returns the
// per-problem total in s_out[p] (threads < P write, then the block syncs).
template <int P, int NT>
__device__ __forceinline__ void block_problem_sum(double sum, double (*s_red)[P]) {
#pragma unroll
    for (int o = P; o < 32; o <<= 1)
        sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane < P)
        s_red[warp][lane] = sum;
    __syncthreads();
}

// K2: binary forward projector. One block per (view, line, problem chunk).
template <int P>
__global__ void __launch_bounds__(Shape<P>::NT) project_kernel(TraceArgs A,
                                                               const float* __restrict__ field,
                                                               int Sp, int nchunks, int max_recs,
                                                               float* __restrict__ out) {
    constexpr int NT = Shape<P>::NT, KR = Shape<P>::KR, NCL = NT / P;
    extern __shared__ uint32_t smem[];
    const TraceSmem S = carve_trace_smem<NT>(smem, max_recs);
    __shared__ double s_red[NT / 32][P];
    const int unit = blockIdx.x / nchunks, chunk = blockIdx.x % nchunks;
    const int v = unit / A.lines, line = unit % A.lines;
    const int n = block_trace<NT>(A, line, A.theta[v], S, true);
    const int p = threadIdx.x % P, cl = threadIdx.x / P;
    const size_t col = size_t(chunk) * P + p;
    float x[KR];
#pragma unroll
    for (int i = 0; i < KR; ++i) {
        const int c = cl + i * NCL;
        x[i] = c < n ? field[size_t(S.idx[c]) * Sp + col] : 0.f;
    }
    double sum = 0;
#pragma unroll
    for (int i = 0; i < KR; ++i)
        sum += double(x[i]);
    for (int c = cl + KR * NCL; c < n; c += NCL)
        sum += double(field[size_t(S.idx[c]) * Sp + col]);
    block_problem_sum<P, NT>(sum, s_red);
    if (threadIdx.x < P) {
        double t = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w)
            t += s_red[w][threadIdx.x];
        out[size_t(unit) * Sp + size_t(chunk) * P + threadIdx.x] = float(t);
    }
}

template <int P>
static void project_impl(const TraceArgs& A, int views, const float* field, int Sp, int max_recs,
                         int max_cells, float* out, cudaStream_t st) {
    constexpr int NT = Shape<P>::NT;
    const size_t sm = trace_smem_bytes(NT, max_recs, max_cells);
    UB_CUDA(cudaFuncSetAttribute(project_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(sm)));
    const int nchunks = Sp / P;
    const long long blocks = (long long)views * A.lines * nchunks;
    project_kernel<P><<<unsigned(blocks), NT, sm, st>>>(A, field, Sp, nchunks, max_recs, out);
    check_launch();
}

// K2 for problem stacks (S_pad % 4 == 0): one block per (view, line) traces
// once and streams every problem of every cell as float4s. Warp w covers cell
// lane w (all S_pad problems of a cell: contiguous 4*S_pad bytes), 4 cells in
// flight per thread; per-problem sums reduce across warps in shared memory.
constexpr int kProjNT = 512;

__global__ void __launch_bounds__(kProjNT) project_stack_kernel(TraceArgs A,
                                                                const float* __restrict__ field,
                                                                int Sp, int max_recs,
                                                                float* __restrict__ out) {
    extern __shared__ uint32_t smem[];
    const TraceSmem S = carve_trace_smem<kProjNT>(smem, max_recs);
    __shared__ double s_red[kProjNT * 4];
    const int unit = blockIdx.x;
    const int v = unit / A.lines, line = unit % A.lines;
    const int n = block_trace<kProjNT>(A, line, A.theta[v], S, true);
    const int C4 = Sp / 4;
    const int NCL = kProjNT / C4;
    const int t = threadIdx.x;
    const int col4 = t % C4, cl = t / C4;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if (cl < NCL) {
        const float4* __restrict__ f4 = reinterpret_cast<const float4*>(field);
        const uint32_t C4u = uint32_t(C4);
        int c = cl;
        for (; c + 3 * NCL < n; c += 4 * NCL) {
            float4 y[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                y[j] = __ldg(f4 + (S.idx[c + j * NCL] * C4u + uint32_t(col4)));
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                s0 += double(y[j].x);
                s1 += double(y[j].y);
                s2 += double(y[j].z);
                s3 += double(y[j].w);
            }
        }
        for (; c < n; c += NCL) {
            const float4 y = __ldg(f4 + (S.idx[c] * C4u + uint32_t(col4)));
            s0 += double(y.x);
            s1 += double(y.y);
            s2 += double(y.z);
            s3 += double(y.w);
        }
    }
    double* r = s_red + 4 * t;
    r[0] = s0;
    r[1] = s1;
    r[2] = s2;
    r[3] = s3;
    __syncthreads();
    for (int q = t; q < Sp; q += kProjNT) {
        const int c4 = q / 4, j = q % 4;
        double tot = 0;
        for (int k = 0; k < NCL; ++k)
            tot += s_red[4 * (k * C4 + c4) + j];
        out[size_t(unit) * Sp + q] = float(tot);
    }
}

void launch_project(const TraceArgs& A, int views, const float* field, int Sp, int max_recs,
                    int max_cells, float* out, cudaStream_t st) {
    if ((long long)views * A.lines == 0)
        return;
    if (Sp % 4 == 0 && Sp / 4 <= kProjNT) {
        const size_t sm = trace_smem_bytes(kProjNT, max_recs, max_cells);
        UB_CUDA(cudaFuncSetAttribute(project_stack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sm)));
        const long long blocks = (long long)views * A.lines;
        project_stack_kernel<<<unsigned(blocks), kProjNT, sm, st>>>(A, field, Sp, max_recs, out);
        check_launch();
        return;
    }
    UB_DISPATCH_P(stride_chunk(Sp), project_impl<PP>(A, views, field, Sp, max_recs, max_cells, out, st));
}

// K2 for one problem, fed by the tracer's traced lists (built once per
// geometry by the first reconstruction, api.cu build_lists): a warp per
// (view, line) streams the line's list (coalesced u32) and gathers the field,
// fp64 sum (generate_projections Binary, phantom.cpp:193-211); the same index
// sets in the same emission order as the trace-based kernel, without
// re-rotating and expanding the records.
constexpr int kProjListNT = 256;

__global__ void __launch_bounds__(kProjListNT) project_lists_kernel(const uint32_t* __restrict__ lists,
                                                                    const unsigned long long* __restrict__ lpos,
                                                                    uint64_t units, const float* __restrict__ field,
                                                                    float* __restrict__ out) {
    const uint64_t u = uint64_t(blockIdx.x) * (kProjListNT / 32) + (threadIdx.x >> 5);
    const int lane = int(threadIdx.x & 31);
    if (u >= units)
        return;
    const unsigned long long b = __ldg(lpos + u), e = __ldg(lpos + u + 1);
    double s = 0;
    unsigned long long k = b + unsigned(lane);
    for (; k + 96 < e; k += 128) {
        const uint32_t c0 = __ldcs(lists + k), c1 = __ldcs(lists + k + 32), c2 = __ldcs(lists + k + 64),
                       c3 = __ldcs(lists + k + 96);
        const float v0 = __ldg(field + c0), v1 = __ldg(field + c1), v2 = __ldg(field + c2), v3 = __ldg(field + c3);
        s += double(v0);
        s += double(v1);
        s += double(v2);
        s += double(v3);
    }
    for (; k < e; k += 32)
        s += double(__ldg(field + __ldcs(lists + k)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (lane == 0)
        out[u] = float(s);
}

void launch_project_lists(const uint32_t* lists, const unsigned long long* lpos, uint64_t units, const float* field,
                          float* out, cudaStream_t st) {
    if (units == 0)
        return;
    const uint64_t blocks = (units + kProjListNT / 32 - 1) / (kProjListNT / 32);
    project_lists_kernel<<<unsigned(blocks), kProjListNT, 0, st>>>(lists, lpos, units, field, out);
    check_launch();
}

// =============================================================================
// per-problem reductions over [n][Sp] arrays: blockIdx.y = 32-column tile,
// threadIdx.x = column in the tile, threadIdx.y = row lane.
// =============================================================================

// ProjectionSet::validate + auto_p_floor + all-zero test (solver.cpp:76-95)
// per problem: block partials (no atomics), then an in-order fold, so the
// positive-measurement sum (and with it p_floor) is the same on every run.
constexpr int kStatBlocks = 256;

__global__ void __launch_bounds__(256) proj_stats_kernel(const float* __restrict__ proj, int units, int S, int Sp,
                                                         double* __restrict__ part) {
    __shared__ double sh[8][32][4];
    const int col = blockIdx.y * 32 + threadIdx.x;
    double cnt = 0, sum = 0, nz = 0, bad = 0;
    if (col < S) {
        for (int u = blockIdx.x * blockDim.y + threadIdx.y; u < units; u += gridDim.x * blockDim.y) {
            const float m = proj[size_t(u) * Sp + col];
            if (!isfinite(m) || m < 0)
                bad = 1;
            if (m > 0) {
                cnt += 1;
                sum += double(m);
            }
            if (m != 0)
                nz = 1;
        }
    }
    sh[threadIdx.y][threadIdx.x][0] = cnt;
    sh[threadIdx.y][threadIdx.x][1] = sum;
    sh[threadIdx.y][threadIdx.x][2] = nz;
    sh[threadIdx.y][threadIdx.x][3] = bad;
    __syncthreads();
    if (threadIdx.y < 4 && col < S) {
        const int k = threadIdx.y;
        double acc = 0;
        for (int y = 0; y < 8; ++y)
            acc = k >= 2 ? fmax(acc, sh[y][threadIdx.x][k]) : acc + sh[y][threadIdx.x][k];
        part[(size_t(blockIdx.x) * S + col) * 4 + k] = acc;
    }
}

__global__ void stats_fold_kernel(const double* __restrict__ part, int S, int blocks, double* __restrict__ stats) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // col * 4 + k
    if (i >= 4 * S)
        return;
    const int k = i & 3;
    double acc = 0;
    for (int b = 0; b < blocks; ++b)
        acc = k >= 2 ? fmax(acc, part[size_t(b) * S * 4 + i]) : acc + part[size_t(b) * S * 4 + i];
    stats[i] = acc;
}

size_t proj_stats_words(int S) { return size_t(4) * S * (kStatBlocks + 1); }

void launch_proj_stats(const float* proj, int units, int S, int Sp, double* stats, cudaStream_t st) {
    const int blocks = std::max(1, std::min(cdiv(units, 8), kStatBlocks));
    double* part = stats + size_t(4) * S;
    proj_stats_kernel<<<dim3(unsigned(blocks), unsigned(cdiv(S, 32))), dim3(32, 8), 0, st>>>(proj, units, S, Sp,
                                                                                              part);
    check_launch();
    stats_fold_kernel<<<unsigned(cdiv(4 * S, 128)), 128, 0, st>>>(part, S, blocks, stats);
    check_launch();
}

__global__ void __launch_bounds__(256) sweep_updates_kernel(const float* __restrict__ proj,
                                                            const uint32_t* __restrict__ cells, int units, int S,
                                                            int Sp, unsigned long long* out) {
    __shared__ unsigned long long sh[8][32];
    const int col = blockIdx.y * 32 + threadIdx.x;
    unsigned long long acc = 0;
    if (col < S)
        for (int u = blockIdx.x * blockDim.y + threadIdx.y; u < units; u += gridDim.x * blockDim.y)
            if (proj[size_t(u) * Sp + col] != 0)
                acc += cells[u];
    sh[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && col < S) {
        unsigned long long t = 0;
        for (int y = 0; y < 8; ++y)
            t += sh[y][threadIdx.x];
        if (t)
            atomicAdd(out + col, t);
    }
}

void launch_sweep_updates(const float* proj, const uint32_t* cells, int units, int S, int Sp,
                          unsigned long long* out, cudaStream_t st) {
    dim3 block(32, 8);
    dim3 grid(unsigned(std::min(cdiv(units, 8), kStatBlocks)), unsigned(cdiv(S, 32)));
    sweep_updates_kernel<<<grid, block, 0, st>>>(proj, cells, units, S, Sp, out);
    check_launch();
}

__global__ void residual_kernel(const float* __restrict__ f, const float* __restrict__ prev,
                                const uint8_t* __restrict__ crossed, uint64_t cells, int S, int Sp,
                                unsigned int* out) {
    const int col = blockIdx.y * 32 + threadIdx.x;
    if (col >= S)
        return;
    float best = 0;
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.y + threadIdx.y; c < cells;
         c += uint64_t(gridDim.x) * blockDim.y) {
        if (!crossed[c])
            continue;
        const float a = f[c * Sp + col], b = prev[c * Sp + col];
        const float rel = float(fabs(double(a) - double(b)) / double(b));
        best = fmaxf(best, rel);
    }
    atomicMax(out + col, __float_as_uint(best));
}

void launch_residual(const float* field, const float* prev, const uint8_t* crossed, uint64_t cells,
                     int S, int Sp, unsigned int* out, cudaStream_t st) {
    dim3 block(32, 8);
    dim3 grid(unsigned(std::min<long long>(cdiv((long long)cells, 8), 2368)), unsigned(cdiv(S, 32)));
    residual_kernel<<<grid, block, 0, st>>>(field, prev, crossed, cells, S, Sp, out);
    check_launch();
}

__global__ void nonpositive_kernel(const float* __restrict__ f, uint64_t n,
                                   unsigned long long* out) {
    unsigned long long c = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        if (!(f[i] > 0))
            ++c;
    if (c)
        atomicAdd(out, c);
}

void launch_count_nonpositive(const float* field, uint64_t n, unsigned long long* out,
                              cudaStream_t st) {
    nonpositive_kernel<<<unsigned(std::min<long long>(cdiv((long long)n, 256), 4736)), 256, 0, st>>>(
        field, n, out);
    check_launch();
}

// =============================================================================
// layout transposes [S][n] <-> [n][Sp]
// =============================================================================

__global__ void to_interleaved_kernel(const float* __restrict__ in, float* __restrict__ out,
                                      uint64_t n, int S, int Sp, float pad) {
    __shared__ float tile[32][33];
    const uint64_t i0 = uint64_t(blockIdx.x) * 32;
    const int s0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int s = s0 + r;
        const uint64_t i = i0 + threadIdx.x;
        tile[r][threadIdx.x] = (s < S && i < n) ? in[uint64_t(s) * n + i] : pad;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const uint64_t i = i0 + r;
        const int s = s0 + threadIdx.x;
        if (i < n && s < Sp)
            out[i * Sp + s] = tile[threadIdx.x][r];
    }
}

void launch_to_interleaved(const float* in, float* out, uint64_t n, int S, int Sp, float pad,
                           cudaStream_t st) {
    dim3 grid(unsigned((n + 31) / 32), unsigned(cdiv(Sp, 32)));
    to_interleaved_kernel<<<grid, dim3(32, 8), 0, st>>>(in, out, n, S, Sp, pad);
    check_launch();
}

__global__ void from_interleaved_kernel(const float* __restrict__ in, float* __restrict__ out,
                                        uint64_t n, int S, int Sp) {
    __shared__ float tile[32][33];
    const uint64_t i0 = uint64_t(blockIdx.x) * 32;
    const int s0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const uint64_t i = i0 + r;
        const int s = s0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < n && s < Sp) ? in[i * Sp + s] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int s = s0 + r;
        const uint64_t i = i0 + threadIdx.x;
        if (s < S && i < n)
            out[uint64_t(s) * n + i] = tile[threadIdx.x][r];
    }
}

void launch_from_interleaved(const float* in, float* out, uint64_t n, int S, int Sp,
                             cudaStream_t st) {
    dim3 grid(unsigned((n + 31) / 32), unsigned(cdiv(S, 32)));
    from_interleaved_kernel<<<grid, dim3(32, 8), 0, st>>>(in, out, n, S, Sp);
    check_launch();
}

__global__ void fill_kernel(float* p, uint64_t n, float v) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

void launch_fill(float* p, uint64_t n, float v, cudaStream_t st) {
    if (n == 0)
        return;
    fill_kernel<<<unsigned(std::min<long long>(cdiv((long long)n, 256), 4736)), 256, 0, st>>>(p, n, v);
    check_launch();
}

// =============================================================================
// K4: USPG -> Cartesian.
// =============================================================================

// Inverse of uspg_to_cg_map (grid.cpp:75-99): pixel (row, col) of an n x n
// image -> flat index within a slice. Ring k is the perimeter of the centred
// 2k x 2k block, walked counter-clockwise from (c, c+k-1).
__device__ __forceinline__ uint32_t cg_inverse(int row, int col, int n) {
    const int c = n / 2;
    const int rr = row >= c ? row - c + 1 : c - row;
    const int qq = col >= c ? col - c + 1 : c - col;
    const int k = rr > qq ? rr : qq;
    int pos;
    if (col == c + k - 1 && row >= c)
        pos = row - c;                           // right edge, upward
    else if (row == c + k - 1)
        pos = k + (c + k - 2 - col);             // top edge, leftward
    else if (col == c - k)
        pos = 3 * k - 1 + (c + k - 2 - row);     // left edge, downward
    else if (row == c - k)
        pos = 5 * k - 2 + (col - (c - k + 1));   // bottom edge, rightward
    else
        pos = 7 * k - 3 + (row - (c - k + 1));   // right edge, up to the tail
    return 4u * uint32_t(k - 1) * uint32_t(k - 1) + uint32_t(pos);
}

// out[(p*slices + s)*n*n + pixel]; field element (p, cell) at cell*cs + p*ps
// Four consecutive output pixels per thread (npix is even, so a plane holds a
// multiple of 4 pixels) and kResPlanes output planes per block row
// (blockIdx.y): the pixel's source cells are found once (PERM: the reference
// permutation inverted per pixel, cg_inverse; otherwise the precomputed
// bin-point map, 0xFFFFFFFF = outside the disc) and reused for every plane,
// and the gathers of four planes are in flight at once before their
// streaming float4 stores.
constexpr int kResPlanes = 16;

template <bool PERM, bool VEC>
__global__ void __launch_bounds__(256) resample_kernel(const float* __restrict__ field, uint64_t cps,
                                                       int slices, int planes, uint64_t cs, uint64_t ps,
                                                       const uint32_t* __restrict__ map, int n,
                                                       float* __restrict__ out) {
    const uint32_t npx = uint32_t(n) * uint32_t(n);
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
    if (q >= npx)
        return;
    uint32_t m[4];
    if constexpr (PERM) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t px = q + uint32_t(k);
            m[k] = cg_inverse(int(px / uint32_t(n)), int(px % uint32_t(n)), n);
        }
    } else {
        const uint4 mm = __ldg(reinterpret_cast<const uint4*>(map + q));
        m[0] = mm.x, m[1] = mm.y, m[2] = mm.z, m[3] = mm.w;
    }
    const int p0 = int(blockIdx.y) * kResPlanes, p1 = min(planes, p0 + kResPlanes);
    for (int pl0 = p0; pl0 < p1; pl0 += 4) {
        float v[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int pl = min(pl0 + j, p1 - 1);
            const int s = pl % slices, p = pl / slices;
            const float* f = field + uint64_t(s) * cps * cs + uint64_t(p) * ps;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                v[j][k] = (!PERM && m[k] == 0xFFFFFFFFu) ? 0.f : __ldg(f + uint64_t(m[k]) * cs);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (pl0 + j >= p1)
                break;
            float* o = out + uint64_t(pl0 + j) * npx + q;
            if constexpr (VEC) {
                __stcs(reinterpret_cast<float4*>(o), make_float4(v[j][0], v[j][1], v[j][2], v[j][3]));
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    __stcs(o + k, v[j][k]);
            }
        }
    }
}

template <bool PERM>
static void resample_launch(const float* field, uint64_t cps, int slices, int S, int Sp,
                            const uint32_t* map, int n, float* out, cudaStream_t st) {
    // Sp > 0: interleaved [cells][Sp]; Sp <= 0: problem-major [S][cells]
    const uint64_t cells = cps * slices;
    const uint64_t cs = Sp > 0 ? uint64_t(Sp) : 1, ps = Sp > 0 ? 1 : cells;
    const int planes = slices * S;
    const uint32_t npx = uint32_t(n) * uint32_t(n);
    const int rows = (planes + kResPlanes - 1) / kResPlanes;
    if (rows > 65535)
        throw CudaError("resample: too many output planes for one launch");
    const dim3 grid(unsigned((npx / 4 + 255) / 256), unsigned(rows));
    if ((reinterpret_cast<uintptr_t>(out) & 15) == 0)
        resample_kernel<PERM, true><<<grid, 256, 0, st>>>(field, cps, slices, planes, cs, ps, map, n, out);
    else
        resample_kernel<PERM, false><<<grid, 256, 0, st>>>(field, cps, slices, planes, cs, ps, map, n, out);
    check_launch();
}

void launch_perm_resample(const float* field, uint64_t cps, int slices, int S, int Sp, int n,
                          float* out, cudaStream_t st) {
    if (uint64_t(n) * n * slices * S == 0)
        return;
    resample_launch<true>(field, cps, slices, S, Sp, nullptr, n, out, st);
}

// bin_point (tests/oracles.hpp:36-58) at pixel centres for any ring law
__global__ void bin_map_kernel(DevGrid g, int npix, uint32_t* map) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix * npix)
        return;
    const int row = i / npix, col = i % npix;
    const double px = 2.0 * g.radius / npix;
    const double y = (row + 0.5 - npix / 2) * px;
    const double x = (col + 0.5 - npix / 2) * px;
    const double rho = hypot_cr(x, y);
    uint32_t v = 0xFFFFFFFFu;
    if (rho < g.radius) {
        const int ring = int(floor(rho / g.ring_spacing)) + 1;
        if (ring <= g.n_rings) {
            const int ng = int(g.rings[ring].count);
            const double phi = azimuth_deg(x, y);
            int sector = int(phi * (ng / 360.0));
            if (sector >= ng)
                sector = ng - 1;
            v = g.rings[ring].head + uint32_t(sector);
        }
    }
    map[i] = v;
}

void launch_bin_map(const DevGrid& g, int npix, uint32_t* map, cudaStream_t st) {
    bin_map_kernel<<<cdiv((long long)npix * npix, 256), 256, 0, st>>>(g, npix, map);
    check_launch();
}

void launch_map_resample(const float* field, uint64_t cps, int slices, int S, int Sp,
                         const uint32_t* map, int npix, float* out, cudaStream_t st) {
    if (uint64_t(npix) * npix * slices * S == 0)
        return;
    resample_launch<false>(field, cps, slices, S, Sp, map, npix, out, st);
}

// pixel -> cell of the reference permutation (the inverse of uspg_to_cg_map)
__global__ void perm_map_kernel(int n, uint32_t* map) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * n)
        return;
    map[i] = cg_inverse(i / n, i % n, n);
}

void launch_perm_map(int n, uint32_t* map, cudaStream_t st) {
    perm_map_kernel<<<cdiv((long long)n * n, 256), 256, 0, st>>>(n, map);
    check_launch();
}

// Tiled resample: a block owns one 32 x 32 pixel tile and kResPlanes output
// planes. The tile's distinct source cells (tcells, ascending: a few dozen
// runs of consecutive cells, one per ring crossed) are gathered per plane
// into shared memory with coalesced loads, then every pixel reads its cell
// from shared memory (slot, tile-major) and the rows are written as
// streaming float4s. The scattered per-pixel gathers of resample_kernel
// become per-run loads: the field is read about once and the output written
// once (8 B per output pixel).
constexpr int kTile = 32, kTileNTr = 256;

__global__ void __launch_bounds__(kTileNTr) tiled_resample_kernel(const float* __restrict__ field, uint64_t cps,
                                                                  int slices, int planes, uint64_t cs, uint64_t ps,
                                                                  const uint32_t* __restrict__ toff,
                                                                  const uint32_t* __restrict__ tcells,
                                                                  const uint16_t* __restrict__ slot, int n,
                                                                  float* __restrict__ out) {
    __shared__ float buf[2][kTile * kTile];
    const int tiles_x = n / kTile;
    const int tile = int(blockIdx.x);
    const int ty = tile / tiles_x, tx = tile % tiles_x;
    const int t = int(threadIdx.x);
    const uint32_t b = __ldg(toff + tile), D = __ldg(toff + tile + 1) - b;
    uint32_t cell[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t i = uint32_t(t + k * kTileNTr);
        cell[k] = i < D ? __ldg(tcells + b + i) : 0u;
    }
    const uint2 sl = __ldg(reinterpret_cast<const uint2*>(slot + size_t(tile) * kTile * kTile) + t);
    const uint32_t s4[4] = {sl.x & 0xFFFFu, sl.x >> 16, sl.y & 0xFFFFu, sl.y >> 16};
    const int lp = 4 * t, row = ty * kTile + lp / kTile, col = tx * kTile + lp % kTile;
    const uint32_t npx = uint32_t(n) * uint32_t(n);
    const int p0 = int(blockIdx.y) * kResPlanes, p1 = min(planes, p0 + kResPlanes);
    for (int pl = p0; pl < p1; ++pl) {
        const int s = pl % slices, p = pl / slices;
        const float* f = field + uint64_t(s) * cps * cs + uint64_t(p) * ps;
        float* sb = buf[pl & 1];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = uint32_t(t + k * kTileNTr);
            if (i < D)
                sb[i] = __ldg(f + uint64_t(cell[k]) * cs);
        }
        __syncthreads();
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            v[k] = s4[k] == 0xFFFFu ? 0.f : sb[s4[k]];
        __stcs(reinterpret_cast<float4*>(out + uint64_t(pl) * npx + uint64_t(row) * n + col),
               make_float4(v[0], v[1], v[2], v[3]));
    }
}

void launch_tiled_resample(const float* field, uint64_t cps, int slices, int S, int Sp, const uint32_t* toff,
                           const uint32_t* tcells, const uint16_t* slot, int n, float* out, cudaStream_t st) {
    if (uint64_t(n) * n * slices * S == 0)
        return;
    const uint64_t cells = cps * slices;
    const uint64_t cs = Sp > 0 ? uint64_t(Sp) : 1, ps = Sp > 0 ? 1 : cells;
    const int planes = slices * S;
    const int rows = (planes + kResPlanes - 1) / kResPlanes;
    if (rows > 65535)
        throw CudaError("resample: too many output planes for one launch");
    const dim3 grid(unsigned((n / kTile) * (n / kTile)), unsigned(rows));
    tiled_resample_kernel<<<grid, kTileNTr, 0, st>>>(field, cps, slices, planes, cs, ps, toff, tcells, slot, n, out);
    check_launch();
}

// cartesian_to_field (proj/src/phantom.cpp:165-180): dst[flat] =
// img[map[flat]], i.e. pixel i writes the cell cg_inverse(i). A thread takes
// four consecutive pixels (coalesced float4 reads; n is even) of kResPlanes
// planes; the permutation is computed once per pixel.
__global__ void __launch_bounds__(256) cart_to_field_kernel(const float* __restrict__ img, uint64_t cps,
                                                            int slices, int planes, uint64_t cs, uint64_t ps,
                                                            int n, float* __restrict__ field) {
    const uint32_t npx = uint32_t(n) * uint32_t(n);
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
    if (q >= npx)
        return;
    uint32_t m[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t px = q + uint32_t(k);
        m[k] = cg_inverse(int(px / uint32_t(n)), int(px % uint32_t(n)), n);
    }
    const int p0 = int(blockIdx.y) * kResPlanes, p1 = min(planes, p0 + kResPlanes);
    for (int pl = p0; pl < p1; ++pl) {
        const int s = pl % slices, p = pl / slices;
        const float* src = img + uint64_t(pl) * npx + q;
        float v[4];
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const float4 x = __ldcs(reinterpret_cast<const float4*>(src));
            v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                v[k] = __ldcs(src + k);
        }
        float* f = field + uint64_t(s) * cps * cs + uint64_t(p) * ps;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            f[uint64_t(m[k]) * cs] = v[k];
    }
}

void launch_cart_to_field(const float* img, uint64_t cps, int slices, int S, int Sp, int n, float* field,
                          cudaStream_t st) {
    const uint64_t npx = uint64_t(n) * uint64_t(n);
    if (npx * slices * S == 0)
        return;
    const uint64_t cells = cps * slices;
    const uint64_t cs = Sp > 0 ? uint64_t(Sp) : 1, ps = Sp > 0 ? 1 : cells;
    const int planes = slices * S;
    const int rows = (planes + kResPlanes - 1) / kResPlanes;
    if (rows > 65535)
        throw CudaError("cartesian_to_field: too many planes for one launch");
    const dim3 grid(unsigned((npx / 4 + 255) / 256), unsigned(rows));
    cart_to_field_kernel<<<grid, 256, 0, st>>>(img, cps, slices, planes, cs, ps, n, field);
    check_launch();
}

__global__ void cg_map_kernel(int n, uint32_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * n)
        return;
    const int row = i / n, col = i % n;
    out[cg_inverse(row, col, n)] = uint32_t(i);
}

void launch_cg_map(int n, uint32_t* out, cudaStream_t st) {
    cg_map_kernel<<<cdiv((long long)n * n, 256), 256, 0, st>>>(n, out);
    check_launch();
}

// ---- diagnostics: the device math the generator uses, for parity tests ----
__global__ void diag_math_kernel(int n, const double* __restrict__ x, const double* __restrict__ y,
                                 double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    out[5 * i + 0] = atan2_gen(y[i], x[i]);
    out[5 * i + 1] = hypot_cr(x[i], y[i]);
    out[5 * i + 2] = azimuth_deg(x[i], y[i]);
    out[5 * i + 3] = atan2(y[i], x[i]);
    out[5 * i + 4] = atan2_cr(y[i], x[i]);
}

void launch_diag_math(int n, const double* x, const double* y, double* out, cudaStream_t st) {
    if (n <= 0)
        return;
    diag_math_kernel<<<cdiv(n, 256), 256, 0, st>>>(n, x, y, out);
    check_launch();
}

}  // namespace ub
