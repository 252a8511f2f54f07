// Double-double arithmetic and correctly rounded atan2 / hypot for the
// K1 generator (and the bin-point resample map).
//
// The reference computes chord azimuths with glibc's atan2 and ring radii
// with glibc's hypot (geometry.cpp:39-46,216). CUDA's atan2 / hypot carry up
// to 2 ulp of error, which flips sector bins for points that sit on a sector
// edge. glibc's results are (up to vanishingly rare hard cases) the correctly
// rounded values, so the device evaluates both functions in double-double
// (~2^-100 relative error) and rounds once: the azimuths then match the
// reference bit for bit.
#pragma once

#include <cmath>

namespace ub {
namespace dd {

struct D {
    double hi, lo;
};

__device__ __forceinline__ D quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}
__device__ __forceinline__ D two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ D two_prod(double a, double b) {
    const double p = a * b;
    return {p, fma(a, b, -p)};
}
__device__ __forceinline__ D add(D x, D y) {
    D s = two_sum(x.hi, y.hi);
    const D t = two_sum(x.lo, y.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ D neg(D x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ D sub(D x, D y) { return add(x, neg(y)); }
__device__ __forceinline__ D mul(D x, D y) {
    D p = two_prod(x.hi, y.hi);
    p.lo += x.hi * y.lo;
    p.lo += x.lo * y.hi;
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ D mul_d(D x, double b) {
    D p = two_prod(x.hi, b);
    p.lo += x.lo * b;
    return quick_two_sum(p.hi, p.lo);
}
// a / b with one fp64 division: three quotient terms from the reciprocal of
// b.hi, each correcting the remainder of the previous (fp64 division is a
// multi-instruction sequence, the generator's atan2 needed six of them)
__device__ __forceinline__ D div(D a, D b) {
    const double inv = 1.0 / b.hi;
    const double q1 = a.hi * inv;
    D r = sub(a, mul_d(b, q1));
    const double q2 = r.hi * inv;
    r = sub(r, mul_d(b, q2));
    const double q3 = r.hi * inv;
    const D q = quick_two_sum(q1, q2);
    return add(q, D{q3, 0.0});
}

// atan(k/64), k = 0..64, as double-double (generated with mpmath at 300 bits)
__device__ const double kAtanTab[65][2] = {
    {0x0.0p+0, 0x0.0p+0},  // atan(0/64)
    {0x1.fff555bbb729bp-7, -0x1.220c39d4dff50p-61},  // atan(1/64)
    {0x1.ffd55bba97625p-6, -0x1.5ec431444912cp-60},  // atan(2/64)
    {0x1.7fb818430da2ap-5, -0x1.86ef8f794f105p-63},  // atan(3/64)
    {0x1.ff55bb72cfdeap-5, -0x1.c934d86d23f1dp-60},  // atan(4/64)
    {0x1.3f59f0e7c559dp-4, 0x1.ac4ce285df847p-58},  // atan(5/64)
    {0x1.7ee182602f10fp-4, -0x1.cfb654c0c3d98p-58},  // atan(6/64)
    {0x1.be39ebe6f07c3p-4, 0x1.f7b8f29a05987p-58},  // atan(7/64)
    {0x1.fd5ba9aac2f6ep-4, -0x1.cd37686760c17p-59},  // atan(8/64)
    {0x1.1e1fafb043727p-3, -0x1.b485914dacf8cp-59},  // atan(9/64)
    {0x1.3d6eee8c6626cp-3, 0x1.61a3b0ce9281bp-57},  // atan(10/64)
    {0x1.5c9811e3ec26ap-3, -0x1.054ab2c010f3dp-58},  // atan(11/64)
    {0x1.7b97b4bce5b02p-3, 0x1.347b0b4f881cap-58},  // atan(12/64)
    {0x1.9a6a8e96c8626p-3, 0x1.cf601e7b4348ep-59},  // atan(13/64)
    {0x1.b90d7529260a2p-3, 0x1.17b10d2e0e5abp-61},  // atan(14/64)
    {0x1.d77d5df205736p-3, 0x1.c648d1534597ep-57},  // atan(15/64)
    {0x1.f5b75f92c80ddp-3, 0x1.8ab6e3cf7afbdp-57},  // atan(16/64)
    {0x1.09dc597d86362p-2, 0x1.62e47390cb865p-56},  // atan(17/64)
    {0x1.18bf5a30bf178p-2, 0x1.30ca4748b1bf9p-57},  // atan(18/64)
    {0x1.278372057ef46p-2, -0x1.077cdd36dfc81p-56},  // atan(19/64)
    {0x1.362773707ebccp-2, -0x1.963a544b672d8p-57},  // atan(20/64)
    {0x1.44aa436c2af0ap-2, -0x1.5d5e43c55b3bap-56},  // atan(21/64)
    {0x1.530ad9951cd4ap-2, -0x1.2566480884082p-57},  // atan(22/64)
    {0x1.614840309cfe2p-2, -0x1.a725715711f00p-56},  // atan(23/64)
    {0x1.6f61941e4def1p-2, -0x1.c63aae6f6e918p-56},  // atan(24/64)
    {0x1.7d5604b63b3f7p-2, 0x1.69c885c2b249ap-56},  // atan(25/64)
    {0x1.8b24d394a1b25p-2, 0x1.b6d0ba3748fa8p-56},  // atan(26/64)
    {0x1.98cd5454d6b18p-2, 0x1.9e6c988fd0a77p-56},  // atan(27/64)
    {0x1.a64eec3cc23fdp-2, -0x1.24dec1b50b7ffp-56},  // atan(28/64)
    {0x1.b3a911da65c6cp-2, 0x1.ae187b1ca5040p-56},  // atan(29/64)
    {0x1.c0db4c94ec9f0p-2, -0x1.cc1ce70934c34p-56},  // atan(30/64)
    {0x1.cde53432c1351p-2, -0x1.a2cfa4418f1adp-56},  // atan(31/64)
    {0x1.dac670561bb4fp-2, 0x1.a2b7f222f65e2p-56},  // atan(32/64)
    {0x1.e77eb7f175a34p-2, 0x1.0e53dc1bf3435p-56},  // atan(33/64)
    {0x1.f40dd0b541418p-2, -0x1.a3992dc382a23p-57},  // atan(34/64)
    {0x1.0039c73c1a40cp-1, -0x1.b32c949c9d593p-55},  // atan(35/64)
    {0x1.0657e94db30d0p-1, -0x1.d5b495f6349e6p-56},  // atan(36/64)
    {0x1.0c6145b5b43dap-1, 0x1.974fa13b5404fp-58},  // atan(37/64)
    {0x1.1255d9bfbd2a9p-1, -0x1.2bdaee1c0ee35p-58},  // atan(38/64)
    {0x1.1835a88be7c13p-1, 0x1.c621cec00c301p-55},  // atan(39/64)
    {0x1.1e00babdefeb4p-1, -0x1.928df287a668fp-58},  // atan(40/64)
    {0x1.23b71e2cc9e6ap-1, 0x1.c421c9f38224ep-57},  // atan(41/64)
    {0x1.2958e59308e31p-1, -0x1.09e73b0c6c087p-56},  // atan(42/64)
    {0x1.2ee628406cbcap-1, 0x1.c5d5e9ff0cf8dp-55},  // atan(43/64)
    {0x1.345f01cce37bbp-1, 0x1.1021137c71102p-55},  // atan(44/64)
    {0x1.39c391cd4171ap-1, -0x1.2304331d8bf46p-55},  // atan(45/64)
    {0x1.3f13fb89e96f4p-1, 0x1.ecf8b492644f0p-56},  // atan(46/64)
    {0x1.445065b795b56p-1, -0x1.f76d0163f79c8p-56},  // atan(47/64)
    {0x1.4978fa3269ee1p-1, 0x1.2419a87f2a458p-56},  // atan(48/64)
    {0x1.4e8de5bb6ec04p-1, 0x1.4a33dbeb3796cp-55},  // atan(49/64)
    {0x1.538f57b89061fp-1, -0x1.1bb74abda520cp-55},  // atan(50/64)
    {0x1.587d81f732fbbp-1, -0x1.5e5c9d8c5a950p-56},  // atan(51/64)
    {0x1.5d58987169b18p-1, 0x1.0028e4bc5e7cap-57},  // atan(52/64)
    {0x1.6220d115d7b8ep-1, -0x1.2b785350ee8c1p-57},  // atan(53/64)
    {0x1.66d663923e087p-1, -0x1.6ea6febe8bbbap-56},  // atan(54/64)
    {0x1.6b798920b3d99p-1, -0x1.a80386188c50ep-55},  // atan(55/64)
    {0x1.700a7c5784634p-1, -0x1.8c34d25aadef6p-56},  // atan(56/64)
    {0x1.748978fba8e0fp-1, 0x1.7b2a6165884a1p-59},  // atan(57/64)
    {0x1.78f6bbd5d315ep-1, 0x1.406a089803740p-55},  // atan(58/64)
    {0x1.7d528289fa093p-1, 0x1.560821e2f3aa9p-55},  // atan(59/64)
    {0x1.819d0b7158a4dp-1, -0x1.bf76229d3b917p-56},  // atan(60/64)
    {0x1.85d69576cc2c5p-1, 0x1.6b66e7fc8b8c3p-57},  // atan(61/64)
    {0x1.89ff5ff57f1f8p-1, -0x1.55b9a5e177a1bp-55},  // atan(62/64)
    {0x1.8e17aa99cc05ep-1, -0x1.ec182ab042f61p-56},  // atan(63/64)
    {0x1.921fb54442d18p-1, 0x1.1a62633145c07p-55},  // atan(64/64)
};
constexpr double kPiHi = 0x1.921fb54442d18p+1, kPiLo = 0x1.1a62633145c07p-53;
constexpr double kPi2Hi = 0x1.921fb54442d18p+0, kPi2Lo = 0x1.1a62633145c07p-54;

constexpr double kInv3Hi = 0x1.5555555555555p-2, kInv3Lo = 0x1.5555555555555p-56;
constexpr double kInv5Hi = 0x1.999999999999ap-3, kInv5Lo = -0x1.999999999999ap-57;
constexpr double kInv7Hi = 0x1.2492492492492p-3, kInv7Lo = 0x1.2492492492492p-57;

// atan(t) for t in [0, 1] (double-double): t = c + ..., c = k/64 from the
// table, atan(t) = atan(c) + atan(u), u = (t - c) / (1 + t c), |u| <= 1/128,
// atan(u) = u * P(u^2) with the series to u^19.
__device__ __forceinline__ D atan01(D t) {
    const int k = min(max(int(t.hi * 64.0 + 0.5), 0), 64);
    const double c = k * (1.0 / 64.0);
    const D num = sub(t, D{c, 0.0});
    const D den = add(D{1.0, 0.0}, mul_d(t, c));
    const D u = div(num, den);
    const D z = mul(u, u);
    const double zd = z.hi;
    const double tail =
        1.0 / 9 - zd * (1.0 / 11 - zd * (1.0 / 13 - zd * (1.0 / 15 - zd * (1.0 / 17 - zd * (1.0 / 19)))));
    D r{tail, 0.0};
    r = add(mul(z, r), D{-kInv7Hi, -kInv7Lo});
    r = add(mul(z, r), D{kInv5Hi, kInv5Lo});
    r = add(mul(z, r), D{-kInv3Hi, -kInv3Lo});
    r = add(mul(z, r), D{1.0, 0.0});
    return add(D{kAtanTab[k][0], kAtanTab[k][1]}, mul(u, r));
}

// atan(t) for t = th + tl in [0, 1] to a relative error below 2^-65 (the
// quick form of atan01: double-double only where the error needs it).
//   t - c = (th - c) + tl        th - c exact (Sterbenz; c = 0 trivially)
//   1 + t c = 1 + p + pe + tl c  p + pe = th c exactly (fma)
//   u = (t - c) / (1 + t c)      u1 + u2: one reciprocal and one residual,
//                                error ~2^-100 |u|
//   atan(u) = u + u s            s = -z/3 + z^2/5 - ... - z^5/11, z = u1^2 in
//                                double: |s| <= 2^-15.5, relative error of s
//                                <= 5 * 2^-53 (z's rounding and u1 for u,
//                                Horner), truncation z^6/13 <= 2^-87: the
//                                term u s is good to 2^-66.2 |u|
//   atan(c) + atan(u)            table (hi, lo) + u1 exactly (two_sum), the
//                                small terms summed in double: rounding
//                                <= 2^-66.4 |u| + 2^-104 |R|
// and |u| <= |R| (k = 0: R = atan(u); k >= 1: |u| <= 1/128 < R), so the
// result (normalized) is within 2^-65.2 |R| of atan(t).
__device__ __forceinline__ D atan01_quick(double th, double tl) {
    // th * 64 is exact; rounding it to the nearest integer keeps
    // th >= c / 2 for k >= 1 (Sterbenz) — th * 64 + 0.5 could round up
    const int k = int(rint(th * 64.0));
    const double c = k * (1.0 / 64.0);
    const D num = two_sum(th - c, tl);
    const double p = th * c;
    const double pe = fma(th, c, -p);
    D den = quick_two_sum(1.0, p);
    den.lo += pe + tl * c;
    const double inv = 1.0 / den.hi;
    const double u1 = num.hi * inv;
    const double rr = fma(-u1, den.hi, num.hi) + (num.lo - u1 * den.lo);
    const double u2 = rr * inv;
    const double z = u1 * u1;
    const double s = z * (-1.0 / 3 + z * (1.0 / 5 + z * (-1.0 / 7 + z * (1.0 / 9 - z * (1.0 / 11)))));
    const D h = two_sum(kAtanTab[k][0], u1);
    const double l = h.lo + (kAtanTab[k][1] + (u2 + u1 * s));
    return quick_two_sum(h.hi, l);
}

}  // namespace dd

// Quick form of atan2_cr for the generator's finite, nonzero inputs: the
// quotient as a double-double from one reciprocal (th + tl, error ~2^-102),
// atan01_quick, the quadrant shifts in double-double (π/2 - R >= R and
// π - R >= R: no cancellation), then Ziv's test: with the result H + L
// within 2^-62 H of the true value (margin 8 over the bound above), H is
// its correct rounding whenever |L| + 2^-62 H is below half the spacing of
// the doubles on L's side of H. Otherwise (~0.2% of inputs, or operands
// outside [2^-900, 2^900], or a quotient below 2^-400) ok = false and the
// caller evaluates atan2_cr.
__device__ __forceinline__ double atan2_quick(double y, double x, bool& ok) {
    const double ax = fabs(x), ay = fabs(y);
    const double big = fmax(ax, ay), small = fmin(ax, ay);
    ok = false;
    if (!(small >= 0x1p-900 && big <= 0x1p900))
        return 0.0;
    const double inv = 1.0 / big;
    const double th = small * inv;
    if (!(th >= 0x1p-400))
        return 0.0;
    const double tl = fma(-th, big, small) * inv;
    dd::D r = dd::atan01_quick(th, tl);
    if (ay > ax)
        r = dd::sub(dd::D{dd::kPi2Hi, dd::kPi2Lo}, r);
    if (x < 0.0)
        r = dd::sub(dd::D{dd::kPiHi, dd::kPiLo}, r);
    // r.hi > 0: half the spacing of the doubles around it is ulp(r.hi) / 2,
    // or ulp / 4 below a power of two when r.lo < 0
    const long long b = __double_as_longlong(r.hi);
    double half = __longlong_as_double(b & 0x7ff0000000000000LL) * 0x1p-53;
    if ((b & 0x000fffffffffffffLL) == 0 && r.lo < 0.0)
        half *= 0.5;
    ok = fabs(r.lo) < half - r.hi * 0x1p-62;
    return y < 0.0 ? -r.hi : r.hi;
}

// Correctly rounded atan2 (IEEE special cases as C99 Annex F for finite
// and signed-zero inputs; infinities, NaNs and operands whose larger
// magnitude is outside [2^-900, 2^900] defer to the CUDA libdevice).
__device__ __forceinline__ double atan2_cr(double y, double x) {
    if (isnan(x) || isnan(y) || isinf(x) || isinf(y))
        return atan2(y, x);
    if (y == 0.0) {
        if (x > 0.0 || (x == 0.0 && !signbit(x)))
            return y;
        return copysign(dd::kPiHi, y);
    }
    if (x == 0.0)
        return copysign(dd::kPi2Hi, y);
    const double ax = fabs(x), ay = fabs(y);
    // the reciprocals below need normal operands (grid coordinates are far
    // inside this range; outside it the libdevice atan2)
    if (!(fmax(ax, ay) <= 0x1p900 && fmax(ax, ay) >= 0x1p-900))
        return atan2(y, x);
    dd::D r;
    if (ay <= ax) {
        r = dd::atan01(dd::div(dd::D{ay, 0.0}, dd::D{ax, 0.0}));
    } else {
        r = dd::sub(dd::D{dd::kPi2Hi, dd::kPi2Lo},
                    dd::atan01(dd::div(dd::D{ax, 0.0}, dd::D{ay, 0.0})));
    }
    if (x < 0.0)
        r = dd::sub(dd::D{dd::kPiHi, dd::kPiLo}, r);
    const double res = r.hi + r.lo;
    return y < 0.0 ? -res : res;
}

// The generator's atan2: the quick form, atan2_cr where its rounding is not
// certain (bit-identical to atan2_cr on every input).
__device__ __forceinline__ double atan2_gen(double y, double x) {
    bool ok;
    const double q = atan2_quick(y, x, ok);
    return ok ? q : atan2_cr(y, x);
}

// Correctly rounded hypot for the coordinate range of the grids (|x|,|y| in
// [1e-150, 1e150]; outside it the CUDA libdevice hypot is used).
__device__ __forceinline__ double hypot_cr(double x, double y) {
    const double ax = fabs(x), ay = fabs(y);
    const double big = fmax(ax, ay), small = fmin(ax, ay);
    if (small == 0.0)
        return big;
    if (!(big < 1e150) || small < 1e-150)
        return hypot(x, y);
    const dd::D s = dd::add(dd::two_prod(ax, ax), dd::two_prod(ay, ay));
    const double r = sqrt(s.hi);
    const dd::D r2 = dd::two_prod(r, r);
    const dd::D diff = dd::sub(s, r2);
    const double corr = diff.hi / (2.0 * r);
    return r + corr;
}

}  // namespace ub
