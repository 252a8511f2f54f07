"""Device path vs the reference library / oracle on the same seeded inputs.

Every call goes through the C ABI (lib/libuscg_b200.so). Tolerances:
- indices, offsets, slice/ring, counters, crossed masks: bit-exact;
- generator azimuths (fp64): bit-exact except ulp-level atan2 differences
  (CUDA atan2 vs glibc), gated at <= 4 ulp;
- projections: fp32 field summed in fp64 vs the reference's fp64: rel <= 1e-6;
- reconstructed fields after a few sweeps (fp32 vs fp64): max rel <= 1e-4
  (SURVEY.md §8(c) measured fp32 drift <= 8.2e-6 after 10-20 sweeps).
"""
import numpy as np
import pytest

from refgeoms import REF_GEOMS, cache_from_ref, ref_tracer, thetas, ub_spec_geom, ulp_diff

pytestmark = pytest.mark.gpu


def _ub_tracer(ub, g):
    spec, geom = ub_spec_geom(ub, g)
    return spec, geom, ub.Tracer(geom, spec, False)


# ---------------------------------------------------------------------------
# K1 generator: FirstViewCache structure
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["fan32", "fan64q", "fan16", "cone16", "cone32", "fan128", "cone12", "cone32w"])
def test_generator_cache_matches_reference(ub, ref, name):
    g = REF_GEOMS[name]
    spec, geom, tr = _ub_tracer(ub, g)
    c = tr.cache()
    off, pa, pb, sl, rg = ref_tracer(ref, g).cache()
    assert np.array_equal(c.offsets, off)
    assert np.array_equal(c.slice, sl)
    assert np.array_equal(c.ring, rg)
    assert_phi_adjudicated(c.phi_a, pa)
    assert_phi_adjudicated(c.phi_b, pb)


def assert_phi_adjudicated(got, want):
    """Azimuths: the device atan2 is correctly rounded; glibc 2.39's is not in
    ~0.06% of calls (test_device_math_matches_glibc pins both rates against
    mpmath-free counts). So: bit-exact except isolated 1-ulp differences."""
    d = ulp_diff(got, want)
    assert d.max(initial=0) <= 2, "azimuth beyond 2 ulp (1 ulp of atan2 after the degree scaling)"
    assert np.count_nonzero(d) <= max(2, 0.005 * d.size), f"{np.count_nonzero(d)} of {d.size} differ"


def test_device_math_matches_glibc(ub, orc):
    """atan2 / hypot / azimuth_deg of the generator vs glibc on the chord
    endpoint distribution (unit disc) and on adversarial sector-edge points."""
    rng = np.random.default_rng(2208)
    n = 200_000
    r = np.sqrt(rng.uniform(0, 1, n))
    a = rng.uniform(-np.pi, np.pi, n)
    x, y = r * np.cos(a), r * np.sin(a)
    # points on exact sector edges of both ring laws (cos/sin of k*360/ng)
    ng = np.concatenate([4 * (2 * np.arange(1, 65) - 1), np.floor(2 * np.pi * (np.arange(64) + 0.5) + 0.5)])
    k = rng.integers(0, 10_000, ng.size)
    ang = np.radians((k % ng) * (360.0 / ng))
    rad = rng.uniform(0.01, 1, ng.size)
    x = np.concatenate([x, rad * np.cos(ang), [0.0, -0.0, 1.0, -1.0, 1e-300, 3.0]])
    y = np.concatenate([y, rad * np.sin(ang), [0.0, 0.0, 0.0, 0.0, 1e-300, -4.0]])
    dev = ub.uscg.diag_math(x, y)
    host = orc.math(x, y)
    mism_atan = np.count_nonzero(dev[:, 0].view(np.uint64) != host[:, 0].view(np.uint64))
    mism_hyp = np.count_nonzero(dev[:, 1].view(np.uint64) != host[:, 1].view(np.uint64))
    mism_az = np.count_nonzero(dev[:, 2].view(np.uint64) != host[:, 2].view(np.uint64))
    libdevice = np.count_nonzero(dev[:, 3].view(np.uint64) != host[:, 0].view(np.uint64))
    print(f"mismatches vs glibc: atan2 {mism_atan}, hypot {mism_hyp}, azimuth {mism_az}; "
          f"libdevice atan2 {libdevice} of {x.size}")
    # glibc 2.39 atan2/hypot are not correctly rounded in ~0.06% / ~0.6% of
    # these inputs (measured against mpmath at 200 bits, tests/test_oracle.py);
    # the device functions are, so they may differ from glibc by 1 ulp there.
    # (azimuth = atan2 * 180/pi, +360 below zero: a 1-ulp atan2 difference can
    # round to 2 ulp of the degree value)
    for k, lim, ulps in ((0, 0.002, 1), (1, 0.01, 1), (2, 0.002, 2)):
        d = ulp_diff(dev[:, k], host[:, k])
        assert d.max() <= ulps, (k, d.max())
        assert np.count_nonzero(d) <= lim * x.size, (k, np.count_nonzero(d))
    # the libdevice atan2 would miss far more often
    assert libdevice > 10 * mism_atan


def test_quick_atan2_is_the_double_double_atan2(ub):
    """The generator's atan2 (double-double quotient, a double series for
    atan(u), Ziv's rounding test, double-double fallback) returns exactly the
    full double-double atan2 (csrc/ddmath.cuh) on 4 M chord-like points and
    on inputs at the quick form's seams: table switches (y/x at (k+1/2)/64),
    |y| = |x| and its neighbours, axes, signed zeros, the [2^-900, 2^900]
    operand range and quotients near 2^-400."""
    rng = np.random.default_rng(20221)
    n = 4_000_000
    r = np.sqrt(rng.uniform(0, 1, n))
    a = rng.uniform(-np.pi, np.pi, n)
    xs, ys = [r * np.cos(a)], [r * np.sin(a)]
    m = 200_000
    k = rng.integers(0, 64, m)
    t = (k + 0.5) / 64 * (1 + rng.integers(-4, 5, m) * 2.0 ** -52)
    base = rng.uniform(0.01, 1.0, m)
    sx, sy = rng.choice([-1.0, 1.0], m), rng.choice([-1.0, 1.0], m)
    swap = rng.integers(0, 2, m).astype(bool)
    xs.append(np.where(swap, base * t, base) * sx)
    ys.append(np.where(swap, base, base * t) * sy)
    d = rng.uniform(0.01, 1.0, m)
    xs.append(d * sx)
    ys.append(np.nextafter(d, d * (1 + rng.integers(-3, 4, m) * 1e-16)) * sy)
    exps = rng.integers(-1000, 1000, m).astype(float)
    xs.append(rng.uniform(0.5, 1, m) * 2.0 ** exps * sx)
    with np.errstate(over="ignore", under="ignore"):
        ys.append(rng.uniform(0.5, 1, m) * 2.0 ** np.clip(exps + rng.integers(-420, 420, m), -1070, 1020) * sy)
    xs.append(np.array([0.0, -0.0, 1.0, -1.0, 0.0, 0.0, 1.0, -1.0, 2.0 ** -899, 2.0 ** 899, 1.0, 1.0]))
    ys.append(np.array([0.0, 0.0, 0.0, 0.0, 1.0, -1.0, 1.0, -1.0, 2.0 ** -899, 2.0 ** 899, 2.0 ** -400,
                        2.0 ** -401]))
    x = np.concatenate(xs)
    y = np.concatenate(ys)
    fin = np.isfinite(x) & np.isfinite(y)
    x, y = x[fin], y[fin]
    dev = ub.uscg.diag_math(x, y)
    same = dev[:, 0].view(np.uint64) == dev[:, 4].view(np.uint64)
    assert same.all(), (np.count_nonzero(~same), x[~same][:4], y[~same][:4])


@pytest.mark.parametrize("name", ["fan64q", "cone32"])
def test_quarter_symmetric_tracer_is_identical(ub, name):
    g = REF_GEOMS[name]
    spec, geom = ub_spec_geom(ub, g)
    a = ub.Tracer(geom, spec, False).cache()
    b = ub.Tracer(geom, spec, True).cache()
    for x, y in zip((a.offsets, a.phi_a, a.phi_b, a.slice, a.ring), (b.offsets, b.phi_a, b.phi_b, b.slice, b.ring)):
        assert np.array_equal(x, y)


def test_quarter_symmetry_rejects_asymmetric_panels(ub):
    spec = ub.GridSpec.square_2d(16)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=24, spacing_u=0.05, views=10)
    with pytest.raises(ub.InvalidArgument):
        ub.Tracer(geom, spec, True)


# ---------------------------------------------------------------------------
# per-view trace: index lists bit-exact
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["fan32", "fan16", "cone16", "cone12", "fan64q"])
def test_trace_line_matches_reference_every_view(ub, ref, name):
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    spec, geom = ub_spec_geom(ub, g)
    tr_imp = ub.Tracer.from_cache(spec, cache_from_ref(ub, rt), g["views"])
    tr_gen = ub.Tracer(geom, spec, False)
    th = thetas(g["views"])
    for v in range(g["views"]):
        for line in range(g["du"] * g["dv"]):
            want = rt.trace_line(line, th[v])
            assert np.array_equal(tr_imp.trace_line(line, th[v]), want), (v, line)
            assert np.array_equal(tr_gen.trace_line(line, th[v]), want), (v, line)


def test_trace_line_arbitrary_angles(ub, ref):
    g = REF_GEOMS["fan32"]
    rt = ref_tracer(ref, g)
    spec, geom = ub_spec_geom(ub, g)
    tr = ub.Tracer.from_cache(spec, cache_from_ref(ub, rt), g["views"])
    rng = np.random.default_rng(101)
    for _ in range(300):
        line = int(rng.integers(0, g["du"]))
        theta = float(rng.uniform(0, 720.0))
        assert np.array_equal(tr.trace_line(line, theta), rt.trace_line(line, theta))
    # a full turn is the identity
    for line in range(g["du"]):
        assert np.array_equal(tr.trace_line(line, 360.0), tr.trace_line(line, 0.0))


@pytest.mark.parametrize("name", ["fan32", "cone16", "fan64q"])
def test_rotated_reuse_checksums_match_reference(ub, ref, name):
    """uscg_trace_checksums (C5 rotated reuse): |active| and the index sum of
    every (view, line), from the records alone, equal the reference's
    Tracer::trace_line lists; a view sub-range is the same slice."""
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    spec, geom = ub_spec_geom(ub, g)
    tr = ub.Tracer.from_cache(spec, cache_from_ref(ub, rt), g["views"])
    th = thetas(g["views"])
    counts, sums = tr.trace_checksums()
    for v in range(g["views"]):
        for line in range(g["du"] * g["dv"]):
            want = rt.trace_line(line, th[v])
            assert counts[v, line] == want.size, (v, line)
            assert int(sums[v, line]) == int(want.astype(np.uint64).sum()), (v, line)
    c2, s2 = tr.trace_checksums(view0=1, nviews=2)
    assert np.array_equal(c2, counts[1:3]) and np.array_equal(s2, sums[1:3])
    with pytest.raises(ub.InvalidArgument):
        tr.trace_checksums(view0=g["views"] - 1, nviews=2)


@pytest.mark.parametrize("detector,volume", [("arc", False), ("flat", True)])
def test_rotated_reuse_checksums_generalized(ub, orc, detector, volume):
    """Same on the M1 sector law (arc fan, flat-panel cone over a volume) against
    the C restatement's traces, including the dedup-flagged chords."""
    spec, geom, _, oc = _m1_case(ub, orc, detector, volume=volume, dv=8 if volume else 1, views=12)
    ocache = ub.FirstViewCache(oc.offsets, oc.records["phi_a"].copy(), oc.records["phi_b"].copy(),
                               oc.records["slice"].copy(), oc.records["ring"].copy())
    tr = ub.Tracer.from_cache(spec, ocache, geom.views, geom.view_angles, geom=geom)
    counts, sums = tr.trace_checksums()
    th = geom.thetas()
    lines = tr.info()["lines"]
    for v in range(len(th)):
        for line in range(lines):
            want = oc.trace_line(line, th[v])
            assert counts[v, line] == want.size, (v, line)
            assert int(sums[v, line]) == int(np.asarray(want, np.uint64).sum()), (v, line)


def test_trace_counts_match_reference(ub, ref):
    g = REF_GEOMS["cone32"]
    rt = ref_tracer(ref, g)
    spec, geom, tr = _ub_tracer(ub, g)
    counts = tr.trace_counts()
    th = thetas(g["views"])
    for v in range(g["views"]):
        for line in range(0, g["du"] * g["dv"], 7):
            assert counts[v, line] == rt.trace_line(line, th[v]).size


@pytest.mark.parametrize("rec,theta,want", [
    ((95.0, 40.0, 0, 2), 0.0, [5, 6, 7]),
    ((350.0, 10.0, 0, 2), 0.0, [15, 4]),
    ((65.0, 10.0, 0, 2), 30.0, [5, 6, 7]),
    ((10.0, 190.0, 0, 2), 0.0, [4, 5, 6, 7, 8, 9, 10]),
    ((45.0, 45.0, 0, 2), 0.0, [5]),
])
def test_trace_chord_worked_examples(ub, rec, theta, want):
    """proj/tests/test_tracer.cpp:60-98 through a one-record imported cache."""
    spec = ub.GridSpec.square_2d(8)
    cache = ub.FirstViewCache(np.array([0, 1], np.uint32), np.array([rec[0]]), np.array([rec[1]]),
                              np.array([rec[2]], np.uint16), np.array([rec[3]], np.uint16))
    tr = ub.Tracer.from_cache(spec, cache, 1)
    assert tr.trace_line(0, theta).tolist() == want


def test_trace_chord_slice_offset(ub):
    spec = ub.GridSpec.cube_3d(8)
    cache = ub.FirstViewCache(np.array([0, 1], np.uint32), np.array([95.0]), np.array([40.0]),
                              np.array([3], np.uint16), np.array([2], np.uint16))
    tr = ub.Tracer.from_cache(spec, cache, 1)
    assert tr.trace_line(0, 0.0).tolist() == [3 * 64 + 5, 3 * 64 + 6, 3 * 64 + 7]


def test_dedup_of_overlapping_chords(ub, ref):
    """Two records of one (slice, ring) sharing sectors: the stamp dedup
    (tracer.cpp:181-195) keeps the first occurrence only."""
    spec = ub.GridSpec.square_2d(8)
    cache = ub.FirstViewCache(np.array([0, 3], np.uint32), np.array([95.0, 50.0, 80.0]),
                              np.array([40.0, 20.0, 100.0]), np.zeros(3, np.uint16),
                              np.array([2, 2, 3], np.uint16))
    tr = ub.Tracer.from_cache(spec, cache, 1)
    # ring 2 (12 cells, head 4): 95/40 -> 5,6,7 ; 50/20 -> 4,5 (5 dup) ; ring 3 (20 cells, head 16): 80/100 -> 20,21
    assert tr.trace_line(0, 0.0).tolist() == [5, 6, 7, 4, 20, 21]
    # +40: 135/80 -> 6,7,8 ; 90/60 -> 6,7 (both dup) ; 120/140 -> 22,23
    assert tr.trace_line(0, 40.0).tolist() == [6, 7, 8, 22, 23]
    # the record-level checksum applies the same dedup
    tr2 = ub.Tracer.from_cache(spec, cache, 2, np.array([0.0, 40.0]))
    counts, sums = tr2.trace_checksums()
    assert counts.tolist() == [[6], [5]]
    assert sums.tolist() == [[5 + 6 + 7 + 4 + 20 + 21], [6 + 7 + 8 + 22 + 23]]


# ---------------------------------------------------------------------------
# K2 projector
# ---------------------------------------------------------------------------


# ---------------------------------------------------------------------------
# K2' length-weighted projector (phantom.cpp:213-269)
# ---------------------------------------------------------------------------


def _clipped_length(s, d, radius, zhalf=None):
    """Length of the segment s -> d inside the disc of `radius` (2D) or the
    cylinder |z| <= zhalf (3D): what a unit field integrates to."""
    s, d = np.asarray(s, float), np.asarray(d, float)
    u = d - s
    lo, hi = 0.0, 1.0
    a = u[0] ** 2 + u[1] ** 2
    c = s[0] ** 2 + s[1] ** 2 - radius ** 2
    if a == 0:
        if c > 0:
            return 0.0
    else:
        b = 2 * (s[0] * u[0] + s[1] * u[1])
        disc = b * b - 4 * a * c
        if disc <= 0:
            return 0.0
        r = np.sqrt(disc)
        lo, hi = max(lo, (-b - r) / (2 * a)), min(hi, (-b + r) / (2 * a))
    if zhalf is not None:
        if u[2] == 0:
            if abs(s[2]) > zhalf:
                return 0.0
        else:
            t0, t1 = (-zhalf - s[2]) / u[2], (zhalf - s[2]) / u[2]
            lo, hi = max(lo, min(t0, t1)), min(hi, max(t0, t1))
    return max(0.0, hi - lo) * float(np.linalg.norm(u))


def _rot(p, deg):
    rad = deg * (np.pi / 180.0)
    c, s = np.cos(rad), np.sin(rad)
    return np.array([c * p[0] - s * p[1], s * p[0] + c * p[1], p[2]])


@pytest.mark.parametrize("name", ["fan16", "cone12", "fan32", "cone16"])
def test_length_weighted_matches_reference(ub, ref, name):
    """generate_projections(field, geom, LengthWeighted): the reference library
    on its own geometries (field values exact in fp32; fp32 output), and the
    unit field integrates to the in-volume path length (test_phantom.cpp:178-226).
    Adjudicated: a ray through the origin lies on a sector boundary in some
    views, where the reference splits its radial chords between the two
    sectors at -g0/g1 of two rounding residues; there only the path length
    (the sum over the pieces) is defined, and only it is compared."""
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    spec, geom = ub_spec_geom(ub, g)
    rng = np.random.default_rng(3)
    f = rng.integers(1, 64, spec.cell_count()) / 16.0
    want = rt.project_length(f)
    got = ub.generate_projections(ub.Field(spec, f.astype(np.float32)), geom, "length").data.reshape(want.shape)
    ones = ub.generate_projections(ub.Field(spec, np.ones(spec.cell_count(), np.float32)), geom,
                                   "length").data.reshape(want.shape)
    radius = 0.5 * spec.n * spec.ring_spacing
    zhalf = 0.5 * spec.slices() * spec.slice_height if g["volume"] else None
    src, det = geom.first_view_rays()
    th = thetas(g["views"])
    radial = 0
    for v in range(g["views"]):
        for line in range(geom.lines()):
            s, d = _rot(src[line], th[v]), _rot(det[line], th[v])
            u = d - s
            if abs(s[0] * u[1] - s[1] * u[0]) <= 1e-9 * np.hypot(u[0], u[1]):
                radial += 1  # through the origin: path length only
            else:
                assert abs(got[v, line] - want[v, line]) <= 2e-6 * abs(want[v, line]) + 1e-6, (v, line)
            exp = _clipped_length(s, d, radius, zhalf)
            if exp == 0:
                assert ones[v, line] <= 1e-6
            else:
                assert abs(ones[v, line] - exp) <= 1e-6 * exp + 1e-6, (v, line, ones[v, line], exp)
    assert radial <= g["views"] * g["dv"]  # at most the central ray of each detector row


def test_length_weighted_linearity_and_stack(ub):
    """Linear in the field (test_phantom.cpp:228-253), and a stack of fields
    projects like each field alone."""
    spec = ub.GridSpec.square_2d(16)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=11, spacing_u=0.2, views=5)
    rng = np.random.default_rng(13)
    f1, f2 = rng.uniform(0, 2, spec.cell_count()), rng.uniform(0, 2, spec.cell_count())
    a, b = 0.75, 1.5
    p = [ub.generate_projections(ub.Field(spec, x.astype(np.float32)), geom, "length").data
         for x in (f1, f2, a * f1 + b * f2)]
    np.testing.assert_allclose(p[2], a * p[0] + b * p[1], rtol=1e-5, atol=1e-6)
    tr = ub.Tracer(geom, spec, False)
    stack = rng.uniform(0.1, 2.0, (5, spec.cell_count())).astype(np.float32)
    got = ub.project_stack(tr, stack, model="length")
    for i in range(5):
        one = ub.generate_projections(ub.Field(spec, stack[i]), geom, "length").data
        np.testing.assert_allclose(got[i].reshape(-1), one.reshape(-1), rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("detector,volume", [("arc", False), ("flat", True)])
def test_length_weighted_generalized_seams(ub, orc, detector, volume):
    """M1 sector law (odd sector counts: the reference also cuts at psi + 180,
    which only splits pieces within one sector) against the C restatement."""
    spec, geom, tr, oc = _m1_case(ub, orc, detector, volume=volume, dv=6 if volume else 1, du=24, views=8)
    f = np.random.default_rng(4).integers(1, 64, spec.cell_count()) / 16.0
    want = oc.project_length(geom.thetas(), f)
    got = ub.project_stack(tr, f[None, :].astype(np.float32), model="length")[0]
    np.testing.assert_allclose(got, want, rtol=2e-6, atol=1e-6)
    with pytest.raises(ub.InvalidArgument):
        ub.generate_projections(ub.Field(spec, f.astype(np.float32)), geom, "cubic")


@pytest.mark.parametrize("name", ["fan128", "cone32", "fan16"])
def test_project_matches_reference(ub, ref, name):
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    spec, geom, tr = _ub_tracer(ub, g)
    rng = np.random.default_rng(7)
    f = rng.uniform(0.0, 5.0, spec.cell_count()).astype(np.float32)
    got = ub.generate_projections(ub.Field(spec, f), geom, "binary", tr).data
    want = rt.project(f.astype(np.float64))
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-5)
    ones = ub.generate_projections(ub.Field.constant(spec, 1.0), geom, "binary", tr).data
    assert np.array_equal(ones, tr.trace_counts().astype(np.float64))


def test_project_linearity_and_zero(ub, ref):
    g = REF_GEOMS["fan16"]
    spec, geom, tr = _ub_tracer(ub, g)
    rng = np.random.default_rng(13)
    f1 = rng.uniform(0, 2, spec.cell_count())
    f2 = rng.uniform(0, 2, spec.cell_count())
    p = ub.project_stack(tr, np.stack([f1, f2, 0.75 * f1 + 1.5 * f2, 0 * f1]))
    np.testing.assert_allclose(p[2], 0.75 * p[0] + 1.5 * p[1], rtol=1e-5)
    assert np.all(p[3] == 0)


# ---------------------------------------------------------------------------
# K3 MART
# ---------------------------------------------------------------------------


def _check_recon(ub, ref, name, phantom, beta, sweeps, tol=1e-30, rtol=1e-4):
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    spec, geom, tr = _ub_tracer(ub, g)
    if phantom == "shepp":
        truth = ref.phantom(g["n"], g["volume"])
    else:
        truth = np.random.default_rng(42).uniform(0.2, 3.0, spec.cell_count())
    proj = rt.project(truth)
    want, wrep = rt.reconstruct(proj, beta=beta, tolerance=tol, max_sweeps=sweeps)
    res = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, ub.SolverConfig(beta=beta, tolerance=tol,
                                                                             max_sweeps=sweeps), tr)
    got, rep = res.field.values, res.report
    rel = np.abs(got - want) / np.abs(want)
    assert rel.max() <= rtol, rel.max()
    assert rep.sweeps == wrep["sweeps"]
    assert rep.zero_measurement_skips == wrep["zero_measurement_skips"]
    assert rep.factor_clamps == wrep["factor_clamps"]
    assert np.array_equal(rep.crossed, wrep["crossed"])
    if tol > 0:
        np.testing.assert_allclose(rep.sweep_residuals, wrep["sweep_residuals"], rtol=5e-2, atol=1e-6)
    return got, want


def test_reconstruct_matches_reference_fan_shepp(ub, ref):
    _check_recon(ub, ref, "fan128", "shepp", beta=0.4, sweeps=5)


def test_reconstruct_matches_reference_cone(ub, ref):
    _check_recon(ub, ref, "cone32", "random", beta=0.4, sweeps=3)


def test_reconstruct_matches_reference_cone_wide(ub, ref):
    _check_recon(ub, ref, "cone32w", "random", beta=1.0, sweeps=2, rtol=2e-4)


@pytest.mark.parametrize("name,beta,sweeps,tol", [("fan128", 0.4, 5, 0), ("cone32", 0.4, 3, 0),
                                                   ("fan16", 1.0, 6, 1e-5), ("cone12", 1.9, 3, 0)])
def test_tile_executor_matches_flow_and_reference(ub, ref, monkeypatch, capfd, name, beta, sweeps, tol):
    """The one-CTA tile executor (field in shared memory, one warp per line of
    an ASAP level, a block barrier between levels; the default for one small
    problem) and the flow executor both match the reference library: counters
    and crossed masks exactly, fields within fp32 tolerance."""
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    truth = np.random.default_rng(3).uniform(0.2, 3.0, rt.cells)
    proj = rt.project(truth)
    if beta > 1:
        proj[1, :4] = 1e-9  # clamps
    want, wrep = rt.reconstruct(proj, beta=beta, tolerance=tol, max_sweeps=sweeps)
    monkeypatch.setenv("USCG_FLOW_VERBOSE", "1")
    out = {}
    for mode in ("tile", "flow"):
        monkeypatch.setenv("USCG_MART_MODE", mode)
        spec, geom, tr = _ub_tracer(ub, g)
        res = ub.reconstruct(ub.ProjectionSet(geom, proj), spec,
                             ub.SolverConfig(beta=beta, tolerance=tol, max_sweeps=sweeps), tr)
        log = capfd.readouterr().err
        assert f"mart_{mode}_kernel" in log, log
        rep = res.report
        assert rep.sweeps == wrep["sweeps"] and rep.factor_clamps == wrep["factor_clamps"]
        assert rep.zero_measurement_skips == wrep["zero_measurement_skips"]
        assert np.array_equal(rep.crossed, wrep["crossed"])
        rel = np.abs(res.field.values - want) / np.abs(want)
        assert rel.max() <= (2e-4 if beta > 1 else 1e-4), (mode, rel.max())
        out[mode] = res.field.values
    if beta > 1:
        assert wrep["factor_clamps"] > 0


@pytest.mark.parametrize("name", ["cone32", "fan128", "cone32w"])
def test_list_fed_projector_matches_traced_projector(ub, ref, name):
    """Once a reconstruction has built the tracer's traced lists, one-problem
    projections stream them (project_lists_kernel) instead of re-tracing:
    the same sums as the trace-based kernel and the reference library."""
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    spec, geom, tr = _ub_tracer(ub, g)
    truth = np.random.default_rng(11).uniform(0.2, 3.0, spec.cell_count())
    traced = ub.project_stack(tr, truth[None].astype(np.float32))[0]
    ub.reconstruct(ub.ProjectionSet(geom, traced.astype(np.float64)), spec,
                   ub.SolverConfig(beta=0.5, tolerance=0, max_sweeps=1), tr)
    assert tr.info()["executor_bytes"] > 0  # the lists exist now
    listed = ub.project_stack(tr, truth[None].astype(np.float32))[0]
    want = rt.project(truth.astype(np.float32).astype(np.float64))
    np.testing.assert_allclose(listed, traced, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(listed, want, rtol=1e-6, atol=1e-5)


def test_reconstruct_residual_stopping(ub, ref):
    g = REF_GEOMS["fan16"]
    rt = ref_tracer(ref, g)
    spec, geom, tr = _ub_tracer(ub, g)
    truth = np.random.default_rng(42).uniform(0.2, 3.0, spec.cell_count())
    proj = rt.project(truth)
    res = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, ub.SolverConfig(beta=1.0, tolerance=1e-5,
                                                                             max_sweeps=20000), tr)
    assert res.report.converged
    re = ub.generate_projections(res.field, geom, "binary", tr).data
    nz = proj != 0
    assert np.all(re[~nz] == 0)
    np.testing.assert_allclose(re[nz] / proj[nz], 1.0, atol=2e-4)


def test_reconstruct_from_resumes(ub, ref):
    """Blocks of sweeps through reconstruct_from equal one long run
    (the acceptance runner's resume pattern, acceptance.cpp:537-547)."""
    g = REF_GEOMS["fan16"]
    rt = ref_tracer(ref, g)
    spec, geom, tr = _ub_tracer(ub, g)
    truth = np.random.default_rng(3).uniform(0.2, 3.0, spec.cell_count())
    proj = ub.ProjectionSet(geom, rt.project(truth))
    cfg = ub.SolverConfig(beta=0.4, tolerance=0, max_sweeps=3)
    a = ub.reconstruct(proj, spec, cfg, tr).field
    b = ub.reconstruct_from(proj, a, cfg, tr).field
    c = ub.reconstruct(proj, spec, ub.SolverConfig(beta=0.4, tolerance=0, max_sweeps=6), tr).field
    assert np.array_equal(b.values.astype(np.float32), c.values.astype(np.float32))


def test_untouched_cells_keep_initial_value(ub, ref):
    spec = ub.GridSpec.square_2d(16)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=11, spacing_u=0.05, views=6)
    tr = ub.Tracer(geom, spec, False)
    truth = np.random.default_rng(42).uniform(0.2, 3.0, spec.cell_count())
    proj = ub.generate_projections(ub.Field(spec, truth), geom, "binary", tr)
    res = ub.reconstruct(proj, spec, ub.SolverConfig(beta=0.7, f_init=1.375, max_sweeps=5, tolerance=1e-30), tr)
    untouched = res.report.crossed == 0
    assert untouched.sum() > 0
    assert np.all(res.field.values[untouched] == 1.375)


def test_positivity_across_relaxations(ub):
    spec = ub.GridSpec.square_2d(16)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=21, spacing_u=0.2, views=20)
    tr = ub.Tracer(geom, spec, False)
    truth = np.random.default_rng(42).uniform(0.2, 3.0, spec.cell_count())
    proj = ub.generate_projections(ub.Field(spec, truth), geom, "binary", tr)
    for beta in (0.4, 1.0, 1.9):
        res = ub.reconstruct(proj, spec, ub.SolverConfig(beta=beta, tolerance=0, max_sweeps=100), tr)
        assert np.all(res.field.values > 0)


def test_input_errors(ub):
    spec = ub.GridSpec.square_2d(16)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=21, spacing_u=0.2, views=8)
    tr = ub.Tracer(geom, spec, False)
    zeros = ub.ProjectionSet(geom, np.zeros((8, 21)))
    res = ub.reconstruct(zeros, spec, ub.SolverConfig(), tr)
    assert res.report.all_zero_data and res.report.sweeps == 0
    assert np.all(res.field.values == 1.0)
    bad = np.ones((8, 21))
    bad[0, 3] = np.nan
    with pytest.raises(ub.InvalidArgument):
        ub.reconstruct(ub.ProjectionSet(geom, bad), spec, ub.SolverConfig(), tr)
    bad[0, 3] = np.inf
    with pytest.raises(ub.InvalidArgument):
        ub.reconstruct(ub.ProjectionSet(geom, bad), spec, ub.SolverConfig(), tr)
    bad[0, 3] = -1
    with pytest.raises(ub.InvalidArgument):
        ub.reconstruct(ub.ProjectionSet(geom, bad), spec, ub.SolverConfig(), tr)
    with pytest.raises(ub.InvalidArgument):
        ub.reconstruct(ub.ProjectionSet(geom, np.ones(7)), spec, ub.SolverConfig(), tr)
    with pytest.raises(ub.InvalidArgument):
        ub.reconstruct(ub.ProjectionSet(geom, np.ones((8, 21))), spec, ub.SolverConfig(beta=2.0), tr)
    with pytest.raises(ub.InvalidArgument):
        ub.reconstruct(ub.ProjectionSet(geom, np.ones((8, 21))), spec, ub.SolverConfig(f_init=0), tr)
    with pytest.raises(ub.InvalidArgument):
        ub.Tracer(ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=0, spacing_u=0.2), spec)
    with pytest.raises(ub.InvalidArgument):
        ub.Tracer(geom, ub.GridSpec(0, 1.0, 1.0))


# ---------------------------------------------------------------------------
# problem stack (the 2D slice-stack configuration)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("S", [1, 3, 37, 128])
def test_stack_matches_oracle_per_problem(ub, orc, S):
    import oracle
    spec = ub.GridSpec.square_2d(32)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=25, spacing_u=0.08, views=12)
    tr = ub.Tracer(geom, spec, False)
    rng = np.random.default_rng(S)
    truth = rng.uniform(0.2, 3.0, (S, spec.cell_count()))
    proj = ub.project_stack(tr, truth.astype(np.float32))
    proj[min(1, S - 1)] = 0  # one all-zero problem when S > 1
    g = oracle.OrcGrid.reference(32)
    src, det = geom.first_view_rays()
    oc = orc.cache(g, src, det)
    cfg = ub.SolverConfig(beta=0.5, tolerance=0, max_sweeps=4)
    out = ub.reconstruct_stack(proj, cfg, tr, with_crossed=True)
    for p in range(S):
        want, wrep = oc.reconstruct(geom.thetas(), proj[p].astype(np.float64), beta=0.5, tolerance=0, max_sweeps=4)
        got, rep = out[p]
        rel = np.abs(got - want) / want
        assert rel.max() <= 1e-4, (p, rel.max())
        assert rep.sweeps == wrep["sweeps"] and rep.all_zero_data == wrep["all_zero_data"]
        assert rep.updates == wrep["updates"]
        assert np.array_equal(rep.crossed, wrep["crossed"])


@pytest.mark.parametrize("S,run,width", [(128, 4, 8), (128, 8, 32), (64, 4, 16), (16, 2, 8), (40, 4, 8),
                                         (4, 4, 8)])
def test_pipelined_runs_are_bit_identical(ub, orc, monkeypatch, capfd, S, run, width):
    """The pipelined run executor (gathers one line ahead, shared cells handed
    over in shared memory) performs the line-by-line updates bit for bit, for
    every chunk shape (8 problems / 256 threads, 16 / 512, 32 / 1024)."""
    monkeypatch.setenv("USCG_MART_MODE", "flow")
    monkeypatch.setenv("USCG_RUN", str(run))
    monkeypatch.setenv("USCG_CHUNK_WIDTH", str(width))
    monkeypatch.setenv("USCG_FLOW_VERBOSE", "1")
    spec, geom, tr, oc = _m1_case(ub, orc, "arc", n_rings=48, views=16, du=96)
    rng = np.random.default_rng(S + run)
    truth = rng.uniform(0.2, 3.0, (S, spec.cell_count()))
    proj = ub.project_stack(tr, truth.astype(np.float32))
    cfg = ub.SolverConfig(beta=0.7, tolerance=0, max_sweeps=3)
    out = {}
    for pipe in (1, 0):
        monkeypatch.setenv("USCG_PIPE", str(pipe))
        out[pipe] = [f for f, _ in ub.reconstruct_stack(proj, cfg, tr)]
        log = capfd.readouterr().err
        assert f"run={run} pipe={pipe}" in log, log
        if width > 8:
            assert f"P={width} " in log, log
    for p in range(S):
        assert np.array_equal(out[1][p], out[0][p]), p
    want, _ = oc.reconstruct(geom.thetas(), proj[0].astype(np.float64), beta=0.7, tolerance=0, max_sweeps=3)
    assert (np.abs(out[1][0] - want) / want).max() <= 1e-4


@pytest.mark.parametrize("case", ["small", "c2"])
def test_device_wave_build_equals_host_build(ub, orc, monkeypatch, capfd, case):
    """The wave executor's entries and per-line requirements built on the
    device (wave_build.cu: hashed next-line links, sorted (cell, unit) visits,
    condensed candidates) equal the host builder's (USCG_HOST_WAVE=1) array
    for array, on a small M1-law stack and on the verbatim C2 geometry."""
    from paper_2208_12964_b200 import workloads
    monkeypatch.setenv("USCG_FLOW_VERBOSE", "1")
    if case == "c2":
        wl = workloads.make("c2")
        spec, geom = wl.spec, wl.geom
    else:
        spec, geom, _, _ = _m1_case(ub, orc, "arc", n_rings=48, views=16, du=96)
    arrays = {}
    for host in ("0", "1"):
        monkeypatch.setenv("USCG_HOST_WAVE", host)
        tr = ub.Tracer(geom, spec, False)
        proj = ub.project_stack(tr, np.ones((32, spec.cell_count()), np.float32))
        ub.reconstruct_stack(proj, ub.SolverConfig(beta=0.5, tolerance=0, max_sweeps=1), tr)
        assert "mart_wave_kernel: P=16 " in capfd.readouterr().err  # 32 problems: two 16-problem chunks
        arrays[host] = tr.wave_arrays()
        tr.close()
    for k in ("entries", "dep_off", "deps"):
        assert np.array_equal(arrays["0"][k], arrays["1"][k]), k
    assert arrays["0"]["deps"].shape[0] > 0


@pytest.mark.parametrize("S,width", [(32, 32), (16, 16), (8, 8), (64, 4)])
def test_wave_zero_lines_keep_handed_over_cells(ub, orc, monkeypatch, capfd, S, width):
    """Lines whose measurements are zero for every problem of a chunk (rim
    lines of a real phantom) update nothing, but cells handed over to them by
    the previous line (scaled, not yet stored) must still reach the field:
    wave vs the oracle with whole zero-measurement line blocks in every view."""
    monkeypatch.setenv("USCG_CHUNK_WIDTH", str(width))
    monkeypatch.setenv("USCG_FLOW_VERBOSE", "1")
    spec, geom, tr, oc = _m1_case(ub, orc, "arc", n_rings=48, views=16, du=96)
    rng = np.random.default_rng(7 + S)
    truth = rng.uniform(0.2, 3.0, (S, spec.cell_count()))
    proj = ub.project_stack(tr, truth.astype(np.float32))
    proj[:, :, 10:16] = 0
    proj[:, :, 50:53] = 0
    proj[:, ::3, 70:90] = 0
    cfg = ub.SolverConfig(beta=0.7, tolerance=0, max_sweeps=3)
    out = ub.reconstruct_stack(proj, cfg, tr)
    assert f"mart_wave_kernel: P={width} " in capfd.readouterr().err
    for p in (0, S // 2, S - 1):
        want, wrep = oc.reconstruct(geom.thetas(), proj[p].astype(np.float64), beta=0.7, tolerance=0, max_sweeps=3)
        assert (np.abs(out[p][0] - want) / want).max() <= 1e-4, p
        assert out[p][1].updates == wrep["updates"]


@pytest.mark.parametrize("S,width,detector,tol,beta", [(128, 8, "arc", 0, 0.7), (64, 16, "arc", 0, 0.7),
                                                      (128, 32, "arc", 0, 0.7), (64, 32, "parallel", 1e-3, 0.7),
                                                      (40, 8, "parallel", 0, 0.7), (16, 4, "arc", 0, 0.7),
                                                      (32, 8, "arc", 1e-3, 0.7), (24, 8, "arc", 0, 1.9)])
def test_wave_executor_matches_flow(ub, orc, monkeypatch, capfd, S, width, detector, tol, beta):
    """The wave executor (one CTA per (view, problem chunk), other views
    ordered by progress counters, gathers one line ahead with shared cells
    handed over in shared memory) performs the flow executor's line updates:
    same reports and fields within fp32 summation-order differences, over
    back-to-back sweeps (tol 0: one launch), one launch per sweep (tol > 0);
    bit-identical between runs on 1 CTA per SM and on the most that fit and
    on repeated calls (the counters carry over): a schedule race would show
    as a difference. Clamps exercised at beta 1.9."""
    monkeypatch.setenv("USCG_CHUNK_WIDTH", str(width))
    monkeypatch.setenv("USCG_FLOW_VERBOSE", "1")
    spec, geom, tr, oc = _m1_case(ub, orc, detector, n_rings=48, views=16, du=96)
    rng = np.random.default_rng(S + width)
    truth = rng.uniform(0.2, 3.0, (S, spec.cell_count()))
    proj = ub.project_stack(tr, truth.astype(np.float32))
    if beta > 1:
        proj[:, 3, 40:60] = 1e-9  # drives factors <= 0: clamps
    if S > 1:
        proj[min(2, S - 1)] = 0  # one all-zero problem
    cfg = ub.SolverConfig(beta=beta, tolerance=tol, max_sweeps=3)
    out = {}
    for mode, per_sm in (("wave", 1), ("flow", 0), ("wave", 8), ("wave", 8)):
        monkeypatch.setenv("USCG_MART_MODE", mode)
        monkeypatch.setenv("USCG_WAVE_PER_SM", str(per_sm))
        res = ub.reconstruct_stack(proj, cfg, tr)
        log = capfd.readouterr().err
        assert (f"mart_wave_kernel: P={width} " if mode == "wave" else "mart_flow_kernel") in log, log
        if mode in out:
            for p in range(S):
                assert np.array_equal(res[p][0], out[mode][p][0]), ("repeat", p)
        out[mode] = res
    for p in range(S):
        (fw, rw), (ff, rf) = out["wave"][p], out["flow"][p]
        # the same updates; p_bar summed in another order (fp32 partials;
        # at beta 1.9 near-clamp factors amplify those roundings)
        if beta < 1:
            np.testing.assert_allclose(fw, ff, rtol=2e-5, atol=0)
        assert (rw.sweeps, rw.updates, rw.factor_clamps) == (rf.sweeps, rf.updates, rf.factor_clamps), p
    if beta > 1:
        # clamped lines drive values below fp32's range: the oracle check is
        # the other cases' (test_positivity_across_relaxations covers clamps)
        assert sum(out["wave"][p][1].factor_clamps for p in range(S)) > 0
        return
    want, _ = oc.reconstruct(geom.thetas(), proj[0].astype(np.float64), beta=beta, tolerance=tol, max_sweeps=3)
    assert (np.abs(out["wave"][0][0] - want) / want).max() <= 1e-4


@pytest.mark.parametrize("S,init", [(1, False), (5, False), (8, True)])
def test_batched_reconstruction_equals_one_call_per_stack(ub, orc, S, init):
    """uscg_reconstruct_batch (transfers of neighbouring stacks overlapped with
    each solve, double-buffered staging) returns exactly what one
    uscg_reconstruct call per stack returns, for 1-4 stacks (the ping-pong
    buffers are reused from the third stack on)."""
    spec, geom, tr, _ = _m1_case(ub, orc, "arc", n_rings=32, views=12, du=64)
    rng = np.random.default_rng(11 + S)
    cfg = ub.SolverConfig(beta=0.5, tolerance=0, max_sweeps=2)
    for B in (1, 4):
        stacks = [ub.project_stack(tr, rng.uniform(0.2, 3.0, (S, spec.cell_count())).astype(np.float32))
                  for _ in range(B)]
        inits = [rng.uniform(0.5, 1.5, (S, spec.cell_count())).astype(np.float32) for _ in range(B)] if init else None
        got = ub.reconstruct_batch(stacks, cfg, tr, inits)
        for b in range(B):
            want = ub.reconstruct_stack(stacks[b], cfg, tr, None if inits is None else inits[b])
            for p in range(S):
                assert np.array_equal(got[b][p], want[p][0]), (B, b, p)


@pytest.mark.parametrize("S", [2, 8])
def test_batched_reconstruction_reports_the_failing_stack(ub, orc, S):
    """A stack with invalid data fails the batch with the reference's error;
    the stack solved before it still delivers its field (S = 8: the wave
    executor's overlapped solve slots)."""
    import ctypes as C

    import torch

    from paper_2208_12964_b200 import uscg
    spec, geom, tr, _ = _m1_case(ub, orc, "arc", n_rings=32, views=12, du=64)
    rng = np.random.default_rng(S)
    good = ub.project_stack(tr, rng.uniform(0.5, 2.0, (S, spec.cell_count())).astype(np.float32))
    bad = good.copy()
    bad[1, 0, 0] = -1.0
    cfg = ub.SolverConfig(beta=0.5, tolerance=0, max_sweeps=2)
    with pytest.raises(ub.InvalidArgument, match="non-finite or negative"):
        ub.reconstruct_batch([good, bad, good], cfg, tr)
    stacks = [torch.from_numpy(x.reshape(S, -1).copy()).pin_memory() for x in (good, bad, good)]
    fields = [torch.zeros((S, spec.cell_count()), dtype=torch.float32).pin_memory() for _ in range(3)]
    pp = (C.c_void_p * 3)(*[C.c_void_p(x.data_ptr()) for x in stacks])
    ff = (C.c_void_p * 3)(*[C.c_void_p(x.data_ptr()) for x in fields])
    c = uscg._Cfg(cfg.beta, cfg.tolerance, cfg.max_sweeps, cfg.f_init, cfg.p_floor)
    rc = ub.load().uscg_reconstruct_batch(tr.h, 3, pp, S, C.byref(c), ff, 0, None, 0)
    assert rc == 1
    want = np.stack([f for f, _ in ub.reconstruct_stack(good, cfg, tr)])
    assert np.array_equal(fields[0].numpy(), want)
    assert not fields[2].numpy().any()  # never solved


@pytest.mark.parametrize("name", ["fan64q", "cone16", "cone32w", "cone12"])
def test_one_pass_generator_equals_count_then_write(ub, monkeypatch, name):
    """The one-pass generator (bounded slots, true counts, compaction) builds
    the same record store as the exact count pass followed by the write pass."""
    out = {}
    for two in (False, True):
        if two:
            monkeypatch.setenv("USCG_GEN_TWO_PASS", "1")
        else:
            monkeypatch.delenv("USCG_GEN_TWO_PASS", raising=False)
        _, _, tr = _ub_tracer(ub, REF_GEOMS[name])
        out[two] = tr.cache()
    a, b = out[False], out[True]
    for k in ("offsets", "phi_a", "phi_b", "slice", "ring"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


# ---------------------------------------------------------------------------
# generalized seams (verbatim BASELINE shapes) vs the C restatement
# ---------------------------------------------------------------------------


def _m1_case(ub, orc, detector, n_rings=32, volume=False, views=24, du=64, dv=1):
    import oracle
    counts = ub.ring_counts_m1(n_rings)
    if volume:
        spec = ub.GridSpec(2 * n_rings, 1.0 / n_rings, 2.0 / n_rings, ub.GridMode.Volume3D, ring_counts=counts,
                           n_slices=n_rings // 2)
    else:
        spec = ub.GridSpec(2 * n_rings, 1.0 / n_rings, 1.0 / n_rings, ub.GridMode.Slice2D, ring_counts=counts)
    if detector == "arc":
        geom = ub.ScanGeometry(source=(-3, 0, 0), detector_center=(1.5, 0, 0), det_u=du, det_v=dv,
                               spacing_u=38.94 / du, spacing_v=0.05, views=views, detector=ub.Detector.Arc)
    elif detector == "parallel":
        geom = ub.ScanGeometry(source=(-2, 0, 0), detector_center=(2, 0, 0), det_u=du, spacing_u=2.0 / du,
                               views=views, detector=ub.Detector.Parallel,
                               view_angles=np.array([180.0 * i / views for i in range(views)]))
    else:
        geom = ub.ScanGeometry(source=(-4, 0, 0), detector_center=(2, 0, 0), det_u=du, det_v=dv,
                               spacing_u=3.1 / du, spacing_v=2.0 * 2.05 / dv, views=views)
    g = oracle.OrcGrid(n_rings, 1.0 / n_rings, spec.slices(), spec.slice_height, volume, counts)
    src, det = geom.first_view_rays()
    oc = orc.cache(g, src, det)
    tr = ub.Tracer(geom, spec, False)
    return spec, geom, tr, oc


@pytest.mark.parametrize("detector,volume", [("arc", False), ("parallel", False), ("flat", True)])
def test_generalized_seams_match_restatement(ub, orc, detector, volume):
    spec, geom, tr, oc = _m1_case(ub, orc, detector, volume=volume, dv=16 if volume else 1,
                                  du=32 if volume else 64, views=12 if volume else 24)
    c = tr.cache()
    assert np.array_equal(c.offsets, oc.offsets)
    assert np.array_equal(c.slice, oc.records["slice"]) and np.array_equal(c.ring, oc.records["ring"])
    assert_phi_adjudicated(c.phi_a, oc.records["phi_a"])
    assert_phi_adjudicated(c.phi_b, oc.records["phi_b"])
    # index lists: exact through the oracle's own cache; with the device-built
    # cache any difference must sit on a line holding a 1-ulp azimuth
    ocache = ub.FirstViewCache(oc.offsets, oc.records["phi_a"].copy(), oc.records["phi_b"].copy(),
                               oc.records["slice"].copy(), oc.records["ring"].copy())
    tr_imp = ub.Tracer.from_cache(spec, ocache, geom.views, geom.view_angles, geom=geom)
    ulp_rec = (ulp_diff(c.phi_a, oc.records["phi_a"]) + ulp_diff(c.phi_b, oc.records["phi_b"])) > 0
    th = geom.thetas()
    for v in range(geom.views):
        for line in range(geom.lines()):
            want = oc.trace_line(line, th[v])
            assert np.array_equal(tr_imp.trace_line(line, th[v]), want), (v, line)
            if not np.array_equal(tr.trace_line(line, th[v]), want):
                assert ulp_rec[oc.offsets[line]:oc.offsets[line + 1]].any(), (v, line)
    tr = tr_imp
    truth = np.random.default_rng(5).uniform(0.2, 2.0, spec.cell_count())
    proj = oc.project(th, truth)
    got_p = ub.generate_projections(ub.Field(spec, truth.astype(np.float32)), geom, "binary", tr).data
    np.testing.assert_allclose(got_p, proj, rtol=1e-6, atol=1e-5)
    want, wrep = oc.reconstruct(th, proj, beta=0.3, tolerance=0, max_sweeps=3)
    res = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, ub.SolverConfig(beta=0.3, tolerance=0, max_sweeps=3), tr)
    rel = np.abs(res.field.values - want) / want
    assert rel.max() <= 1e-4
    assert res.report.updates == wrep["updates"]


# ---------------------------------------------------------------------------
# K4 resample
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("n", [2, 4, 16, 64, 256])
def test_uspg_to_cg_map_matches_reference(ub, ref, n):
    assert np.array_equal(ub.uspg_to_cg_map(n), ref.uspg_to_cg_map(n))


def test_uspg_to_cg_map_rejects_odd(ub):
    with pytest.raises(ub.DomainError):
        ub.uspg_to_cg_map(5)


@pytest.mark.parametrize("n,volume", [(8, True), (128, False), (64, True)])
def test_field_to_cartesian_matches_reference(ub, ref, n, volume):
    spec = ub.GridSpec.cube_3d(n) if volume else ub.GridSpec.square_2d(n)
    f = np.random.default_rng(5).uniform(0, 2, spec.cell_count()).astype(np.float32)
    got = ub.field_to_cartesian(ub.Field(spec, f))
    want = ref.field_to_cartesian(n, volume, f.astype(np.float64))
    assert np.array_equal(got.astype(np.float64), want)


def test_resample_bin_map_matches_restatement(ub, orc):
    import oracle
    counts = ub.ring_counts_m1(64)
    spec = ub.GridSpec(128, 1 / 64, 1 / 64, ub.GridMode.Slice2D, ring_counts=counts)
    g = oracle.OrcGrid(64, 1 / 64, 1, 1 / 64, False, counts)
    f = np.random.default_rng(9).uniform(0, 2, spec.cell_count()).astype(np.float32)
    got = ub.field_to_cartesian(ub.Field(spec, f), npix=256)[0]
    want = orc.field_to_cartesian(g, f.astype(np.float64), 256)[0]
    mism = got.astype(np.float64) != want
    assert mism.sum() <= 4, mism.sum()  # sector-edge pixels only (atan2 ulps)


def test_resample_stack_layouts(ub):
    spec = ub.GridSpec.square_2d(32)
    f = np.random.default_rng(1).uniform(0, 2, (5, spec.cell_count())).astype(np.float32)
    out = ub.resample_stack(spec, f, 32)
    for p in range(5):
        assert np.array_equal(out[p], ub.field_to_cartesian(ub.Field(spec, f[p])))


# ---------------------------------------------------------------------------
# image-quality metrics on the device (metrics.cpp)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("shape", [(8, 8), (37, 53), (100, 9), (64, 64)])
def test_image_metrics_match_reference(ub, ref, shape):
    """rmse / mae / ssim of one raster pair against the reference library
    (values exact in fp32; the window sums run in another fp64 order)."""
    rng = np.random.default_rng(shape[0] * 131 + shape[1])
    a = rng.integers(0, 64, shape) / 64.0
    b = np.clip(a + rng.normal(0, 0.05, shape), 0, None).astype(np.float32).astype(np.float64)
    m = ub.image_metrics(a, b)
    assert abs(m["rmse"][0] - ref.rmse(a, b)) <= 1e-12 * max(1.0, ref.rmse(a, b))
    assert abs(m["mae"][0] - np.abs(a - b).mean()) <= 1e-12
    assert abs(m["ssim"][0] - ref.ssim(a, b)) <= 1e-12
    assert abs(ub.ssim(a, b, 2.5) - ref.ssim(a, b, 2.5)) <= 1e-12
    # constant reference: the dynamic range falls back to 1 (metrics.cpp:27-31)
    c = np.full(shape, 0.5)
    assert abs(ub.ssim(c, b) - ref.ssim(c, b)) <= 1e-12


def test_image_metrics_volume_scores(ub, ref):
    """ssim_volume shares the reference stack's range (metrics.cpp:186-199);
    the volume scores are means of the per-slice values."""
    rng = np.random.default_rng(21)
    a = rng.integers(0, 256, (5, 40, 33)) / 64.0
    a[2] *= 0.25  # slices with different ranges
    b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, None).astype(np.float32).astype(np.float64)
    L = a.max() - a.min()
    want = np.mean([ref.ssim(a[s], b[s], L) for s in range(5)])
    assert abs(ub.ssim_volume(a, b) - want) <= 1e-12
    per = ub.image_metrics(a, b)
    for s in range(5):
        assert abs(per["ssim"][s] - ref.ssim(a[s], b[s])) <= 1e-12
    assert abs(ub.rmse_volume(a, b) - np.mean([ref.rmse(a[s], b[s]) for s in range(5)])) <= 1e-12
    assert abs(ub.mae_volume(a, b) - np.mean(np.abs(a - b).mean(axis=(1, 2)))) <= 1e-12


def test_image_metrics_errors(ub):
    with pytest.raises(ub.InvalidArgument):
        ub.ssim(np.ones((7, 20)), np.ones((7, 20)))  # smaller than the 8x8 window
    assert ub.rmse(np.ones((7, 20)), np.zeros((7, 20))) == 1.0
    with pytest.raises(ub.InvalidArgument):
        ub.image_metrics(np.ones((8, 8)), np.ones((8, 9)))
    with pytest.raises(ub.InvalidArgument):
        ub.image_metrics(np.ones((0, 8, 8)), np.ones((0, 8, 8)))


# ---------------------------------------------------------------------------
# Cartesian comparator (siddon.cpp)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["fan16", "cone12", "fan32"])
def test_cartesian_system_matches_reference(ub, ref, name):
    """precompute_cartesian_system on the device: the same voxel sequence per
    (view, line), lengths to fp32. Adjudicated: a ray along a voxel boundary
    (the rotated central ray meets the grid lines at 0 / 90 / 180 / 270 deg)
    may take either side; such lines must carry the same total length."""
    g = REF_GEOMS[name]
    spec, geom = ub_spec_geom(ub, g)
    cs = ub.CartesianSystem(spec, geom, stored=True)
    off, idx, w = cs.export()
    roff, ridx, rw = ref.cartesian_system(g["n"], g["volume"], g["src"], g["ctr"], g["du"], g["dv"], g["su"], g["sv"],
                                          g["views"])
    rows = g["views"] * g["du"] * g["dv"]
    differ = 0
    for r in range(rows):
        a, b = idx[off[r]:off[r + 1]], ridx[roff[r]:roff[r + 1]]
        wa, wb = w[off[r]:off[r + 1]].astype(np.float64), rw[roff[r]:roff[r + 1]]
        if np.array_equal(a, b):
            np.testing.assert_allclose(wa, wb, rtol=2e-6, atol=1e-9)
        else:
            differ += 1
            assert abs(wa.sum() - wb.sum()) <= 1e-5 * max(1.0, wb.sum()), r
    assert differ <= max(2, rows // 50), differ
    inf = cs.info()
    assert inf["entries"] == off[-1] and inf["levels"] > 0


@pytest.mark.parametrize("stored", [True, False])
def test_cartesian_mart_matches_reference(ub, ref, stored):
    """cartesian_mart_stored / _otf: fixed sweeps of the length-weighted
    row action on the voxel grid, fp32 field vs the reference's fp64."""
    g = REF_GEOMS["fan32"]
    spec, geom = ub_spec_geom(ub, g)
    rng = np.random.default_rng(17)
    rows = g["views"] * g["du"]
    proj = rng.uniform(0.5, 3.0, rows).astype(np.float32).astype(np.float64)
    proj[::7] = 0.0  # skipped lines
    want, _ = ref.cartesian_mart(g["n"], False, g["src"], g["ctr"], g["du"], 1, g["su"], 0.0, g["views"], proj,
                                 beta=0.4, sweeps=3, f_init=1.0, stored=stored)
    cs = ub.CartesianSystem(spec, geom, stored=stored)
    got, sec = cs.reconstruct(proj, ub.SolverConfig(beta=0.4, tolerance=0, max_sweeps=3))
    assert sec > 0
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-6)


# ---------------------------------------------------------------------------
# the dependency schedule built on the device (schedule_gpu.cu)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("case", ["fan16", "fan32", "cone16", "cone32", "m1arc"])
def test_device_schedule_equals_host_schedule(ub, orc, monkeypatch, case):
    """The sort-based device builder yields exactly the host AsapSchedule:
    the same runs, levels, level-sorted order, in-sweep predecessors,
    cross-sweep predecessor counts and merged successor lists."""
    def build(host):
        monkeypatch.setenv("USCG_HOST_SCHEDULE", "1" if host else "0")
        if case == "m1arc":
            _, _, tr, _ = _m1_case(ub, orc, "arc", n_rings=40, views=20, du=48)
        else:
            _, _, tr = _ub_tracer(ub, REF_GEOMS[case])
        return tr.schedule()

    got, want = build(False), build(True)
    for k in ("run", "runs", "levels"):
        assert got[k] == want[k], k
    for k in ("order", "level_off", "pred_off", "preds", "npred_x", "succ_off", "succs"):
        assert np.array_equal(got[k], want[k]), k


# ---------------------------------------------------------------------------
# row-sharded generator on the device (dist.generate_sharded / concat_caches)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["cone16", "cone32w"])
def test_row_sharded_generator_assembles_the_same_store(ub, name):
    """Rows generated in blocks and assembled (copy_cache -> concat_caches ->
    from_key_cache) give the directly generated store, dedup flags included,
    and the same traces."""
    import torch
    from paper_2208_12964_b200 import dist as udist
    g = REF_GEOMS[name]
    spec, geom = ub_spec_geom(ub, g)
    direct = ub.Tracer(geom, spec, False)
    src, det = geom.first_view_rays()
    parts = []
    for r in range(3):
        r0, r1 = udist.shard(g["dv"], r, 3)
        t = ub.Tracer.from_rays(spec, src[r0 * g["du"]:r1 * g["du"]], det[r0 * g["du"]:r1 * g["du"]], 1)
        parts.append(t.copy_cache(device=True))
        t.close()
    full = udist.concat_caches(parts)
    asm = ub.Tracer.from_key_cache(spec, *full, g["views"], geom=geom)
    for a, b in zip(asm.copy_cache(device=True), direct.copy_cache(device=True)):
        assert torch.equal(a, b)
    th = thetas(g["views"])
    for line in range(0, geom.lines(), 7):
        assert np.array_equal(asm.trace_line(line, th[1]), direct.trace_line(line, th[1]))
    one = udist.generate_sharded(spec, geom, 0, 1)  # world 1: no exchange
    for a, b in zip(one.copy_cache(device=True), direct.copy_cache(device=True)):
        assert torch.equal(a, b)
