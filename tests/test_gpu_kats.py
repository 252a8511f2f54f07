"""The reference's own known-answer and behaviour tests, through the device
path: solver arithmetic (proj/tests/test_solver.cpp),
cache facts (proj/tests/test_tracer.cpp, acceptance.cpp) and forward-model
facts (proj/tests/test_phantom.cpp). Where the reference's check depends on
fp64 (bitwise fixed point, 1e-9 convergence) the inputs are chosen so that it
holds exactly in the device's fp32 field too, or the tolerance says why."""
import numpy as np
import pytest

from refgeoms import REF_GEOMS, thetas, ub_spec_geom

pytestmark = pytest.mark.gpu


def _one_line(ub):
    """square_2d(8), one view, one detector line through the grid."""
    spec = ub.GridSpec.square_2d(8)
    geom = ub.ScanGeometry(source=(-8, 0.1, 0), detector_center=(8, 0.1, 0), det_u=1, spacing_u=0.1, views=1)
    tr = ub.Tracer(geom, spec, False)
    k = int(tr.trace_counts()[0, 0])
    assert k > 0
    return spec, geom, tr, k


@pytest.mark.parametrize("beta,ratio,want", [(1.0, 1.5, 3.0), (0.4, 1.5, 2.4), (1.0, 0.5, 1.0)])
def test_row_update_arithmetic(ub, beta, ratio, want):
    """mart_update_line (solver.cpp:33-51; test_solver.cpp 'row update
    arithmetic'): f *= 1 - beta (1 - m / p_bar) on the active cells only."""
    spec, geom, tr, k = _one_line(ub)
    m = ratio * 2.0 * k  # p_bar = 2 k at f = 2
    res = ub.reconstruct(ub.ProjectionSet(geom, np.array([[m]])), spec,
                         ub.SolverConfig(beta=beta, f_init=2.0, tolerance=0, max_sweeps=1), tr)
    active = tr.trace_line(0, 0.0)
    f = res.field.values
    assert np.all(f[active] == np.float32(want))
    rest = np.ones(f.size, bool)
    rest[active] = False
    assert np.all(f[rest] == 2.0)  # inactive cells untouched
    assert res.report.updates == k and res.report.factor_clamps == 0


def test_row_update_clamp_and_skip(ub):
    """A non-positive factor is clamped to p_floor (solver.cpp:42-45, beta
    1.9 with a near-zero measurement), and a zero measurement skips the line."""
    spec, geom, tr, k = _one_line(ub)
    m = 1e-9
    res = ub.reconstruct(ub.ProjectionSet(geom, np.array([[m]])), spec,
                         ub.SolverConfig(beta=1.9, f_init=2.0, tolerance=0, max_sweeps=1), tr)
    p_floor = 1e-12 * m  # auto_p_floor: 1e-12 x the mean positive measurement
    active = tr.trace_line(0, 0.0)
    np.testing.assert_allclose(res.field.values[active], 2.0 * p_floor, rtol=1e-6)
    assert res.report.factor_clamps == 1
    # all-zero data: the initial field comes back, nothing is updated
    res0 = ub.reconstruct(ub.ProjectionSet(geom, np.array([[0.0]])), spec,
                          ub.SolverConfig(beta=1.0, f_init=2.0, tolerance=0, max_sweeps=3), tr)
    assert res0.report.all_zero_data and np.all(res0.field.values == 2.0)


def test_truth_is_a_fixed_point_bitwise(ub):
    """test_solver.cpp 'initializing at the truth is a fixed point, bitwise':
    with dyadic field values every sum is exact in fp32 and fp64 alike, so
    every ratio is exactly 1 and nothing moves."""
    spec = ub.GridSpec.square_2d(16)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=21, spacing_u=0.2, views=20)
    tr = ub.Tracer(geom, spec, False)
    truth = (np.random.default_rng(42).integers(4, 48, spec.cell_count()) / 16.0).astype(np.float32)
    proj = ub.generate_projections(ub.Field(spec, truth), geom, "binary", tr)
    res = ub.reconstruct_from(proj, ub.Field(spec, truth), ub.SolverConfig(beta=1.0, max_sweeps=1, tolerance=1e-30),
                              tr)
    assert list(res.report.sweep_residuals) == [0.0]
    assert np.array_equal(res.field.values, truth)


def test_self_consistency_closure(ub):
    """test_solver.cpp 'self-consistency': a converged reconstruction
    reproduces its measurements line by line (fp32 field: tolerance 1e-6 on
    the residual, 1e-4 on the closure instead of 1e-9 / 1e-6)."""
    spec = ub.GridSpec.square_2d(16)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=21, spacing_u=0.2, views=20)
    tr = ub.Tracer(geom, spec, False)
    truth = np.random.default_rng(42).uniform(0.5, 2.0, spec.cell_count()).astype(np.float32)
    proj = ub.generate_projections(ub.Field(spec, truth), geom, "binary", tr)
    res = ub.reconstruct(proj, spec, ub.SolverConfig(beta=1.0, tolerance=1e-6, max_sweeps=20000), tr)
    assert res.report.converged
    re = ub.generate_projections(ub.Field(spec, res.field.values), geom, "binary", tr).data.reshape(-1)
    d = proj.data.reshape(-1)
    assert np.all(re[d == 0] == 0)
    assert np.abs(re[d != 0] / d[d != 0] - 1.0).max() <= 1e-4


def test_sweep_residuals_nonincreasing(ub):
    """test_solver.cpp 'reference 2d scan has nonincreasing sweep residuals':
    square_2d(128), 101 detectors, 50 views, beta 0.4, 15 sweeps (a seeded
    ellipse phantom stands in for Shepp-Logan)."""
    from paper_2208_12964_b200 import workloads
    spec = ub.GridSpec.square_2d(128)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=101, spacing_u=0.05, views=50)
    tr = ub.Tracer(geom, spec, True)
    wl = workloads.make("c1-ref")
    wl.spec = spec
    truth = workloads.phantom_fields(wl, 1)[0].astype(np.float32)
    proj = ub.generate_projections(ub.Field(spec, truth), geom, "binary", tr)
    res = ub.reconstruct(proj, spec, ub.SolverConfig(beta=0.4, tolerance=1e-30, max_sweeps=15), tr)
    r = res.report.sweep_residuals
    assert len(r) == 15
    for i in range(3, 15):
        assert r[i] <= r[i - 1], (i, r[i], r[i - 1])


def test_cache_facts(ub):
    """test_tracer.cpp / acceptance.cpp: the central ray's chords have
    azimuths exactly 0 or 180; the cache does not depend on the view count;
    256^2 with 101 detectors is 247,200 bytes in the reference's layout
    (24 B per record + 4 B per offset)."""
    spec = ub.GridSpec.square_2d(256)
    c = []
    for views in (10, 50):
        geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=101, spacing_u=0.05, views=views)
        c.append(ub.Tracer(geom, spec, False).cache())
    a, b = c
    for x, y in zip((a.offsets, a.phi_a, a.phi_b, a.slice, a.ring), (b.offsets, b.phi_a, b.phi_b, b.slice, b.ring)):
        assert np.array_equal(x, y)
    assert 24 * a.phi_a.size + 4 * a.offsets.size == 247200
    mid = 50  # the central detector line
    pa = a.phi_a[a.offsets[mid]:a.offsets[mid + 1]]
    pb = a.phi_b[a.offsets[mid]:a.offsets[mid + 1]]
    assert np.all(np.isin(pa, [0.0, 180.0])) and np.all(np.isin(pb, [0.0, 180.0]))


def test_rim_missing_lines_are_empty_and_project_to_zero(ub):
    """test_tracer.cpp 'rim miss empty' and test_phantom.cpp: a line that
    misses the disc traces to nothing and projects to 0; a unit field
    projects to each line's active count; views differ."""
    g = REF_GEOMS["fan16"]
    spec, _ = ub_spec_geom(ub, g)
    geom = ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=31, spacing_u=1.0, views=8)
    tr = ub.Tracer(geom, spec, False)
    counts = tr.trace_counts()
    assert counts[0, 0] == 0 and tr.trace_line(0, 0.0).size == 0  # far off-axis: misses
    ones = ub.generate_projections(ub.Field(spec, np.ones(spec.cell_count(), np.float32)), geom, "binary", tr)
    assert np.array_equal(ones.data.reshape(counts.shape), counts.astype(np.float64))
    zero = ub.generate_projections(ub.Field(spec, np.zeros(spec.cell_count(), np.float32)), geom, "binary", tr)
    assert np.all(zero.data == 0)
    rnd = np.random.default_rng(3).uniform(0.1, 1.0, spec.cell_count()).astype(np.float32)
    p = ub.generate_projections(ub.Field(spec, rnd), geom, "binary", tr).data.reshape(8, -1)
    assert not np.array_equal(p[0], p[1])
