"""The CPU oracle is pinned before it is trusted (CPU only, no GPU).

1. Against the committed golden fixtures produced by the unmodified reference
   library (tests/golden/make_golden.py): caches, traces, projections,
   reconstructions, maps and worked-example KATs, all bit-exact.
2. Against the reference library itself, run here (oracle/_ref), on the
   reference's own test geometries (proj/tests/test_tracer.cpp:15-36,
   acceptance.cpp:33-56): bit-exact caches, every (view, line) trace,
   projections, fp64 reconstructions, residuals, crossed masks, the
   permutation map, field_to_cartesian, RMSE and SSIM.
3. Generalized seams (ring-count table, decoupled slices, arc / parallel rays,
   view lists) are checked for the invariants the reference tests assert:
   periodicity, dedup, closure, positivity.
"""
import json
import os

import numpy as np
import pytest

import oracle
from refgeoms import REF_GEOMS, ref_tracer, thetas

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _orc_cache(orc, g):
    grid = oracle.OrcGrid.reference(g["n"], g["volume"])
    s, d = orc.rays_flat(g["src"], g["ctr"], g["du"], g["dv"], g["su"], g["sv"])
    return grid, orc.cache(grid, s, d)


# ---------------------------------------------------------------------------
# 1. golden fixtures (reference outputs committed to the repo)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["fan32", "fan16", "cone16", "cone12"])
def test_oracle_matches_golden_fixtures(orc, name):
    g = REF_GEOMS[name]
    grid, oc = _orc_cache(orc, g)
    gc = np.load(os.path.join(GOLDEN, f"cache_{name}.npz"))
    assert np.array_equal(oc.offsets, gc["offsets"])
    assert np.array_equal(oc.records["phi_a"].view(np.uint64), gc["phi_a"].view(np.uint64))
    assert np.array_equal(oc.records["phi_b"].view(np.uint64), gc["phi_b"].view(np.uint64))
    assert np.array_equal(oc.records["slice"], gc["slice"])
    assert np.array_equal(oc.records["ring"], gc["ring"])
    # FirstViewCache::byte_size (tracer.hpp:31-33): 24 B records + u32 offsets
    assert int(gc["bytes"][0]) == 24 * oc.records.size + 4 * oc.offsets.size
    gt = np.load(os.path.join(GOLDEN, f"trace_{name}.npz"))
    th = thetas(g["views"])
    for k, (v, line) in enumerate(gt["picks"]):
        want = gt["idx"][gt["pos"][k]:gt["pos"][k + 1]]
        assert np.array_equal(oc.trace_line(int(line), th[v]), want)
    gp = np.load(os.path.join(GOLDEN, f"proj_{name}.npz"))
    assert np.array_equal(oc.project(th, gp["field"]), gp["proj"])
    gr = np.load(os.path.join(GOLDEN, f"recon_{name}.npz"))
    f, rep = oc.reconstruct(th, gp["proj"], beta=0.4, tolerance=1e-30, max_sweeps=3)
    assert np.array_equal(f, gr["field"])
    assert np.array_equal(rep["sweep_residuals"], gr["residuals"])
    assert np.array_equal(rep["crossed"], gr["crossed"])
    assert [rep["sweeps"], rep["zero_measurement_skips"], rep["factor_clamps"]] == list(gr["counters"])


@pytest.mark.parametrize("n", [2, 4, 16, 64])
def test_oracle_map_matches_golden(orc, n):
    assert np.array_equal(orc.uspg_to_cg_map(n), np.load(os.path.join(GOLDEN, f"map_{n}.npz"))["map"])


def test_oracle_trace_chord_kats(orc):
    """proj/tests/test_tracer.cpp:60-98 (via the golden KAT file)."""
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    import ctypes as C
    for case in kat["trace_chord"]:
        grid = oracle.OrcGrid.reference(case["n"], case["volume"])
        rec = np.zeros(1, oracle.REC_DTYPE)
        rec["phi_a"], rec["phi_b"], rec["slice"], rec["ring"] = case["rec"]
        out = np.zeros(64, np.uint32)
        k = orc.L.orc_trace_chord(C.byref(grid._c), rec.ctypes.data, case["theta"],
                                  out.ctypes.data_as(C.POINTER(C.c_uint32)), out.size)
        assert out[:k].tolist() == case["cells"]
    expected = {(95.0, 40.0): [5, 6, 7], (350.0, 10.0): [15, 4], (10.0, 190.0): [4, 5, 6, 7, 8, 9, 10],
                (45.0, 45.0): [5]}
    for case in kat["trace_chord"]:
        key = tuple(case["rec"][:2])
        if key in expected and not case["volume"] and case["theta"] == 0.0:
            assert case["cells"] == expected[key]


# ---------------------------------------------------------------------------
# 2. the reference library run here
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["fan32", "fan64q", "fan16", "cone16", "cone32", "cone12"])
def test_oracle_bit_exact_vs_reference_library(ref, orc, name):
    g = REF_GEOMS[name]
    rt = ref_tracer(ref, g)
    off, pa, pb, sl, rg = rt.cache()
    grid, oc = _orc_cache(orc, g)
    assert np.array_equal(off, oc.offsets)
    assert np.array_equal(pa.view(np.uint64), oc.records["phi_a"].view(np.uint64))
    assert np.array_equal(pb.view(np.uint64), oc.records["phi_b"].view(np.uint64))
    assert np.array_equal(sl, oc.records["slice"]) and np.array_equal(rg, oc.records["ring"])
    th = thetas(g["views"])
    for v in range(g["views"]):
        for line in range(g["du"] * g["dv"]):
            assert np.array_equal(rt.trace_line(line, th[v]), oc.trace_line(line, th[v]))
    f = np.random.default_rng(1).uniform(0.2, 3, grid.cell_count())
    p = rt.project(f)
    assert np.array_equal(p, oc.project(th, f))
    a, ra = rt.reconstruct(p, beta=0.4, tolerance=1e-30, max_sweeps=4)
    b, rb = oc.reconstruct(th, p, beta=0.4, tolerance=1e-30, max_sweeps=4)
    assert np.array_equal(a, b)
    assert np.array_equal(ra["sweep_residuals"], rb["sweep_residuals"])
    assert np.array_equal(ra["crossed"], rb["crossed"])
    assert ra["zero_measurement_skips"] == rb["zero_measurement_skips"]


def test_quarter_symmetric_reference_cache_equals_direct(ref, orc):
    """proj/tests/test_tracer.cpp:142-156: the mirrored build is bit-identical,
    which is why the oracle (and the device generator) build directly."""
    for name in ("fan64q", "cone32"):
        g = REF_GEOMS[name]
        a = ref_tracer(ref, g, quarter=True).cache()
        grid, oc = _orc_cache(orc, g)
        assert np.array_equal(a[0], oc.offsets)
        assert np.array_equal(a[1].view(np.uint64), oc.records["phi_a"].view(np.uint64))


def test_oracle_reconstruct_from_and_errors(ref, orc):
    g = REF_GEOMS["fan16"]
    rt = ref_tracer(ref, g)
    grid, oc = _orc_cache(orc, g)
    th = thetas(g["views"])
    f = np.random.default_rng(2).uniform(0.2, 3, grid.cell_count())
    p = rt.project(f)
    init = np.random.default_rng(3).uniform(0.5, 2, grid.cell_count())
    a, _ = rt.reconstruct(p, init=init, beta=1.0, tolerance=0, max_sweeps=3)
    b, _ = oc.reconstruct(th, p, init=init, beta=1.0, tolerance=0, max_sweeps=3)
    assert np.array_equal(a, b)
    # fixed point: initializing at the truth leaves it unchanged (test_solver.cpp:131-141)
    c, rep = oc.reconstruct(th, p, init=f, beta=1.0, tolerance=1e-30, max_sweeps=1)
    assert rep["sweep_residuals"][0] == 0.0 and np.array_equal(c, f)
    # all-zero data, invalid inputs (test_solver.cpp:197-241)
    z, rz = oc.reconstruct(th, np.zeros_like(p), beta=0.4)
    assert rz["all_zero_data"] and rz["sweeps"] == 0 and np.all(z == 1.0)
    bad = p.copy()
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        oc.reconstruct(th, bad)
    with pytest.raises(ValueError):
        rt.reconstruct(bad)
    with pytest.raises(ValueError):
        oc.reconstruct(th, p, beta=2.0)


@pytest.mark.parametrize("n,volume", [(8, True), (64, False), (16, True)])
def test_oracle_field_to_cartesian_vs_reference(ref, orc, n, volume):
    grid = oracle.OrcGrid.reference(n, volume)
    f = np.random.default_rng(5).uniform(0, 2, grid.cell_count())
    assert np.array_equal(orc.field_to_cartesian(grid, f, n), ref.field_to_cartesian(n, volume, f))


def test_oracle_metrics_vs_reference(ref, orc):
    rng = np.random.default_rng(3)
    a = rng.uniform(0, 1, (64, 64))
    b = a + rng.normal(0, 0.05, a.shape)
    assert orc.rmse(a, b) == ref.rmse(a, b)
    assert orc.ssim(a, b) == ref.ssim(a, b)
    assert orc.ssim(a, a) == 1.0


@pytest.mark.parametrize("n,volume", [(8, True), (64, False), (16, True), (2, False)])
def test_oracle_cartesian_to_field_vs_reference(ref, orc, n, volume):
    """cartesian_to_field (phantom.cpp:165-180), and its round trip with field_to_cartesian"""
    grid = oracle.OrcGrid.reference(n, volume)
    imgs = np.random.default_rng(6).uniform(0, 2, (grid.n_slices, n, n))
    got = orc.cartesian_to_field(grid, imgs, n)
    assert np.array_equal(got, ref.cartesian_to_field(n, volume, imgs))
    assert np.array_equal(orc.field_to_cartesian(grid, got, n), imgs)


def test_oracle_cartesian_to_field_errors(ref, orc):
    grid = oracle.OrcGrid.reference(8, False)
    with pytest.raises(ValueError):
        orc.cartesian_to_field(grid, np.zeros((1, 6, 6)), 6)
    with pytest.raises(ValueError, match="slice shape"):
        ref.cartesian_to_field(8, False, np.zeros((1, 6, 6)), img_n=6)


def test_oracle_sharpness_and_profile_vs_reference(ref, orc):
    rng = np.random.default_rng(8)
    for shape in [(64, 64), (2, 2), (3, 17), (31, 2)]:
        a = rng.uniform(0, 1, shape)
        assert orc.sharpness(a) == ref.sharpness(a)
    flat = np.full((5, 5), 2.5)
    assert ref.sharpness(flat) == 0.0 == orc.sharpness(flat)
    board = np.indices((16, 16)).sum(axis=0) % 2 * 1.0
    blurred = (board + np.roll(board, 1, 0) + np.roll(board, 1, 1) + np.roll(board, (1, 1), (0, 1))) / 4
    assert orc.sharpness(board) > orc.sharpness(blurred)  # proj/tests/test_metrics.cpp:132-147
    with pytest.raises(ValueError, match="2x2"):
        ref.sharpness(np.zeros((1, 5)))
    assert np.isnan(orc.sharpness(np.zeros((1, 5))))
    ramp = np.arange(12.0).reshape(3, 4)
    assert np.array_equal(ref.intensity_profile(ramp, 2), ramp[2])
    with pytest.raises(ValueError, match="out of range"):
        ref.intensity_profile(ramp, 3)


def test_oracle_images_match_golden(orc):
    z = np.load(os.path.join(GOLDEN, "images.npz"))
    g2, g3 = oracle.OrcGrid.reference(16, False), oracle.OrcGrid.reference(8, True)
    assert np.array_equal(orc.cartesian_to_field(g2, z["im2"], 16), z["field2"])
    assert np.array_equal(orc.cartesian_to_field(g3, z["im3"], 8), z["field3"])
    off = 0
    for (r, c), want in zip(z["sharp_shapes"], z["sharpness"]):
        img = z["sharp_pixels"][off:off + r * c].reshape(r, c)
        off += r * c
        assert orc.sharpness(img) == want


def test_glibc_atan2_is_not_always_correctly_rounded(orc):
    """Adjudication evidence for the device generator's azimuths: glibc
    2.39's atan2 differs from the correctly rounded value (mpmath, 200 bits)
    on a small fraction of inputs, so a correctly rounded device atan2 can
    disagree with the reference by 1 ulp there (test_gpu_parity.py)."""
    mp = pytest.importorskip("mpmath")
    mp.mp.prec = 200
    rng = np.random.default_rng(2208)
    n = 4000
    r = np.sqrt(rng.uniform(0, 1, n))
    ang = rng.uniform(-np.pi, np.pi, n)
    x, y = r * np.cos(ang), r * np.sin(ang)
    host = orc.math(x, y)
    bad = sum(float(mp.atan2(mp.mpf(y[i]), mp.mpf(x[i]))) != host[i, 0] for i in range(n))
    assert 0 <= bad <= 0.005 * n


# ---------------------------------------------------------------------------
# 3. generalized seams
# ---------------------------------------------------------------------------


def test_m1_sector_law_sizes(orc):
    """sum of round(2 pi (i + 0.5)) over rings."""
    assert int(orc.ring_counts_m1(64).sum()) == 12868
    assert int(orc.ring_counts_m1(256).sum()) == 205888
    assert int(orc.ring_counts_m1(512).sum()) == 823550
    assert int(orc.ring_counts_m1(128).sum()) * 128 == 6588416


@pytest.mark.parametrize("kind", ["arc", "parallel", "cone"])
def test_generalized_restatement_invariants(orc, kind):
    counts = orc.ring_counts_m1(24)
    if kind == "cone":
        grid = oracle.OrcGrid(24, 1 / 24, 12, 2 / 24, True, counts)
        s, d = orc.rays_flat((-4, 0, 0), (2, 0, 0), 16, 12, 0.2, 0.15)
    elif kind == "arc":
        grid = oracle.OrcGrid(24, 1 / 24, 1, 1 / 24, False, counts)
        s, d = orc.rays_arc((-3, 0, 0), (1.5, 0, 0), 48, 38.94 / 48)
    else:
        grid = oracle.OrcGrid(24, 1 / 24, 1, 1 / 24, False, counts)
        s, d = orc.rays_parallel(48, 2 / 48, 2.0)
    oc = orc.cache(grid, s, d)
    th = np.array([7.5 * i for i in range(24)])
    for line in range(0, s.shape[0], 5):
        a = oc.trace_line(line, 0.0)
        assert np.array_equal(a, oc.trace_line(line, 360.0))  # full turn is the identity
        assert len(np.unique(a)) == a.size                    # deduplicated
        assert np.all(a < grid.cell_count())
    truth = np.random.default_rng(4).uniform(0.2, 2, grid.cell_count())
    p = oc.project(th, truth)
    f, rep = oc.reconstruct(th, p, beta=1.0, tolerance=1e-9, max_sweeps=5000)
    assert np.all(f > 0)
    re = oc.project(th, f)
    nz = p != 0
    np.testing.assert_allclose(re[nz] / p[nz], 1.0, atol=1e-5)


# ---------------------------------------------------------------------------
# length-weighted coefficients (phantom.cpp:213-269) and MART over stored
# (voxel, length) lists (siddon.cpp:141-154, 185-209)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["fan32", "fan16", "cone16", "cone12"])
def test_length_projector_and_lists_pinned_to_reference(orc, ref, name):
    """The restated LengthWeighted projector equals the reference library's bit
    for bit; the (voxel, chord length) lists are the same pieces with a cell's
    pieces merged: they reproduce the projections of random fields, list each
    cell of a line once, and a unit field gives the line's path length."""
    g = REF_GEOMS[name]
    grid, oc = _orc_cache(orc, g)
    rt = ref_tracer(ref, g)
    th = thetas(g["views"])
    rng = np.random.default_rng(23)
    fields = [rng.uniform(0.1, 2.0, grid.cell_count()) for _ in range(3)] + [np.ones(grid.cell_count())]
    for f in fields:
        assert np.array_equal(oc.project_length(th, f), rt.project_length(f))
    off, idx, ln = oc.length_lists(th)
    rows = th.size * oc.lines
    assert off.size == rows + 1 and off[-1] == idx.size == ln.size
    assert idx.max() < grid.cell_count() and (ln > 0).all()
    row_of = np.repeat(np.arange(rows), np.diff(off).astype(np.int64))
    for f in fields:
        got = np.bincount(row_of, weights=ln * f[idx], minlength=rows).reshape(th.size, oc.lines)
        np.testing.assert_allclose(got, oc.project_length(th, f), rtol=1e-12, atol=1e-13)
    key = row_of.astype(np.int64) * grid.cell_count() + idx
    assert np.unique(key).size == key.size  # a cell once per line
    # the binary model (azimuth range of a chord's end points, tracer.cpp:104-142)
    # and the length model (sector of each piece's midpoint) are two models of
    # the reference and differ on chords that pass near the axis: nearly all
    # cells agree
    extra = total = 0
    for v in range(th.size):
        for line in range(0, oc.lines, max(1, oc.lines // 16)):
            r = v * oc.lines + line
            mine = set(idx[off[r]:off[r + 1]].tolist())
            total += len(mine)
            extra += len(mine - set(oc.trace_line(line, th[v]).tolist()))
    assert extra <= 0.02 * total


def test_weighted_mart_restatement_matches_reference(orc, ref):
    """orc_weighted_mart on the reference's own Cartesian system reproduces
    cartesian_mart_stored bit for bit (weighted_update, auto_p_floor, clamp)."""
    g = REF_GEOMS["fan32"]
    off, idx, w = ref.cartesian_system(g["n"], False, g["src"], g["ctr"], g["du"], 1, g["su"], 0.0, g["views"])
    rng = np.random.default_rng(17)
    proj = rng.uniform(0.5, 3.0, g["views"] * g["du"])
    proj[::7] = 0.0
    proj[3::11] *= 1e-9
    for beta in (0.4, 1.9):
        want, _ = ref.cartesian_mart(g["n"], False, g["src"], g["ctr"], g["du"], 1, g["su"], 0.0, g["views"], proj,
                                     beta=beta, sweeps=3, f_init=1.0, stored=True)
        got, clamps = orc.weighted_mart(off, idx, w, proj, beta=beta, sweeps=3, f_init=1.0, cells=want.size)
        assert np.array_equal(got, np.asarray(want).reshape(-1))
        assert (clamps > 0) == (beta > 1)
