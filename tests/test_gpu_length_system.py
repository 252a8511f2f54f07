"""The polar grid's (voxel index, chord length) lists and the length-weighted
row action on them (uscg_tracer_length_system, include/uscg_b200.h): the device
lists against the oracle's (oracle.OrcCache.length_lists, pinned to the
reference's LengthWeighted projector, phantom.cpp:213-269, in
tests/test_oracle.py) and the device MART against the restated
weighted_update (siddon.cpp:141-154, pinned to cartesian_mart_stored)."""
import numpy as np
import pytest

from refgeoms import REF_GEOMS, ub_spec_geom
from test_gpu_parity import _m1_case

pytestmark = pytest.mark.gpu


def _ref_case(ub, orc, name):
    import oracle
    g = REF_GEOMS[name]
    spec, geom = ub_spec_geom(ub, g)
    grid = oracle.OrcGrid.reference(g["n"], g["volume"])
    s, d = orc.rays_flat(g["src"], g["ctr"], g["du"], g["dv"], g["su"], g["sv"])
    return spec, geom, ub.Tracer(geom, spec, False), orc.cache(grid, s, d)


def _cases(ub, orc, name):
    if name == "m1cone":
        return _m1_case(ub, orc, "flat", volume=True, du=32, dv=16, views=12)
    if name == "m1arc":
        return _m1_case(ub, orc, "arc", n_rings=48, views=16, du=96)
    return _ref_case(ub, orc, name)


@pytest.mark.parametrize("name", ["fan32", "cone16", "cone12", "m1cone", "m1arc"])
def test_length_lists_match_the_oracle(ub, orc, name):
    """Per (view, line): the same cells in the same order, lengths to fp32
    (slivers aside).
    Adjudicated like the projector (test_length_weighted_matches_reference): a
    ray through the axis is cut by the reference at a quotient of two rounding
    residues, so such a line may split one length between two sectors
    differently; those lines must carry the same total length."""
    spec, geom, tr, oc = _cases(ub, orc, name)
    ls = ub.LengthSystem(tr)
    off, idx, w = ls.export()
    ooff, oidx, ow = oc.length_lists(geom.thetas())
    rows = geom.views * geom.lines()
    assert off.size == rows + 1 == ooff.size
    differ = 0
    for r in range(rows):
        a, b = idx[off[r]:off[r + 1]], oidx[ooff[r]:ooff[r + 1]]
        wa, wb = w[off[r]:off[r + 1]].astype(np.float64), ow[ooff[r]:ooff[r + 1]]
        # slivers (a cut within rounding of a chord's end: a piece of ~1e-16 on
        # one side only) carry no weight and are not compared
        ka, kb = wa > 1e-9, wb > 1e-9
        if np.array_equal(a[ka], b[kb]):
            np.testing.assert_allclose(wa[ka], wb[kb], rtol=2e-6, atol=1e-9)
            assert wa[~ka].sum() <= 1e-8 and wb[~kb].sum() <= 1e-8
        else:
            # only a ray through the axis (the centre column of an odd panel)
            assert geom.det_u % 2 == 1 and (r % geom.lines()) % geom.det_u == geom.det_u // 2, r
            differ += 1
            assert abs(wa.sum() - wb.sum()) <= 1e-6 * max(1.0, wb.sum()), r
    assert differ <= geom.views * max(1, geom.det_v), differ
    inf = ls.info()
    assert inf["entries"] == off[-1] and inf["levels"] > 0
    # the lists reproduce the length-weighted projector
    f = np.random.default_rng(3).uniform(0.2, 2.0, spec.cell_count()).astype(np.float32)
    row_of = np.repeat(np.arange(rows), np.diff(off.astype(np.int64)))
    mine = np.bincount(row_of, weights=w.astype(np.float64) * f[idx], minlength=rows)
    proj = ub.project_stack(tr, f[None], model="length")[0].reshape(-1)
    np.testing.assert_allclose(mine, proj, rtol=2e-6, atol=1e-6)


@pytest.mark.parametrize("name,beta", [("fan32", 0.4), ("m1cone", 0.4), ("m1arc", 1.0), ("cone12", 1.0)])
def test_length_weighted_mart_matches_the_restated_row_action(ub, orc, name, beta):
    """Fixed sweeps of weighted_update over the polar lists (fp32 field on the
    device, fp64 in the oracle), zero measurements skipped; the oracle runs on
    the device's exported lists, so the arithmetic and the order of the updates
    are what is compared here (the clamp of a non-positive factor is pinned for
    the same kernel by test_cartesian_mart_matches_reference)."""
    spec, geom, tr, oc = _cases(ub, orc, name)
    ls = ub.LengthSystem(tr)
    off, idx, w = ls.export()
    truth = np.random.default_rng(29).uniform(0.3, 2.5, spec.cell_count()).astype(np.float32)
    proj = ub.project_stack(tr, truth[None], model="length")[0].reshape(-1).astype(np.float64)
    proj[::9] = 0.0
    sweeps = 3
    got, sec = ls.reconstruct(proj, ub.SolverConfig(beta=beta, tolerance=0, max_sweeps=sweeps))
    want, clamps = oc.weighted_mart(off, idx, w.astype(np.float64), proj, beta=beta, sweeps=sweeps)
    assert sec > 0 and got.shape == want.shape and clamps == 0
    touched = np.zeros(spec.cell_count(), bool)
    touched[idx] = True
    assert np.array_equal(got[~touched], np.ones((~touched).sum(), np.float32))
    np.testing.assert_allclose(got, want, rtol=1e-4)
    # closure: the reconstruction's length-weighted projections move towards the data
    if beta <= 1.0:
        row_of = np.repeat(np.arange(proj.size), np.diff(off.astype(np.int64)))
        re = np.bincount(row_of, weights=w * got[idx], minlength=proj.size)
        r0 = np.bincount(row_of, weights=w.astype(np.float64), minlength=proj.size)
        live = proj > 0
        assert np.abs(re[live] - proj[live]).mean() < 0.5 * np.abs(r0[live] - proj[live]).mean()


def test_length_system_needs_the_tracer_rays(ub, orc):
    """A tracer built from an imported cache has no rays: invalid argument, as
    for the length-weighted projector."""
    spec, geom, tr, _ = _ref_case(ub, orc, "fan16")
    tr2 = ub.Tracer.from_cache(spec, tr.cache(), geom.views)
    with pytest.raises(ub.InvalidArgument):
        ub.LengthSystem(tr2)
