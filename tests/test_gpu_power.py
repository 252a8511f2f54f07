"""The power-form update (USCG_UPDATE_POWER: x *= (m/p)^beta, BASELINE
north_star's (m/p)^(lambda a_v / max a) with binary coefficients). The
reference has only the linear form (proj/src/solver.cpp:41), so this is the
builder's extension: every executor is checked against the oracle's power
variant (oracle/uscg_oracle.c, orc_set_update_power), which shares every
other line of the restatement pinned to the reference library."""
import numpy as np
import pytest

import oracle
from refgeoms import REF_GEOMS, ub_spec_geom

pytestmark = pytest.mark.gpu


def _orc_case(orc, g, spec, geom):
    grid = oracle.OrcGrid.reference(g["n"], g["volume"])
    src, det = geom.first_view_rays()
    return orc.cache(grid, src, det)


@pytest.mark.parametrize("name,mode,sweeps", [("fan32", "tile", 4), ("fan128", "tile", 3), ("cone16", "flow", 3),
                                              ("fan32", "flow", 3)])
def test_power_update_matches_oracle(ub, orc, monkeypatch, name, mode, sweeps):
    monkeypatch.setenv("USCG_MART_MODE", mode)
    g = REF_GEOMS[name]
    spec, geom = ub_spec_geom(ub, g)
    tr = ub.Tracer(geom, spec, False)
    oc = _orc_case(orc, g, spec, geom)
    truth = np.random.default_rng(9).uniform(0.2, 3.0, spec.cell_count())
    proj = oc.project(geom.thetas(), truth.astype(np.float32).astype(np.float64)).astype(np.float32)
    beta = 0.7
    want, wrep = oc.reconstruct(geom.thetas(), proj.astype(np.float64), beta=beta, tolerance=0,
                                max_sweeps=sweeps, power=True)
    lin, _ = oc.reconstruct(geom.thetas(), proj.astype(np.float64), beta=beta, tolerance=0, max_sweeps=sweeps)
    res = ub.reconstruct(ub.ProjectionSet(geom, proj), spec,
                         ub.SolverConfig(beta=beta, tolerance=0, max_sweeps=sweeps, update="power"), tr)
    rel = np.abs(res.field.values - want) / want
    assert rel.max() <= 1e-4, rel.max()
    assert res.report.updates == wrep["updates"]
    assert res.report.factor_clamps == wrep["factor_clamps"] == 0
    assert np.abs(lin - want).max() > 1e-3  # the two forms differ


def test_power_update_stack_wave(ub, orc):
    """32 problems of a 48-ring M1 grid on an arc: the clustered wave executor"""
    n_rings, S, sweeps, beta = 48, 32, 3, 0.3
    counts = ub.ring_counts_m1(n_rings)
    spec = ub.GridSpec(2 * n_rings, 1.0 / n_rings, 1.0 / n_rings, ub.GridMode.Slice2D, ring_counts=counts)
    geom = ub.ScanGeometry(source=(-3, 0, 0), detector_center=(1.5, 0, 0), det_u=96, spacing_u=38.94 / 96,
                           views=16, detector=ub.Detector.Arc)
    tr = ub.Tracer(geom, spec, False)
    rng = np.random.default_rng(4)
    truth = rng.uniform(0.2, 2.0, (S, spec.cell_count())).astype(np.float32)
    proj = ub.project_stack(tr, truth)
    out = ub.reconstruct_stack(proj, ub.SolverConfig(beta=beta, tolerance=0, max_sweeps=sweeps, update="power"), tr)
    assert tr.info()["executor"] == 3
    g = oracle.OrcGrid(n_rings, 1.0 / n_rings, 1, 1.0 / n_rings, False, counts)
    src, det = geom.first_view_rays()
    oc = orc.cache(g, src, det)
    for p in (0, 13, 31):
        want, wrep = oc.reconstruct(geom.thetas(), proj[p].reshape(-1).astype(np.float64), beta=beta, tolerance=0,
                                    max_sweeps=sweeps, power=True)
        got, rep = out[p]
        rel = np.abs(got - want) / want
        assert rel.max() <= 1e-4, (p, rel.max())
        assert rep.updates == wrep["updates"]


def test_power_update_rejects_unknown_form(ub):
    with pytest.raises(ub.InvalidArgument):
        ub.SolverConfig(update="exp")._flags()
