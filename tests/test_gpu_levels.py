"""The level executor (mart_level_kernel, csrc/mart_levels.cu): one launch per
ASAP level of the line DAG, chained by programmatic dependent launch, a block
per line with a non-zero measurement. Against the oracle (solver.cpp:33-51,
76-162) and the dataflow executor on cone-beam and 2D cases that the default
policy would hand to the tile executor."""
import numpy as np
import pytest

from test_gpu_parity import _m1_case

pytestmark = pytest.mark.gpu


def _case(ub, orc, kind):
    if kind == "volume":
        return _m1_case(ub, orc, "flat", volume=True, du=32, dv=16, views=12)
    return _m1_case(ub, orc, "arc", n_rings=48, views=16, du=96)


def _data(ub, tr, spec, seed):
    rng = np.random.default_rng(seed)
    truth = rng.uniform(0.2, 3.0, spec.cell_count())
    proj = ub.project_stack(tr, truth[None].astype(np.float32))[0].astype(np.float64)
    flat = proj.reshape(-1)
    flat[rng.choice(flat.size, flat.size // 5, replace=False)] = 0  # skipped lines: no block is launched for them
    return proj


@pytest.mark.parametrize("kind", ["volume", "slice"])
@pytest.mark.parametrize("threads,graph,sweeps", [("256", "0", 4), ("128", "1", 3), ("64", "0", 2), ("256", None, 17)])
def test_level_executor_matches_oracle_and_flow(ub, orc, monkeypatch, kind, threads, graph, sweeps):
    """Fields within 1e-4 of the oracle and 2e-5 of the dataflow executor,
    exact counters and crossed masks; plain launches, the graph replay
    (forced, and by the 16-sweep policy) and every block size."""
    monkeypatch.setenv("USCG_LEVEL_THREADS", threads)
    if graph is not None:
        monkeypatch.setenv("USCG_LEVEL_GRAPH", graph)
    spec, geom, tr, oc = _case(ub, orc, kind)
    proj = _data(ub, tr, spec, 5)
    cfg = ub.SolverConfig(beta=0.6, tolerance=0, max_sweeps=sweeps)
    out = {}
    for mode in ("levels", "flow"):
        monkeypatch.setenv("USCG_MART_MODE", mode)
        out[mode] = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, cfg, tr)
        assert tr.info()["executor"] == (5 if mode == "levels" else 0)
    got, flow = out["levels"], out["flow"]
    want, wrep = oc.reconstruct(geom.thetas(), proj, beta=0.6, tolerance=0, max_sweeps=sweeps)
    assert (np.abs(got.field.values - want) / want).max() <= 1e-4
    assert (np.abs(got.field.values - flow.field.values) / flow.field.values).max() <= 2e-5
    rep = got.report
    assert rep.sweeps == wrep["sweeps"] and rep.updates == wrep["updates"]
    assert rep.zero_measurement_skips == wrep["zero_measurement_skips"]
    assert rep.factor_clamps == wrep["factor_clamps"]
    assert np.array_equal(rep.crossed, wrep["crossed"])


def test_level_executor_residuals_convergence_and_initial_field(ub, orc, monkeypatch):
    """tolerance > 0 (one sweep per launch, the residual after each,
    solver.cpp:138-158) and reconstruct_from an initial field."""
    monkeypatch.setenv("USCG_MART_MODE", "levels")
    spec, geom, tr, oc = _case(ub, orc, "volume")
    proj = _data(ub, tr, spec, 9)
    cfg = ub.SolverConfig(beta=0.5, tolerance=2e-2, max_sweeps=12)
    res = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, cfg, tr)
    want, wrep = oc.reconstruct(geom.thetas(), proj, beta=0.5, tolerance=2e-2, max_sweeps=12)
    assert res.report.sweeps == wrep["sweeps"] and res.report.converged == wrep["converged"]
    np.testing.assert_allclose(res.report.sweep_residuals, wrep["sweep_residuals"], rtol=2e-3, atol=1e-6)
    assert (np.abs(res.field.values - want) / want).max() <= 1e-4
    init = np.random.default_rng(2).uniform(0.5, 1.5, spec.cell_count())
    cfg2 = ub.SolverConfig(beta=0.5, tolerance=0, max_sweeps=2)
    res2 = ub.reconstruct_from(ub.ProjectionSet(geom, proj), ub.Field(spec, init.astype(np.float32)), cfg2, tr)
    want2, _ = oc.reconstruct(geom.thetas(), proj, init=init.astype(np.float32).astype(np.float64), beta=0.5,
                              tolerance=0, max_sweeps=2)
    assert (np.abs(res2.field.values - want2) / want2).max() <= 1e-4


def test_level_executor_clamps_and_power_form(ub, orc, monkeypatch):
    """Non-positive factors clamp to p_floor and are counted like the
    oracle's (solver.cpp:42-45); the power-form update (m/p)^beta."""
    monkeypatch.setenv("USCG_MART_MODE", "levels")
    spec, geom, tr, oc = _case(ub, orc, "volume")
    proj = _data(ub, tr, spec, 13)
    tiny = proj.copy()
    tiny.reshape(-1)[::5] *= 1e-9
    res = ub.reconstruct(ub.ProjectionSet(geom, tiny), spec, ub.SolverConfig(beta=1.9, tolerance=0, max_sweeps=1), tr)
    _, wrep = oc.reconstruct(geom.thetas(), tiny, beta=1.9, tolerance=0, max_sweeps=1)
    assert wrep["factor_clamps"] > 0 and res.report.factor_clamps == wrep["factor_clamps"]
    assert (res.field.values > 0).all()
    cfg = ub.SolverConfig(beta=0.7, tolerance=0, max_sweeps=3, update="power")
    got = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, cfg, tr)
    want, _ = oc.reconstruct(geom.thetas(), proj, beta=0.7, tolerance=0, max_sweeps=3, power=True)
    assert (np.abs(got.field.values - want) / want).max() <= 1e-4


def test_level_executor_all_zero_data_returns_the_initial_field(ub, orc, monkeypatch):
    monkeypatch.setenv("USCG_MART_MODE", "levels")
    spec, geom, tr, oc = _case(ub, orc, "slice")
    proj = np.zeros((geom.views, geom.lines()))
    res = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, ub.SolverConfig(beta=0.5, tolerance=0, max_sweeps=3,
                                                                            f_init=1.25), tr)
    assert res.report.all_zero_data and np.all(res.field.values == np.float32(1.25))


def test_level_executor_graph_cache_replays_and_follows_the_data(ub, orc, monkeypatch):
    """The tracer keeps a sweep's launches as a graph once a solve repeats
    (call 2 builds it, later calls replay it): every call returns the first
    call's field bit for bit; other data (other live lines, another beta) are
    not served by the stale graph."""
    monkeypatch.setenv("USCG_MART_MODE", "levels")
    spec, geom, tr, oc = _case(ub, orc, "volume")
    proj = _data(ub, tr, spec, 21)
    cfg = ub.SolverConfig(beta=0.6, tolerance=0, max_sweeps=3)
    first = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, cfg, tr).field.values
    for _ in range(4):
        again = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, cfg, tr).field.values
        assert np.array_equal(again, first)
    other = _data(ub, tr, spec, 22)  # other zero lines: other grid sizes per level
    got = ub.reconstruct(ub.ProjectionSet(geom, other), spec, cfg, tr).field.values
    want, _ = oc.reconstruct(geom.thetas(), other, beta=0.6, tolerance=0, max_sweeps=3)
    assert (np.abs(got - want) / want).max() <= 1e-4
    scaled = proj * 1.5  # the same live lines, other measurements: the graph reads them at run time
    got = ub.reconstruct(ub.ProjectionSet(geom, scaled), spec, cfg, tr).field.values
    want, _ = oc.reconstruct(geom.thetas(), scaled, beta=0.6, tolerance=0, max_sweeps=3)
    assert (np.abs(got - want) / want).max() <= 1e-4
    cfg2 = ub.SolverConfig(beta=0.9, tolerance=0, max_sweeps=3)  # beta is a kernel parameter: a new key
    for _ in range(3):
        got = ub.reconstruct(ub.ProjectionSet(geom, proj), spec, cfg2, tr).field.values
    want, _ = oc.reconstruct(geom.thetas(), proj, beta=0.9, tolerance=0, max_sweeps=3)
    assert (np.abs(got - want) / want).max() <= 1e-4
    assert np.array_equal(ub.reconstruct(ub.ProjectionSet(geom, proj), spec, cfg, tr).field.values, first)
