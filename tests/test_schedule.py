"""The MART dependency schedule (host C++ in the product library, no GPU).

The device executors run the sweep out of order: by ASAP level (level
executors) or as soon as a unit's predecessors are done (dataflow). This is
exact only if (a) units of one level have pairwise disjoint supports, (b) the
order of updates on every cell is the sweep order, (c) every unit's
predecessors are exactly the last writers of its cells. Each is checked on the
reference geometries' real supports (oracle traces), and the strongest form is
checked numerically: replaying the reference's fp64 row action in schedule
order gives a field BIT-IDENTICAL to the sequential reference.
"""
import numpy as np
import pytest

import oracle
from refgeoms import REF_GEOMS, thetas


def _supports(orc, name):
    g = REF_GEOMS[name]
    grid = oracle.OrcGrid.reference(g["n"], g["volume"])
    s, d = orc.rays_flat(g["src"], g["ctr"], g["du"], g["dv"], g["su"], g["sv"])
    oc = orc.cache(grid, s, d)
    th = thetas(g["views"])
    sup = [oc.trace_line(l, th[v]) for v in range(g["views"]) for l in range(g["du"] * g["dv"])]
    return grid, oc, th, sup


@pytest.mark.parametrize("name", ["fan32", "cone16", "fan64q"])
def test_schedule_levels_are_disjoint_and_order_preserving(ub, orc, name):
    grid, oc, th, sup = _supports(orc, name)
    sch = ub.uscg.schedule_build(sup, grid.cell_count())
    order, loff = sch["order"], sch["level_off"]
    assert sorted(order.tolist()) == list(range(len(sup)))
    level = np.zeros(len(sup), np.int64)
    for lv in range(sch["levels"]):
        members = order[loff[lv]:loff[lv + 1]]
        level[members] = lv
        assert list(members) == sorted(members)  # stable: sweep order inside a level
        seen = set()
        for u in members:
            cells = set(sup[u].tolist())
            assert not (cells & seen), "two units of one level share a cell"
            seen |= cells
    # per cell, the writers appear in increasing level in sweep order
    last = {}
    for u, s in enumerate(sup):
        for c in s.tolist():
            if c in last:
                assert level[u] > level[last[c]]
            last[c] = u


@pytest.mark.parametrize("name", ["fan32", "cone16"])
def test_schedule_predecessors_are_last_writers(ub, orc, name):
    grid, oc, th, sup = _supports(orc, name)
    sch = ub.uscg.schedule_build(sup, grid.cell_count())
    last = {}
    for u, s in enumerate(sup):
        want = sorted({last[c] for c in s.tolist() if c in last})
        got = sch["preds"][sch["pred_off"][u]:sch["pred_off"][u + 1]].tolist()
        assert got == want
        for c in s.tolist():
            last[c] = u


@pytest.mark.parametrize("name", ["fan16", "cone12", "fan32"])
def test_schedule_order_replays_the_sequential_reference_bit_exactly(ub, orc, name):
    """fp64 row action in schedule (level) order == the oracle's sequential
    reconstruct (pinned to the reference library), bit for bit."""
    grid, oc, th, sup = _supports(orc, name)
    sch = ub.uscg.schedule_build(sup, grid.cell_count())
    truth = np.random.default_rng(9).uniform(0.2, 3.0, grid.cell_count())
    proj = oc.project(th, truth).reshape(-1)
    beta, sweeps = 0.4, 3
    want, rep = oc.reconstruct(th, proj.reshape(len(th), -1), beta=beta, tolerance=0, max_sweeps=sweeps)
    pos = proj[proj > 0]
    p_floor = 1e-12 * (pos.sum() / pos.size)  # auto_p_floor (solver.cpp:64-74), same order
    f = np.ones(grid.cell_count())
    for _ in range(sweeps):
        for u in sch["order"]:
            m = proj[u]
            if m == 0:
                continue
            s = sup[u]
            p_bar = 0.0
            for c in s:  # sequential sum, the reference's emission order
                p_bar += f[c]
            factor = 1.0 - beta * (1.0 - m / max(p_bar, p_floor))
            if factor <= 0:
                factor = p_floor
            f[s] = f[s] * factor
    assert np.array_equal(f, want)


def _replay(grid, sup, proj, tasks, beta, p_floor):
    """fp64 row action over (sweep, line) tasks in the given order."""
    f = np.ones(grid.cell_count())
    for _, u in tasks:
        m = proj[u]
        if m == 0:
            continue
        s = sup[u]
        p_bar = 0.0
        for c in s:
            p_bar += f[c]
        factor = 1.0 - beta * (1.0 - m / max(p_bar, p_floor))
        if factor <= 0:
            factor = p_floor
        f[s] = f[s] * factor
    return f


@pytest.mark.parametrize("name,run", [("fan32", 5), ("cone16", 9), ("fan16", 7)])
def test_run_dag_with_cross_sweep_edges_replays_bit_exactly(ub, orc, name, run):
    """Runs of `run` lines, two sweeps back to back: any topological order of
    the (sweep, run) DAG — in-sweep preds from the library, cross-sweep preds
    derived independently here and checked against the library's counts —
    reproduces two sequential reference sweeps bit for bit."""
    g = REF_GEOMS[name]
    grid, oc, th, sup = _supports(orc, name)
    L = g["du"] * g["dv"]
    sch = ub.uscg.schedule_build(sup, grid.cell_count(), lines_per_view=L, run=run)
    nruns = len(sup) // run
    assert sch["order"].size == nruns
    # independent derivation: cross preds = final writers of first-touch cells
    first_writer = {}
    last_writer = {}
    for u, s in enumerate(sup):
        for c in s.tolist():
            first_writer.setdefault(c, u // run)
            last_writer[c] = u // run
    xpreds = [set() for _ in range(nruns)]
    for c, r in first_writer.items():
        xpreds[r].add(last_writer[c])
    assert [len(x) for x in xpreds] == sch["npred_x"].tolist()
    preds = [set(sch["preds"][sch["pred_off"][r]:sch["pred_off"][r + 1]].tolist()) for r in range(nruns)]
    # random topological order of (sweep, run) for 2 sweeps
    rng = np.random.default_rng(run)
    deps = {}
    for sw in range(2):
        for r in range(nruns):
            d = {(sw, p) for p in preds[r]}
            if sw == 1:
                d |= {(0, p) for p in xpreds[r]}
            deps[(sw, r)] = d
    done, order = set(), []
    ready = [k for k, d in deps.items() if not d]
    while ready:
        k = ready.pop(int(rng.integers(len(ready))))
        done.add(k)
        order.append(k)
        for k2, d in deps.items():
            if k2 not in done and k2 not in ready and k2 not in [o for o in order] and d <= done:
                ready.append(k2)
    assert len(order) == 2 * nruns
    if name == "cone16":
        assert order != sorted(order)  # the 3D DAG leaves real freedom: out of sweep order
    truth = np.random.default_rng(9).uniform(0.2, 3.0, grid.cell_count())
    proj = oc.project(th, truth).reshape(-1)
    pos = proj[proj > 0]
    p_floor = 1e-12 * (pos.sum() / pos.size)
    tasks = [(sw, r * run + j) for sw, r in order for j in range(run)]
    got = _replay(grid, sup, proj, tasks, 0.4, p_floor)
    want, _ = oc.reconstruct(th, proj.reshape(len(th), -1), beta=0.4, tolerance=0, max_sweeps=2)
    assert np.array_equal(got, want)


def test_schedule_rejects_bad_supports(ub):
    with pytest.raises(ub.InvalidArgument):
        ub.uscg.schedule_build([np.array([0, 5])], 4)


def test_schedule_sizes_for_c1_reference_analogue(ub, orc):
    """the c1 analogue (128^2, 36 views, 128 detectors,
    near-parallel beam) has 548 ASAP levels over 4,608 lines."""
    grid = oracle.OrcGrid.reference(128)
    s, d = orc.rays_flat((-1e4, 0, 0), (1.5, 0, 0), 128, 1, 2.0 / 128, 0.0)
    oc = orc.cache(grid, s, d)
    th = thetas(36)
    sup = [oc.trace_line(l, th[v]) for v in range(36) for l in range(128)]
    sch = ub.uscg.schedule_build(sup, grid.cell_count())
    assert len(sup) == 4608
    assert sch["levels"] == 548
