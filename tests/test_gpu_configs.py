"""Parity at the BASELINE.json configurations themselves (verbatim C1-C4),
through the default executors the bench times, against the oracle port
(oracle/uscg_oracle.c, itself pinned bit-exactly to the unmodified reference
library on the reference's own configurations, tests/test_oracle.py).

Gates:
- U (updates), zero-measurement skips, factor clamps, sweeps, all-zero flags and
  crossed masks: exact;
- fields (fp32 on the device, fp64 in the oracle): max rel <= 1e-4;
- image quality: RMSE against the truth phantom equal to the oracle's within
  1e-5 (relative), in field space and on the Cartesian rasters
  (rmse_volume, proj/src/metrics.cpp:42-60,178-184);
- Pearson correlation against the truth: the builder's own figure (the
  reference has no correlation metric: parity unpinned),
  reported beside RMSE and gated at the same 1e-5.

Inputs are the bench's own: seeded phantoms (workloads.phantom_fields), binary
projections of them, the configuration's noise.
"""
import dataclasses
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 1e-4
QTOL = 1e-5


def pearson(a, b):
    a = np.asarray(a, np.float64).ravel() - np.mean(a)
    b = np.asarray(b, np.float64).ravel() - np.mean(b)
    return float(a @ b / np.sqrt((a @ a) * (b @ b)))


def _oracle_side(orc, spec, geom):
    import oracle
    g = oracle.OrcGrid.of(spec)
    src, det = orc.rays_for(geom)
    return g, src, det


def _oracle_many(orc, g, src, det, thetas, projs, beta, sweeps):
    """One oracle reconstruct per problem, one host thread each (ctypes
    releases the GIL; each thread owns its cache and scratch)."""
    out = [None] * len(projs)

    def work(i):
        oc = orc.cache(g, src, det)
        out[i] = oc.reconstruct(thetas, np.asarray(projs[i], np.float64), beta=beta, tolerance=0,
                                max_sweeps=sweeps)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(projs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return out


def _quality(ub, orc, g, spec, got, want, truth, npix):
    """RMSE / correlation vs truth of the device and oracle fields: field
    space, and on Cartesian rasters (device resample + device metrics vs the
    oracle's resample + rmse)."""
    r_got, r_want = orc.rmse(got, truth), orc.rmse(want, truth)
    c_got, c_want = pearson(got, truth), pearson(want, truth)
    assert abs(r_got - r_want) <= QTOL * max(r_want, 1e-12), (r_got, r_want)
    assert abs(c_got - c_want) <= QTOL, (c_got, c_want)
    img_t = orc.field_to_cartesian(g, truth, npix)
    img_w = orc.field_to_cartesian(g, want, npix)
    img_g = ub.resample_stack(spec, got.astype(np.float32)[None], npix)[0]
    img_t32 = ub.resample_stack(spec, truth.astype(np.float32)[None], npix)[0]
    rv_dev = ub.rmse_volume(img_t32, img_g)
    rv_orc = float(np.mean([orc.rmse(img_t[s], img_w[s]) for s in range(img_t.shape[0])]))
    assert abs(rv_dev - rv_orc) <= QTOL * max(rv_orc, 1e-12) + 1e-7, (rv_dev, rv_orc)
    print(f"rmse vs truth: device {r_got:.7g} oracle {r_want:.7g}; corr device {c_got:.8f} oracle {c_want:.8f}; "
          f"raster rmse_volume device {rv_dev:.7g} oracle {rv_orc:.7g}")
    return dict(rmse=(r_got, r_want), corr=(c_got, c_want), rmse_volume=(rv_dev, rv_orc))


def _check_report(rep, wrep, crossed=True):
    assert rep.sweeps == wrep["sweeps"]
    assert rep.all_zero_data == wrep["all_zero_data"]
    assert rep.updates == wrep["updates"]
    assert rep.zero_measurement_skips == wrep["zero_measurement_skips"]
    assert rep.factor_clamps == wrep["factor_clamps"]
    if crossed:
        assert np.array_equal(rep.crossed, wrep["crossed"])


def _maxrel(got, want):
    return float((np.abs(got - want) / np.abs(want)).max())


def test_c1_verbatim_all_iterations(ub, orc):
    """C1 as BASELINE states it (64 rings, M1 law, parallel beam, 36 views at
    5 deg, lambda 0.1): all 10 iterations through the default single-problem
    executor; solver.cpp:76-162."""
    from paper_2208_12964_b200 import workloads
    wl = workloads.make("c1")
    spec, geom = wl.spec, wl.geom
    tr = ub.Tracer(geom, spec, False)
    truth = workloads.phantom_fields(wl, 1)[0]
    proj = ub.project_stack(tr, truth[None].astype(np.float32))[0]
    res = ub.reconstruct(ub.ProjectionSet(geom, proj.astype(np.float64)), spec,
                         ub.SolverConfig(beta=wl.beta, tolerance=0, max_sweeps=wl.sweeps), tr)
    g, src, det = _oracle_side(orc, spec, geom)
    (want, wrep), = _oracle_many(orc, g, src, det, geom.thetas(), [proj], wl.beta, wl.sweeps)
    got = res.field.values
    _check_report(res.report, wrep)
    assert _maxrel(got, want) <= RTOL
    _quality(ub, orc, g, spec, got, want, truth, 128)


def test_c2_verbatim_wave_twenty_sweeps(ub, orc, capfd, monkeypatch):
    """C2 as the bench runs it: 256 rings (M1 law), 512-detector arc, 90
    views, 128 slices with 1% noise, lambda 0.05, all 20 sweeps in one
    reconstruct call through the default mart_wave_kernel<32>. Problems from
    the first and the last 32-problem chunk and two between are compared with
    the oracle; every problem's counters are compared with the oracle's
    closed form (U = sum of |active| over non-skipped lines x sweeps)."""
    from paper_2208_12964_b200 import workloads
    monkeypatch.setenv("USCG_FLOW_VERBOSE", "1")
    wl = workloads.make("c2")
    spec, geom, S = wl.spec, wl.geom, wl.problems
    tr = ub.Tracer(geom, spec, False)
    truth = workloads.phantom_fields(wl, S)
    proj = workloads.add_noise(wl, ub.project_stack(tr, truth.astype(np.float32))).astype(np.float32)
    out = ub.reconstruct_stack(proj, ub.SolverConfig(beta=wl.beta, tolerance=0, max_sweeps=wl.sweeps), tr,
                               with_crossed=True)
    if os.environ.get("USCG_MART_MODE", "auto") in ("auto", "wave"):
        assert "mart_wave_kernel: P=32 " in capfd.readouterr().err
    counts = tr.trace_counts().reshape(-1).astype(np.int64)
    for p in range(S):
        nz = proj[p].reshape(-1) != 0
        assert out[p][1].updates == int(counts[nz].sum()) * wl.sweeps, p
        assert out[p][1].zero_measurement_skips == int((~nz).sum()) * wl.sweeps, p
    pick = [0, 31, 77, 127]
    g, src, det = _oracle_side(orc, spec, geom)
    ref = _oracle_many(orc, g, src, det, geom.thetas(), [proj[p] for p in pick], wl.beta, wl.sweeps)
    print("c2 max rel per problem:", {p: _maxrel(out[p][0], want) for p, (want, _) in zip(pick, ref)})
    for p, (want, wrep) in zip(pick, ref):
        got, rep = out[p]
        _check_report(rep, wrep)
        assert _maxrel(got, want) <= RTOL, (p, _maxrel(got, want))
    _quality(ub, orc, g, spec, out[0][0].astype(np.float64), ref[0][0], truth[0], 512)
    _quality(ub, orc, g, spec, out[127][0].astype(np.float64), ref[3][0], truth[127], 512)


@pytest.mark.parametrize("S,width,cl", [(64, 16, 2), (16, 16, 2), (32, 16, 4), (96, 32, 4)])
def test_c2_shard_per_gpu_paired_wave(ub, orc, capfd, monkeypatch, S, width, cl):
    """The C2 stack as one GPU of 2 / 4 / 8 holds it (64 / 32 / 16 slices, in
    16-problem chunks) and a 96-slice stack (32-problem chunks): all 20 sweeps
    through the clustered wave form (a view task on a 2-CTA cluster, or the
    opt-in 4-CTA one; cells split by index mod cluster size, partial sums
    exchanged through distributed shared memory), problems of the first and
    last slots against the oracle."""
    from paper_2208_12964_b200 import workloads
    monkeypatch.setenv("USCG_FLOW_VERBOSE", "1")
    if cl != 2:
        monkeypatch.setenv("USCG_WAVE_PAIR", str(cl))
    wl = workloads.make("c2", problems=S)
    spec, geom = wl.spec, wl.geom
    tr = ub.Tracer(geom, spec, False)
    truth = workloads.phantom_fields(wl, S, first=64)
    proj = workloads.add_noise(wl, ub.project_stack(tr, truth.astype(np.float32)), first=64).astype(np.float32)
    out = ub.reconstruct_stack(proj, ub.SolverConfig(beta=wl.beta, tolerance=0, max_sweeps=wl.sweeps), tr,
                               with_crossed=True)
    assert f"mart_wave_kernel: P={width} pair cluster={cl}" in capfd.readouterr().err
    pick = [0, S - 1]
    g, src, det = _oracle_side(orc, spec, geom)
    ref = _oracle_many(orc, g, src, det, geom.thetas(), [proj[p] for p in pick], wl.beta, wl.sweeps)
    for p, (want, wrep) in zip(pick, ref):
        got, rep = out[p]
        _check_report(rep, wrep)
        assert _maxrel(got, want) <= RTOL, (p, _maxrel(got, want))


def test_c3_verbatim_two_sweeps(ub, orc):
    """C3 as BASELINE states it (128 rings x 128 layers, M1 law, cone beam,
    256x256 flat panel, 36 views, lambda 0.05): two back-to-back sweeps (the
    cross-sweep dependencies included) through the default volume executor."""
    from paper_2208_12964_b200 import workloads
    wl = workloads.make("c3")
    spec, geom = wl.spec, wl.geom
    tr = ub.Tracer(geom, spec, False)
    truth = workloads.phantom_fields(wl, 1)[0]
    proj = ub.project_stack(tr, truth[None].astype(np.float32))[0]
    sweeps = 2
    res = ub.reconstruct(ub.ProjectionSet(geom, proj.astype(np.float64)), spec,
                         ub.SolverConfig(beta=wl.beta, tolerance=0, max_sweeps=sweeps), tr)
    g, src, det = _oracle_side(orc, spec, geom)
    (want, wrep), = _oracle_many(orc, g, src, det, geom.thetas(), [proj], wl.beta, sweeps)
    got = res.field.values
    _check_report(res.report, wrep)
    assert _maxrel(got, want) <= RTOL
    _quality(ub, orc, g, spec, got, want, truth, 256)


def test_c4_verbatim_view_subset(ub, orc):
    """C4 (256 rings x 256 layers, M1 law, 512x512 panel, source 5R, the lump
    phantom with 0.5% noise, lambda 0.02) over its first 8 views (0..35 deg;
    the full 72-view sweep takes ~2.5 min in the oracle), two back-to-back
    sweeps through the default volume executor."""
    from paper_2208_12964_b200 import workloads
    wl = workloads.make("c4")
    spec = wl.spec
    geom = dataclasses.replace(wl.geom, views=8, view_angles=np.array([5.0 * i for i in range(8)]))
    tr = ub.Tracer(geom, spec, False)
    truth = workloads.phantom_fields(wl, 1)[0]
    proj = workloads.add_noise(wl, ub.project_stack(tr, truth[None].astype(np.float32)))[0].astype(np.float32)
    sweeps = 2
    res = ub.reconstruct(ub.ProjectionSet(geom, proj.astype(np.float64)), spec,
                         ub.SolverConfig(beta=wl.beta, tolerance=0, max_sweeps=sweeps), tr)
    g, src, det = _oracle_side(orc, spec, geom)
    (want, wrep), = _oracle_many(orc, g, src, det, geom.thetas(), [proj], wl.beta, sweeps)
    got = res.field.values
    _check_report(res.report, wrep)
    assert _maxrel(got, want) <= RTOL
    _quality(ub, orc, g, spec, got, want, truth, 512)
