"""Sharded device paths on one GPU: every rank's share is
computed by the same library calls a rank makes, one rank after another, and
the assembled result must equal the single-GPU result bit for bit. The
exchanges themselves are tested over gloo in test_multiproc.py.

- projector by view (proj/src/phantom.cpp:182-211: every (view, line)
  independent, the field read-only): dist.project_views_local + concat_views;
- resampling by slice (proj/src/phantom.cpp:149-163): dist.resample_local.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _stack_case(ub):
    n_rings = 48
    spec = ub.GridSpec(2 * n_rings, 1 / n_rings, 1 / n_rings, ub.GridMode.Slice2D, ring_counts=ub.ring_counts_m1(n_rings))
    geom = ub.ScanGeometry(source=(-3, 0, 0), detector_center=(1.5, 0, 0), det_u=96, spacing_u=38.94 / 96, views=23,
                           detector=ub.Detector.Arc)
    return spec, geom


def _volume_case(ub):
    n_rings = 24
    spec = ub.GridSpec(2 * n_rings, 1 / n_rings, 2 / n_rings, ub.GridMode.Volume3D,
                       ring_counts=ub.ring_counts_m1(n_rings), n_slices=20)
    geom = ub.ScanGeometry(source=(-4, 0, 0), detector_center=(2, 0, 0), det_u=40, det_v=24, spacing_u=3.1 / 40,
                           spacing_v=2.2 / 24, views=13)
    return spec, geom


@pytest.mark.parametrize("case,S", [("stack", 5), ("volume", 1)])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_view_sharded_projection_equals_full(ub, case, S, world):
    from paper_2208_12964_b200 import dist as udist
    spec, geom = (_stack_case if case == "stack" else _volume_case)(ub)
    tr = ub.Tracer(geom, spec, False)
    fields = np.random.default_rng(world).uniform(0.1, 2.0, (S, spec.cell_count())).astype(np.float32)
    full = ub.project_stack(tr, fields)
    parts = [udist.project_views_local(tr, fields, r, world) for r in range(world)]
    assert sum(p.shape[1] for p in parts) == geom.views
    assert np.array_equal(udist.concat_views(parts), full)


@pytest.mark.parametrize("world", [2, 3, 7])
def test_slice_sharded_resample_equals_full(ub, world):
    from paper_2208_12964_b200 import dist as udist
    spec, _ = _volume_case(ub)
    field = np.random.default_rng(world).uniform(0, 1, spec.cell_count()).astype(np.float32)
    npix = 64
    full = ub.resample_stack(spec, field[None], npix)[0]
    parts = [udist.resample_local(spec, field, npix, r, world) for r in range(world)]
    assert np.array_equal(np.concatenate(parts), full)
