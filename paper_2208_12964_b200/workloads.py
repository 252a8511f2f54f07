"""Seeded synthetic workloads for the BASELINE.json configurations.

BASELINE.json names five configurations (C1-C5); SURVEY.md §0.1 / §8(d) fix
the choices they leave open. Each config comes in two forms:

* ``cN``      the configuration as BASELINE.json states it (generalized seams:
              sector law round(2*pi*(i+0.5)), decoupled slice count, parallel /
              arc detectors, 180-degree view list);
* ``cN-ref``  the closest configuration the unmodified reference library can
              express (4(2k-1) law, n slices, point source + flat panel,
              360 degrees) — runnable on oracle/_ref.

Phantoms are random additive ellipses/ellipsoids sampled at cell centroids
(the reference's sampling rule, proj/src/phantom.cpp:119-130); projections come
from the binary forward model; noise is multiplicative and clipped at zero
(SURVEY.md M9). These are input generators, not part of the hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .uscg import Detector, GridMode, GridSpec, ScanGeometry, ring_counts_m1


@dataclass
class Workload:
    name: str
    spec: GridSpec
    geom: ScanGeometry
    beta: float
    sweeps: int
    problems: int = 1
    phantom: str = "ellipses"        # ellipses | ellipsoids | lump
    n_shapes: int = 10
    axes: tuple = (0.05, 0.4)
    centre_frac: float = 0.6
    noise: str = "none"              # none | gauss | poisson
    noise_level: float = 0.0
    seed: int = 12345
    notes: dict = field(default_factory=dict)


def _r(n_rings: int) -> float:
    return 1.0 / n_rings  # unit image radius


def make(name: str, problems: Optional[int] = None) -> Workload:
    name = name.lower()
    if name == "c1":
        n = 128
        spec = GridSpec(n, _r(64), _r(64), GridMode.Slice2D, ring_counts=ring_counts_m1(64))
        geom = ScanGeometry(source=(-2.0, 0, 0), detector_center=(2.0, 0, 0), det_u=128, spacing_u=2.0 / 128,
                            views=36, detector=Detector.Parallel,
                            view_angles=np.array([5.0 * i for i in range(36)]))
        return Workload(name, spec, geom, beta=0.1, sweeps=10)
    if name == "c1-ref":
        n = 128
        spec = GridSpec.square_2d(n)
        geom = ScanGeometry(source=(-1e4, 0, 0), detector_center=(1.5, 0, 0), det_u=128, spacing_u=2.0 / 128,
                            views=36)
        return Workload(name, spec, geom, beta=0.1, sweeps=10)
    if name == "c2":
        n = 512
        spec = GridSpec(n, _r(256), _r(256), GridMode.Slice2D, ring_counts=ring_counts_m1(256))
        fan = 2.0 * math.degrees(math.asin(1.0 / 3.0))
        geom = ScanGeometry(source=(-3.0, 0, 0), detector_center=(1.5, 0, 0), det_u=512, spacing_u=fan / 512,
                            views=90, detector=Detector.Arc)
        return Workload(name, spec, geom, beta=0.05, sweeps=20, problems=problems or 128, noise="gauss",
                        noise_level=0.01)
    if name == "c2-ref":
        n = 512
        spec = GridSpec.square_2d(n)
        su = 2.0 * 4.5 * math.tan(math.asin(1.0 / 3.0)) / 512
        geom = ScanGeometry(source=(-3.0, 0, 0), detector_center=(1.5, 0, 0), det_u=512, spacing_u=su, views=90)
        return Workload(name, spec, geom, beta=0.05, sweeps=20, problems=problems or 128, noise="gauss",
                        noise_level=0.01)
    if name == "c3":
        spec = GridSpec(256, _r(128), 2 * _r(128), GridMode.Volume3D, ring_counts=ring_counts_m1(128),
                        n_slices=128)
        su = 2.0 * 6.0 * math.tan(math.asin(0.25)) / 256
        geom = ScanGeometry(source=(-4.0, 0, 0), detector_center=(2.0, 0, 0), det_u=256, det_v=256,
                            spacing_u=su, spacing_v=4.1 / 256, views=36)
        return Workload(name, spec, geom, beta=0.05, sweeps=10, phantom="ellipsoids", n_shapes=16,
                        axes=(0.05, 0.35), centre_frac=0.5)
    if name == "c3-ref":
        spec = GridSpec.cube_3d(256)
        s = 2.0 * 6.0 * 0.2582 / 256
        geom = ScanGeometry(source=(-4.0, 0, 0), detector_center=(2.0, 0, 0), det_u=256, det_v=256,
                            spacing_u=s, spacing_v=s, views=36)
        return Workload(name, spec, geom, beta=0.05, sweeps=10, phantom="ellipsoids", n_shapes=16,
                        axes=(0.05, 0.35), centre_frac=0.5)
    if name == "c4":
        spec = GridSpec(512, _r(256), 2 * _r(256), GridMode.Volume3D, ring_counts=ring_counts_m1(256),
                        n_slices=256)
        su = 2.0 * 7.5 * math.tan(math.asin(0.2)) / 512
        geom = ScanGeometry(source=(-5.0, 0, 0), detector_center=(2.5, 0, 0), det_u=512, det_v=512,
                            spacing_u=su, spacing_v=2.0 * 1.875 * 1.02 / 512, views=72)
        return Workload(name, spec, geom, beta=0.02, sweeps=15, phantom="lump", noise="poisson",
                        noise_level=0.005)
    if name == "c5":
        spec = GridSpec(1024, _r(512), 2 * _r(512), GridMode.Volume3D, ring_counts=ring_counts_m1(512),
                        n_slices=512)
        su = 2.0 * 7.5 * math.tan(math.asin(0.2)) / 1024
        geom = ScanGeometry(source=(-5.0, 0, 0), detector_center=(2.5, 0, 0), det_u=1024, det_v=1024,
                            spacing_u=su, spacing_v=2.0 * 1.875 * 1.02 / 1024, views=180)
        return Workload(name, spec, geom, beta=0.02, sweeps=1)
    raise KeyError(f"unknown workload {name!r}")


# ---------------------------------------------------------------------------
# phantoms (cell-centroid sampling, phantom.cpp:119-130)
# ---------------------------------------------------------------------------


def cell_centroids(spec: GridSpec):
    """(x, y) of every cell of one slice in flat order, plus slice centres z."""
    counts = spec.counts().astype(np.int64)
    ring = np.repeat(np.arange(1, counts.size + 1), counts)
    heads = np.concatenate([[0], np.cumsum(counts)[:-1]])
    local = np.arange(counts.sum()) - np.repeat(heads, counts)
    step = 360.0 / counts[ring - 1]
    radius = (ring - 0.5) * spec.ring_spacing
    ang = np.radians((local + 0.5) * step)
    x = radius * np.cos(ang)
    y = radius * np.sin(ang)
    if spec.mode == GridMode.Volume3D:
        zoff = 0.5 * spec.slices() * spec.slice_height
        z = (np.arange(spec.slices()) + 0.5) * spec.slice_height - zoff
    else:
        z = np.zeros(1)
    return x, y, z


def random_shapes(rng: np.random.Generator, wl: Workload, volume: bool):
    """Per shape, draw order: density, ax, ay, (az), centre radius, centre angle,
    (centre z), rotation."""
    shapes = []
    lo, hi = wl.axes
    for _ in range(wl.n_shapes):
        dens = rng.uniform(0.1, 1.0)
        ax = rng.uniform(lo, hi)
        ay = rng.uniform(lo, hi)
        az = rng.uniform(lo, hi) if volume else 1.0
        cr = wl.centre_frac * math.sqrt(rng.uniform())
        ca = rng.uniform(0, 2 * math.pi)
        cz = rng.uniform(-0.5, 0.5) if volume else 0.0
        rot = rng.uniform(0, 360.0)
        shapes.append((dens, ax, ay, az, cr * math.cos(ca), cr * math.sin(ca), cz, rot))
    return shapes


def shapes_value(shapes, x, y, z, volume: bool):
    """Additive shapes (phantom_value, phantom.cpp:50-70), unit-radius coordinates."""
    v = np.zeros(np.broadcast(x, y, z).shape)
    for dens, ax, ay, az, cx, cy, cz, rot in shapes:
        c, s = math.cos(math.radians(rot)), math.sin(math.radians(rot))
        px, py = x - cx, y - cy
        qx = c * px + s * py
        qy = -s * px + c * py
        q = (qx / ax) ** 2 + (qy / ay) ** 2
        if volume:
            q = q + ((z - cz) / az) ** 2
        v = v + np.where(q < 1.0, dens, 0.0)
    return v


def lump_value(rng: np.random.Generator, x, y, z):
    """C4: 8.0 inside the union of 8 overlapping spheres, else 0.2 inside a
    radius-0.9 cylinder, else 0 (an indicator union, not additive)."""
    centres = []
    for _ in range(8):
        r = 0.3 * math.sqrt(rng.uniform())
        a = rng.uniform(0, 2 * math.pi)
        centres.append((r * math.cos(a), r * math.sin(a), rng.uniform(-0.3, 0.3), rng.uniform(0.08, 0.15)))
    inside = np.zeros(np.broadcast(x, y, z).shape, bool)
    for cx, cy, cz, rad in centres:
        inside |= (x - cx) ** 2 + (y - cy) ** 2 + (z - cz) ** 2 < rad * rad
    cyl = x * x + y * y < 0.81
    return np.where(inside, 8.0, np.where(cyl, 0.2, 0.0))


def phantom_fields(wl: Workload, problems: Optional[int] = None, first: int = 0) -> np.ndarray:
    """(S, cell_count) float64 truth fields of problems first .. first+S-1,
    problem p seeded with seed + p (so a slice-sharded rank generates exactly
    its rows of the full stack)."""
    S = wl.problems if problems is None else problems
    spec = wl.spec
    x, y, z = cell_centroids(spec)
    scale = spec.radius()
    volume = spec.mode == GridMode.Volume3D
    out = np.zeros((S, spec.cell_count()))
    for p in range(S):
        rng = np.random.default_rng(wl.seed + first + p)
        if wl.phantom == "lump":
            vals = [lump_value(rng, x / scale, y / scale, zz / scale) for zz in z]
        else:
            shapes = random_shapes(rng, wl, volume)
            vals = [shapes_value(shapes, x / scale, y / scale, zz / scale, volume) for zz in z]
        out[p] = np.concatenate(vals)
    return out


def add_noise(wl: Workload, proj: np.ndarray, seed_offset: int = 7, first: int = 0) -> np.ndarray:
    """Seeded multiplicative noise clipped at zero. proj is
    (S, ...) for problems first .. first+S-1; problem p's noise is seeded
    with seed + 1000003 + seed_offset + p, so shards draw their own rows of
    the full stack's noise."""
    if wl.noise == "none" or wl.noise_level == 0:
        return proj
    out = np.empty_like(proj)
    for p in range(proj.shape[0]):
        rng = np.random.default_rng(wl.seed + 1_000_003 + seed_offset + first + p)
        noisy = proj[p] * (1.0 + wl.noise_level * rng.standard_normal(proj[p].shape))
        out[p] = np.clip(noisy, 0.0, None)
    return out


def counters(cells_per_unit: np.ndarray, proj: np.ndarray, records: int, views: int):
    """U (ray-voxel updates), C (chords traversed) and L (non-skipped lines)
    per sweep, from the reference's own counters (TraceScratch::cells/chords,
    tracer.cpp:198-200): proj is (S, views, lines)."""
    nz = proj.reshape(proj.shape[0], -1) != 0
    U = int((nz * cells_per_unit.reshape(1, -1).astype(np.int64)).sum())
    L = int(nz.sum())
    return U, L
