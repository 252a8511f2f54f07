"""Generate the golden fixtures of tests/golden/ from the UNMODIFIED reference
library (oracle/_ref/libuscg_ref.so, built from /root/reference by
oracle/Makefile). Run in the build container (the GPU box has no
/root/reference); the fixtures are small and committed.

    python tests/golden/make_golden.py

Each fixture pins one reference behaviour the oracle restatement and the
device path must reproduce:
  cache_<geom>.npz   FirstViewCache offsets / phi_a / phi_b / slice / ring
  trace_<geom>.npz   Tracer::trace_line for a subset of (view, line), CSR
  proj_<geom>.npz    generate_projections (binary) of a seeded random field
  recon_<geom>.npz   reconstruct (fp64 field, residuals, counters, crossed)
  map_<n>.npz        uspg_to_cg_map(n)
  images.npz         cartesian_to_field of seeded rasters (2D n=16, 3D n=8),
                     sharpness of seeded / structured images and
                     intensity_profile rows (proj/src/phantom.cpp:165-180,
                     proj/src/metrics.cpp:138-159)
  kat.json           worked examples of proj/tests/test_tracer.cpp:60-98 and
                     the solver arithmetic of proj/tests/test_solver.cpp:68-113
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from refgeoms import REF_GEOMS, ref_tracer, thetas  # noqa: E402

GOLDEN = ["fan32", "fan16", "cone16", "cone12"]


def main():
    oracle.build(ref=True)
    ref = oracle.Ref()
    for name in GOLDEN:
        g = REF_GEOMS[name]
        rt = ref_tracer(ref, g)
        off, pa, pb, sl, rg = rt.cache()
        np.savez_compressed(os.path.join(HERE, f"cache_{name}.npz"), offsets=off, phi_a=pa, phi_b=pb, slice=sl,
                            ring=rg, bytes=np.array([rt.cache_bytes()]))
        th = thetas(g["views"])
        rng = np.random.default_rng(11)
        picks = [(int(v), int(l)) for v, l in zip(rng.integers(0, g["views"], 64),
                                                  rng.integers(0, g["du"] * g["dv"], 64))]
        lists = [rt.trace_line(l, th[v]) for v, l in picks]
        pos = np.concatenate([[0], np.cumsum([x.size for x in lists])]).astype(np.uint32)
        np.savez_compressed(os.path.join(HERE, f"trace_{name}.npz"), picks=np.array(picks, np.int32), pos=pos,
                            idx=np.concatenate(lists).astype(np.uint32))
        cells = (g["n"] if g["volume"] else 1) * g["n"] * g["n"]
        f = np.random.default_rng(7).uniform(0.2, 3.0, cells)
        p = rt.project(f)
        np.savez_compressed(os.path.join(HERE, f"proj_{name}.npz"), field=f, proj=p)
        rec, rep = rt.reconstruct(p, beta=0.4, tolerance=1e-30, max_sweeps=3)
        np.savez_compressed(os.path.join(HERE, f"recon_{name}.npz"), field=rec,
                            residuals=rep["sweep_residuals"], crossed=rep["crossed"],
                            counters=np.array([rep["sweeps"], rep["zero_measurement_skips"],
                                               rep["factor_clamps"]]))
    for n in (2, 4, 16, 64):
        np.savez_compressed(os.path.join(HERE, f"map_{n}.npz"), map=ref.uspg_to_cg_map(n))
    rng = np.random.default_rng(21)
    im2 = rng.uniform(0, 2, (1, 16, 16))
    im3 = rng.uniform(0, 2, (8, 8, 8))
    sharp_imgs = [rng.uniform(0, 1, (9, 13)), np.add.outer(np.arange(6.0), 0.5 * np.arange(4.0)),
                  np.indices((8, 8)).sum(axis=0) % 2 * 1.0, np.full((2, 2), 3.0), rng.normal(0, 1, (2, 7))]
    sharp = np.array([ref.sharpness(x) for x in sharp_imgs])
    packed = np.concatenate([x.ravel() for x in sharp_imgs])
    shapes = np.array([x.shape for x in sharp_imgs], np.int32)
    np.savez_compressed(os.path.join(HERE, "images.npz"), im2=im2, field2=ref.cartesian_to_field(16, False, im2),
                        im3=im3, field3=ref.cartesian_to_field(8, True, im3), sharp_pixels=packed,
                        sharp_shapes=shapes, sharpness=sharp,
                        profile=ref.intensity_profile(sharp_imgs[0], 4))
    kat = {"trace_chord": []}
    for rec, theta in [((95.0, 40.0, 0, 2), 0.0), ((350.0, 10.0, 0, 2), 0.0), ((65.0, 10.0, 0, 2), 30.0),
                       ((10.0, 190.0, 0, 2), 0.0), ((45.0, 45.0, 0, 2), 0.0)]:
        kat["trace_chord"].append({"n": 8, "volume": False, "rec": rec, "theta": theta,
                                   "cells": ref.trace_chord(8, False, *rec, theta).tolist()})
    kat["trace_chord"].append({"n": 8, "volume": True, "rec": (95.0, 40.0, 3, 2), "theta": 0.0,
                               "cells": ref.trace_chord(8, True, 95.0, 40.0, 3, 2, 0.0).tolist()})
    with open(os.path.join(HERE, "kat.json"), "w") as fh:
        json.dump(kat, fh, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
