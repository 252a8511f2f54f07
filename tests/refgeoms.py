"""Reference test geometries (the ones the reference's own tests use) and
helpers to express them on both sides: the reference library (oracle/_ref),
the C restatement (oracle) and the device path (paper_2208_12964_b200)."""
import numpy as np

# fan_geometry / cone_geometry of proj/tests/test_tracer.cpp:15-36,
# fan_table1 / cone_table1 of proj/tests/acceptance.cpp:33-56
REF_GEOMS = {
    "fan32": dict(n=32, volume=False, src=(-8, 0, 0), ctr=(8, 0, 0), du=25, dv=1, su=0.05, sv=0.0, views=12),
    "fan64q": dict(n=64, volume=False, src=(-8, 0, 0), ctr=(8, 0, 0), du=33, dv=1, su=0.05, sv=0.0, views=10),
    "fan16": dict(n=16, volume=False, src=(-8, 0, 0), ctr=(8, 0, 0), du=21, dv=1, su=0.2, sv=0.0, views=20),
    "cone16": dict(n=16, volume=True, src=(-3, 0, 0), ctr=(10, 0, 0), du=9, dv=9, su=0.1, sv=0.1, views=8),
    "cone32": dict(n=32, volume=True, src=(-3, 0, 0), ctr=(10, 0, 0), du=17, dv=17, su=0.1, sv=0.1, views=10),
    "fan128": dict(n=128, volume=False, src=(-8, 0, 0), ctr=(8, 0, 0), du=101, dv=1, su=0.05, sv=0.0, views=50),
    "cone12": dict(n=12, volume=True, src=(-3, 0, 0), ctr=(10, 0, 0), du=15, dv=15, su=1.0, sv=1.0, views=10),
    "cone32w": dict(n=32, volume=True, src=(-3, 0, 0), ctr=(10, 0, 0), du=21, dv=21, su=0.6, sv=0.6, views=20),
}


def ref_tracer(ref, g, quarter=False):
    return ref.tracer(g["n"], g["volume"], g["src"], g["ctr"], g["du"], g["dv"], g["su"], g["sv"], g["views"],
                      quarter)


def ub_spec_geom(ub, g):
    spec = ub.GridSpec.cube_3d(g["n"]) if g["volume"] else ub.GridSpec.square_2d(g["n"])
    geom = ub.ScanGeometry(source=g["src"], detector_center=g["ctr"], det_u=g["du"], det_v=g["dv"],
                           spacing_u=g["su"], spacing_v=g["sv"], views=g["views"])
    return spec, geom


def cache_from_ref(ub, rt):
    off, pa, pb, sl, rg = rt.cache()
    return ub.FirstViewCache(off, pa, pb, sl, rg)


def ulp_diff(a, b):
    ai = np.asarray(a, np.float64).view(np.int64)
    bi = np.asarray(b, np.float64).view(np.int64)
    return np.abs(ai - bi)


def thetas(views, span=360.0):
    step = span / views
    return np.array([v * step for v in range(views)])
