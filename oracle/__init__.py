"""TEST INFRASTRUCTURE ONLY — CPU oracle for the USPG/USCG MART hot path.

Two checkers, both CPU:

* ``Orc``  — ctypes binding of ``liborc.so``, the plain-C generalized
  restatement in ``uscg_oracle.c`` (ring-law table, decoupled slice count,
  explicit first-view rays, view-angle list).
* ``Ref``  — ctypes binding of ``_ref/libuscg_ref.so``: the UNMODIFIED reference
  library compiled from /root/reference/proj/src (see Makefile) behind
  ``ref_shim.cpp``. Used to pin ``Orc`` bit-exactly on the reference's own
  configurations and as the CPU baseline.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package. The product
(``paper_2208_12964_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libuscg_ref.so")
REF_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u16p = C.POINTER(C.c_uint16)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


def build(ref: bool | None = None) -> None:
    """Compile liborc.so (always) and the reference library when the
    reference sources are present (this container; never on the GPU box)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


class _Grid(C.Structure):
    _fields_ = [
        ("n_rings", C.c_int),
        ("ring_spacing", C.c_double),
        ("n_slices", C.c_int),
        ("slice_height", C.c_double),
        ("volume", C.c_int),
        ("counts", _u32p),
    ]


class _Cache(C.Structure):
    _fields_ = [("lines", C.c_int), ("offsets", _u32p), ("records", C.c_void_p), ("n_records", C.c_uint64)]


REC_DTYPE = np.dtype([("phi_a", "<f8"), ("phi_b", "<f8"), ("slice", "<u2"), ("ring", "<u2")], align=True)


class OrcGrid:
    """Generalized grid: rings, ring spacing, slices, slice height, 2D/3D and a
    sector-count table (None = reference 4(2k-1) law)."""

    def __init__(self, n_rings, ring_spacing, n_slices=1, slice_height=None, volume=False, counts=None):
        self.n_rings = int(n_rings)
        self.ring_spacing = float(ring_spacing)
        self.n_slices = int(n_slices) if volume else 1
        self.slice_height = float(ring_spacing if slice_height is None else slice_height)
        self.volume = bool(volume)
        self.counts = None if counts is None else np.ascontiguousarray(counts, dtype=np.uint32)
        self._c = _Grid(self.n_rings, self.ring_spacing, self.n_slices, self.slice_height,
                        int(self.volume), _ptr(self.counts, _u32p))

    @classmethod
    def of(cls, spec):
        """The generalized grid of a GridSpec-like object (duck-typed)."""
        volume = int(getattr(spec.mode, "value", spec.mode)) == 1
        counts = None if spec.ring_counts is None else np.asarray(spec.ring_counts, np.uint32)
        return cls(spec.rings(), spec.ring_spacing, spec.slices(), spec.slice_height, volume, counts)

    @classmethod
    def reference(cls, n, volume=False):
        """GridSpec::square_2d(n) / cube_3d(n) (include/uscg/grid.hpp:38-43)."""
        return cls(n // 2, 2.0 / n, n if volume else 1, 2.0 / n, volume)

    def ring_counts(self):
        if self.counts is not None:
            return self.counts.copy()
        k = np.arange(1, self.n_rings + 1)
        return (4 * (2 * k - 1)).astype(np.uint32)

    def cells_per_slice(self):
        return int(self.ring_counts().astype(np.int64).sum())

    def cell_count(self):
        return self.cells_per_slice() * self.n_slices


class Orc:
    def __init__(self, path: str = ORC_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.orc_cache_build.argtypes = [C.POINTER(_Grid), C.c_int, _dp, _dp, C.POINTER(_Cache)]
        L.orc_cache_free.argtypes = [C.POINTER(_Cache)]
        L.orc_trace_line.argtypes = [C.POINTER(_Grid), C.POINTER(_Cache), C.c_int, C.c_double, _u32p,
                                     _u32p, _u32p, _u64p]
        L.orc_trace_line.restype = C.c_int64
        L.orc_trace_chord.argtypes = [C.POINTER(_Grid), C.c_void_p, C.c_double, _u32p, C.c_int64]
        L.orc_trace_chord.restype = C.c_int64
        L.orc_project.argtypes = [C.POINTER(_Grid), C.POINTER(_Cache), C.c_int, _dp, _dp, _dp]
        L.orc_project_length.argtypes = [C.POINTER(_Grid), C.c_int, _dp, _dp, C.c_int, _dp, _dp, _dp]
        L.orc_length_lists.argtypes = [C.POINTER(_Grid), C.c_int, _dp, _dp, C.c_int, _dp, _u64p, _u32p, _dp,
                                       C.c_uint64]
        L.orc_length_lists.restype = C.c_uint64
        L.orc_weighted_mart.argtypes = [C.c_uint64, _u64p, _u32p, _dp, _dp, _dp, C.c_double, C.c_double, C.c_int]
        L.orc_weighted_mart.restype = C.c_uint64
        L.orc_reconstruct.argtypes = [C.POINTER(_Grid), C.POINTER(_Cache), C.c_int, _dp, _dp, _dp,
                                      C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp, _u8p]
        L.orc_reconstruct.restype = C.c_int
        L.orc_uspg_to_cg_map.argtypes = [C.c_int, _u32p]
        L.orc_bin_map.argtypes = [C.POINTER(_Grid), C.c_int, _u32p]
        L.orc_field_to_cartesian.argtypes = [C.POINTER(_Grid), C.c_int, _dp, _dp]
        L.orc_rays_flat.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.orc_rays_arc.argtypes = [_dp, _dp, C.c_int, C.c_double, _dp, _dp]
        L.orc_rays_parallel.argtypes = [C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.orc_ring_counts_m1.argtypes = [C.c_int, _u32p]
        L.orc_norm360.argtypes = [C.c_double]
        L.orc_norm360.restype = C.c_double
        L.orc_math.argtypes = [C.c_size_t, _dp, _dp, _dp]
        L.orc_rmse.argtypes = [C.c_size_t, _dp, _dp]
        L.orc_rmse.restype = C.c_double
        L.orc_ssim.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_double]
        L.orc_ssim.restype = C.c_double
        L.orc_cartesian_to_field.argtypes = [C.POINTER(_Grid), C.c_int, _dp, _dp]
        L.orc_cartesian_to_field.restype = C.c_int
        L.orc_sharpness.argtypes = [C.c_int, C.c_int, _dp]
        L.orc_set_update_power.argtypes = [C.c_int]
        L.orc_sharpness.restype = C.c_double

    # -- ray generators -------------------------------------------------
    def rays_flat(self, src, ctr, det_u, det_v, su, sv):
        n = det_u * det_v
        s = np.zeros((n, 3)); d = np.zeros((n, 3))
        self.L.orc_rays_flat(_ptr(np.asarray(src, float), _dp), _ptr(np.asarray(ctr, float), _dp),
                             det_u, det_v, su, sv, _ptr(s, _dp), _ptr(d, _dp))
        return s, d

    def rays_arc(self, src, ctr, det_u, du_deg):
        s = np.zeros((det_u, 3)); d = np.zeros((det_u, 3))
        self.L.orc_rays_arc(_ptr(np.asarray(src, float), _dp), _ptr(np.asarray(ctr, float), _dp),
                            det_u, du_deg, _ptr(s, _dp), _ptr(d, _dp))
        return s, d

    def rays_parallel(self, det_u, su, half_len):
        s = np.zeros((det_u, 3)); d = np.zeros((det_u, 3))
        self.L.orc_rays_parallel(det_u, su, half_len, _ptr(s, _dp), _ptr(d, _dp))
        return s, d

    def rays_for(self, geom):
        """First-view rays of a scan description (duck-typed: source,
        detector_center, det_u, det_v, spacing_u, spacing_v, detector kind
        0 flat / 1 arc / 2 parallel), built by the restatement's own ray
        generators (scan.cpp:27-36 and the M4/M7 seams) — never by the
        product library."""
        kind = int(getattr(geom, "detector", 0))
        src, ctr = tuple(map(float, geom.source)), tuple(map(float, geom.detector_center))
        if kind == 0:
            return self.rays_flat(src, ctr, geom.det_u, geom.det_v, geom.spacing_u, geom.spacing_v)
        if geom.det_v != 1:
            raise ValueError("arc / parallel generators are 2D (det_v == 1)")
        if kind == 1:
            return self.rays_arc(src, ctr, geom.det_u, geom.spacing_u)
        if src[1:] != (0.0, 0.0) or ctr[1:] != (0.0, 0.0) or not src[0] == -ctr[0] or ctr[0] <= 0:
            raise ValueError("the parallel generator is restated for an on-axis beam centred on the origin")
        return self.rays_parallel(geom.det_u, geom.spacing_u, ctr[0])

    def ring_counts_m1(self, n_rings):
        out = np.zeros(n_rings, np.uint32)
        self.L.orc_ring_counts_m1(n_rings, _ptr(out, _u32p))
        return out

    def norm360(self, x):
        return self.L.orc_norm360(float(x))

    # -- cache / trace -----------------------------------------------------
    def weighted_mart(self, offsets, idx, w, proj, beta=0.4, sweeps=5, f_init=1.0, p_floor=0.0, cells=None):
        """weighted_update + the loop of cartesian_mart_stored (siddon.cpp:141-154,
        185-209) over (voxel, length) lists: (field f64 [cells], clamps)"""
        off = np.ascontiguousarray(offsets, np.uint64)
        ii = np.ascontiguousarray(idx, np.uint32)
        ww = np.ascontiguousarray(w, np.float64)
        pp = np.ascontiguousarray(proj, np.float64).reshape(-1)
        assert pp.size == off.size - 1
        field = np.full(int(cells), float(f_init))
        clamps = int(self.L.orc_weighted_mart(pp.size, _ptr(off, _u64p), _ptr(ii, _u32p), _ptr(ww, _dp),
                                              _ptr(pp, _dp), _ptr(field, _dp), beta, p_floor, sweeps))
        return field, clamps

    def cache(self, grid: OrcGrid, src, det):
        return OrcCache(self, grid, src, det)

    def field_to_cartesian(self, grid: OrcGrid, field, npix):
        f = np.ascontiguousarray(field, dtype=np.float64)
        out = np.zeros((grid.n_slices, npix, npix))
        self.L.orc_field_to_cartesian(C.byref(grid._c), npix, _ptr(f, _dp), _ptr(out, _dp))
        return out

    def uspg_to_cg_map(self, n):
        out = np.zeros(n * n, np.uint32)
        self.L.orc_uspg_to_cg_map(n, _ptr(out, _u32p))
        return out

    def cartesian_to_field(self, grid: OrcGrid, images, npix):
        """cartesian_to_field (reference law): images (slices, npix, npix) -> cell_count f64"""
        im = np.ascontiguousarray(images, dtype=np.float64)
        out = np.zeros(grid.cell_count())
        if self.L.orc_cartesian_to_field(C.byref(grid._c), npix, _ptr(im, _dp), _ptr(out, _dp)) != 0:
            raise ValueError("slice shape does not match the grid")
        return out

    def sharpness(self, img):
        a = np.ascontiguousarray(img, float)
        return self.L.orc_sharpness(a.shape[0], a.shape[1], _ptr(a, _dp))

    def bin_map(self, grid: OrcGrid, npix):
        out = np.zeros(npix * npix, np.uint32)
        self.L.orc_bin_map(C.byref(grid._c), npix, _ptr(out, _u32p))
        return out

    def rmse(self, a, b):
        a = np.ascontiguousarray(a, float).ravel(); b = np.ascontiguousarray(b, float).ravel()
        return self.L.orc_rmse(a.size, _ptr(a, _dp), _ptr(b, _dp))

    def math(self, x, y):
        """glibc atan2(y, x), hypot(x, y), azimuth_deg(x, y): (n, 3)."""
        x = np.ascontiguousarray(x, float).ravel(); y = np.ascontiguousarray(y, float).ravel()
        out = np.zeros((x.size, 3))
        self.L.orc_math(x.size, _ptr(x, _dp), _ptr(y, _dp), _ptr(out, _dp))
        return out

    def ssim(self, a, b, dynamic_range=-1.0):
        a = np.ascontiguousarray(a, float); b = np.ascontiguousarray(b, float)
        return self.L.orc_ssim(a.shape[0], a.shape[1], _ptr(a, _dp), _ptr(b, _dp), dynamic_range)


class OrcCache:
    """orc_cache (precompute_first_view direct build) + trace/project/reconstruct."""

    def __init__(self, orc: Orc, grid: OrcGrid, src, det):
        self.orc, self.grid = orc, grid
        self.src = np.ascontiguousarray(src, dtype=np.float64)
        self.det = np.ascontiguousarray(det, dtype=np.float64)
        self.lines = self.src.shape[0]
        self._c = _Cache()
        orc.L.orc_cache_build(C.byref(grid._c), self.lines, _ptr(self.src, _dp), _ptr(self.det, _dp),
                              C.byref(self._c))
        n = int(self._c.n_records)
        self.offsets = np.ctypeslib.as_array(self._c.offsets, shape=(self.lines + 1,)).copy()
        if n:
            buf = (C.c_char * (n * REC_DTYPE.itemsize)).from_address(self._c.records)
            self.records = np.frombuffer(bytes(buf), dtype=REC_DTYPE).copy()
        else:
            self.records = np.zeros(0, REC_DTYPE)
        self._stamp = np.zeros(grid.cell_count(), np.uint32)
        self._gen = np.zeros(1, np.uint32)
        self._out = np.zeros(max(grid.cell_count(), 1), np.uint32)

    def __del__(self):
        try:
            self.orc.L.orc_cache_free(C.byref(self._c))
        except Exception:
            pass

    def trace_line(self, line, theta_deg):
        chords = np.zeros(1, np.uint64)
        n = self.orc.L.orc_trace_line(C.byref(self.grid._c), C.byref(self._c), int(line), float(theta_deg),
                                      _ptr(self._stamp, _u32p), _ptr(self._gen, _u32p),
                                      _ptr(self._out, _u32p), _ptr(chords, _u64p))
        return self._out[:n].copy()

    def project(self, thetas, field):
        th = np.ascontiguousarray(thetas, float)
        f = np.ascontiguousarray(field, float)
        out = np.zeros((th.size, self.lines))
        self.orc.L.orc_project(C.byref(self.grid._c), C.byref(self._c), th.size, _ptr(th, _dp),
                               _ptr(f, _dp), _ptr(out, _dp))
        return out

    def project_length(self, thetas, field):
        th = np.ascontiguousarray(thetas, float)
        f = np.ascontiguousarray(field, float)
        out = np.zeros((th.size, self.lines))
        self.orc.L.orc_project_length(C.byref(self.grid._c), self.lines, _ptr(self.src, _dp),
                                      _ptr(self.det, _dp), th.size, _ptr(th, _dp), _ptr(f, _dp),
                                      _ptr(out, _dp))
        return out

    def length_lists(self, thetas):
        """The LengthWeighted model's (voxel, chord length) lists per (view,
        line), a cell's pieces merged: (offsets u64 [views*lines+1], idx u32, len f64)"""
        th = np.ascontiguousarray(thetas, float)
        off = np.zeros(th.size * self.lines + 1, np.uint64)
        args = (C.byref(self.grid._c), self.lines, _ptr(self.src, _dp), _ptr(self.det, _dp), th.size,
                _ptr(th, _dp), _ptr(off, _u64p))
        n = int(self.orc.L.orc_length_lists(*args, None, None, 0))
        idx = np.zeros(max(n, 1), np.uint32)
        ln = np.zeros(max(n, 1), np.float64)
        got = int(self.orc.L.orc_length_lists(*args, _ptr(idx, _u32p), _ptr(ln, _dp), n))
        assert got == n
        return off, idx[:n], ln[:n]

    def weighted_mart(self, offsets, idx, w, proj, beta=0.4, sweeps=5, f_init=1.0, p_floor=0.0):
        """Orc.weighted_mart on this grid's cells"""
        return self.orc.weighted_mart(offsets, idx, w, proj, beta, sweeps, f_init, p_floor,
                                      cells=self.grid.cell_count())

    def reconstruct(self, thetas, proj, init=None, beta=0.4, tolerance=1e-6, max_sweeps=100,
                    f_init=1.0, p_floor=0.0, power=False):
        """orc_reconstruct; power=True: the (m/p)^beta update (the device's
        USCG_UPDATE_POWER), not a reference behaviour"""
        th = np.ascontiguousarray(thetas, float)
        p = np.ascontiguousarray(proj, float)
        if init is None:
            field = np.full(self.grid.cell_count(), float(f_init))
        else:
            field = np.array(init, dtype=np.float64, copy=True)
        report = np.zeros(6)
        residuals = np.zeros(max_sweeps)
        crossed = np.zeros(self.grid.cell_count(), np.uint8)
        self.orc.L.orc_set_update_power(int(bool(power)))
        rc = self.orc.L.orc_reconstruct(C.byref(self.grid._c), C.byref(self._c), th.size, _ptr(th, _dp),
                                        _ptr(p, _dp), _ptr(field, _dp), beta, tolerance, max_sweeps,
                                        p_floor, _ptr(report, _dp), _ptr(residuals, _dp),
                                        _ptr(crossed, _u8p))
        self.orc.L.orc_set_update_power(0)
        if rc != 0:
            raise ValueError("invalid reconstruction input")
        sweeps = int(report[0])
        rep = dict(sweeps=sweeps, converged=bool(report[1]), all_zero_data=bool(report[2]),
                   zero_measurement_skips=int(report[3]), factor_clamps=int(report[4]),
                   updates=int(report[5]),
                   sweep_residuals=residuals[:sweeps].copy() if tolerance > 0 else np.zeros(0),
                   crossed=crossed)
        return field, rep


class Ref:
    """The unmodified reference library (oracle/_ref/libuscg_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref needs /root/reference)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_tracer_create.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_int, C.c_int,
                                        C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p)]
        L.ref_tracer_destroy.argtypes = [C.c_void_p]
        L.ref_cache_records.argtypes = [C.c_void_p]
        L.ref_cache_records.restype = C.c_uint64
        L.ref_cache_bytes.argtypes = [C.c_void_p]
        L.ref_cache_bytes.restype = C.c_uint64
        L.ref_cache_lines.argtypes = [C.c_void_p]
        L.ref_cache_export.argtypes = [C.c_void_p, _u32p, _dp, _dp, _u16p, _u16p]
        L.ref_trace_line.argtypes = [C.c_void_p, C.c_int, C.c_double, _u32p, C.c_int64, _u64p, _u64p]
        L.ref_trace_line.restype = C.c_int64
        L.ref_trace_chord.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                      C.c_int, C.c_int, C.c_double, _u32p, C.c_int64]
        L.ref_trace_chord.restype = C.c_int64
        L.ref_project_binary.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_project_length.argtypes = [C.c_void_p, _dp, _dp]
        _sp = C.POINTER(C.c_char_p)
        L.ref_write_field.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_int, _dp, _sp, _sp, C.c_int]
        L.ref_write_projections.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp,
                                            _dp, _sp, _sp, C.c_int]
        L.ref_write_pgm16.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp, C.c_double, C.c_double, _sp, _sp, C.c_int]
        L.ref_read_pgm16.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, C.c_longlong]
        L.ref_cartesian_system.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_int, C.c_int,
                                           C.c_double, C.c_double, C.c_int, _u64p, _u32p, _dp, _u64p]
        L.ref_cartesian_mart.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_int, C.c_int,
                                         C.c_double, C.c_double, C.c_int, _dp, C.c_double, C.c_int, C.c_double,
                                         C.c_int, _dp, _dp]
        L.ref_reconstruct.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_double, C.c_int, C.c_double,
                                      C.c_double, _dp, _dp, _dp, _u8p]
        L.ref_mart_update_line.argtypes = [C.c_int, _dp, C.c_int64, _u32p, C.c_int64, C.c_double,
                                           C.c_double, C.c_double]
        L.ref_uspg_to_cg_map.argtypes = [C.c_int, _u32p]
        L.ref_field_to_cartesian.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp]
        L.ref_rmse.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.ref_rmse.restype = C.c_double
        L.ref_ssim.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_double]
        L.ref_ssim.restype = C.c_double
        L.ref_phantom.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _dp]
        L.ref_cartesian_to_field.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ref_sharpness.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.ref_intensity_profile.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp]

    def check(self, rc):
        if rc == 1:
            raise ValueError(self.L.ref_last_error().decode())
        if rc == 2:
            raise ArithmeticError(self.L.ref_last_error().decode())
        if rc:
            raise RuntimeError(self.L.ref_last_error().decode())

    def tracer(self, n, volume, src, ctr, det_u, det_v, su, sv, views, quarter=False, threads=1):
        return RefTracer(self, n, volume, src, ctr, det_u, det_v, su, sv, views, quarter, threads)

    def trace_chord(self, n, volume, phi_a, phi_b, slice_, ring, theta):
        out = np.zeros(4096, np.uint32)
        k = self.L.ref_trace_chord(n, 2.0 / n, 2.0 / n, int(volume), phi_a, phi_b, slice_, ring, theta,
                                   _ptr(out, _u32p), out.size)
        return out[:k].copy()

    def uspg_to_cg_map(self, n):
        out = np.zeros(n * n, np.uint32)
        self.check(self.L.ref_uspg_to_cg_map(n, _ptr(out, _u32p)))
        return out

    def field_to_cartesian(self, n, volume, field):
        f = np.ascontiguousarray(field, float)
        slices = n if volume else 1
        out = np.zeros((slices, n, n))
        self.check(self.L.ref_field_to_cartesian(n, 2.0 / n, 2.0 / n, int(volume), _ptr(f, _dp), _ptr(out, _dp)))
        return out

    def cartesian_to_field(self, n, volume, images, img_n=None):
        im = np.ascontiguousarray(images, float)
        img_n = n if img_n is None else img_n
        out = np.zeros((n if volume else 1) * n * n)
        self.check(self.L.ref_cartesian_to_field(n, 2.0 / n, 2.0 / n, int(volume), img_n, _ptr(im, _dp),
                                                 _ptr(out, _dp)))
        return out

    def sharpness(self, img):
        a = np.ascontiguousarray(img, float)
        out = np.zeros(1)
        self.check(self.L.ref_sharpness(a.shape[0], a.shape[1], _ptr(a, _dp), _ptr(out, _dp)))
        return float(out[0])

    def intensity_profile(self, img, row):
        a = np.ascontiguousarray(img, float)
        out = np.zeros(a.shape[1])
        self.check(self.L.ref_intensity_profile(a.shape[0], a.shape[1], _ptr(a, _dp), row, _ptr(out, _dp)))
        return out

    def cartesian_system(self, n, volume, src, ctr, det_u, det_v, su, sv, views):
        """precompute_cartesian_system on CartesianSpec::like(reference grid n):
        (offsets u64 [rows+1], idx u32, weight f64)"""
        s3, c3 = np.ascontiguousarray(src, float), np.ascontiguousarray(ctr, float)
        r = h = 2.0 / n
        ent = np.zeros(1, np.uint64)
        args = (n, r, h, int(volume), _ptr(s3, _dp), _ptr(c3, _dp), det_u, det_v, su, sv, views)
        self.check(self.L.ref_cartesian_system(*args, None, None, None, _ptr(ent, _u64p)))
        rows = views * det_u * det_v
        off = np.zeros(rows + 1, np.uint64)
        idx = np.zeros(int(ent[0]), np.uint32)
        w = np.zeros(int(ent[0]))
        self.check(self.L.ref_cartesian_system(*args, _ptr(off, _u64p), _ptr(idx, _u32p), _ptr(w, _dp), _ptr(ent, _u64p)))
        return off, idx, w

    def cartesian_mart(self, n, volume, src, ctr, det_u, det_v, su, sv, views, proj, beta=0.4, sweeps=5,
                       f_init=1.0, stored=True):
        """cartesian_mart_stored / cartesian_mart_otf: (values, seconds)"""
        s3, c3 = np.ascontiguousarray(src, float), np.ascontiguousarray(ctr, float)
        p = np.ascontiguousarray(proj, float)
        cells = n * n * (n if volume else 1)
        out = np.zeros(cells)
        sec = np.zeros(1)
        r = h = 2.0 / n
        self.check(self.L.ref_cartesian_mart(n, r, h, int(volume), _ptr(s3, _dp), _ptr(c3, _dp), det_u, det_v, su, sv,
                                             views, _ptr(p, _dp), beta, sweeps, f_init, int(stored), _ptr(out, _dp),
                                             _ptr(sec, _dp)))
        return out, float(sec[0])

    def phantom(self, n, volume):
        out = np.zeros((n if volume else 1) * n * n)
        self.check(self.L.ref_phantom(n, 2.0 / n, 2.0 / n, int(volume), 1 if volume else 0, _ptr(out, _dp)))
        return out

    def rmse(self, a, b):
        a = np.ascontiguousarray(a, float); b = np.ascontiguousarray(b, float)
        return self.L.ref_rmse(a.shape[0], a.shape[1], _ptr(a, _dp), _ptr(b, _dp))

    def ssim(self, a, b, dynamic_range=-1.0):
        a = np.ascontiguousarray(a, float); b = np.ascontiguousarray(b, float)
        return self.L.ref_ssim(a.shape[0], a.shape[1], _ptr(a, _dp), _ptr(b, _dp), dynamic_range)


def _kv(side):
    """parallel (keys, values) C string arrays of a dict / list of pairs"""
    items = list(side.items()) if isinstance(side, dict) else list(side or [])
    keys = (C.c_char_p * max(1, len(items)))(*[k.encode() for k, _ in items])
    vals = (C.c_char_p * max(1, len(items)))(*[str(v).encode() for _, v in items])
    return keys, vals, len(items)


class RefIO:
    """The reference's file writers / PGM reader (proj/src/io.cpp) through the shim."""

    def __init__(self, ref: "Ref"):
        self.ref = ref

    def write_field(self, path, n, r, h, volume, values, side=None):
        v = np.ascontiguousarray(values, float)
        self.ref.check(self.ref.L.ref_write_field(str(path).encode(), n, r, h, int(volume), _ptr(v, _dp), *_kv(side)))

    def write_projections(self, path, views, det_u, det_v, su, sv, src, ctr, data, side=None):
        d = np.ascontiguousarray(data, float)
        s3 = np.ascontiguousarray(src, float)
        c3 = np.ascontiguousarray(ctr, float)
        self.ref.check(self.ref.L.ref_write_projections(str(path).encode(), views, det_u, det_v, su, sv, _ptr(s3, _dp),
                                                        _ptr(c3, _dp), _ptr(d, _dp), *_kv(side)))

    def write_pgm16(self, path, img, wmin, wmax, side=None):
        im = np.ascontiguousarray(img, float)
        self.ref.check(self.ref.L.ref_write_pgm16(str(path).encode(), im.shape[0], im.shape[1], _ptr(im, _dp), wmin,
                                                  wmax, *_kv(side)))

    def read_pgm16(self, path, cap=1 << 24):
        out = np.zeros(cap)
        rows, cols = C.c_int(), C.c_int()
        self.ref.check(self.ref.L.ref_read_pgm16(str(path).encode(), C.byref(rows), C.byref(cols), _ptr(out, _dp), cap))
        return out[: rows.value * cols.value].reshape(rows.value, cols.value)


class RefTracer:
    def __init__(self, ref: Ref, n, volume, src, ctr, det_u, det_v, su, sv, views, quarter, threads):
        self.ref = ref
        self.n, self.volume, self.views = n, bool(volume), views
        self.lines = det_u * det_v
        self.cells = (n if volume else 1) * n * n
        h = C.c_void_p()
        s = np.asarray(src, float); c = np.asarray(ctr, float)
        ref.check(ref.L.ref_tracer_create(n, 2.0 / n, 2.0 / n, int(volume), _ptr(s, _dp), _ptr(c, _dp),
                                          det_u, det_v, su, sv, views, int(quarter), threads, C.byref(h)))
        self.h = h
        self._out = np.zeros(self.cells, np.uint32)

    def __del__(self):
        try:
            self.ref.L.ref_tracer_destroy(self.h)
        except Exception:
            pass

    def cache(self):
        n = int(self.ref.L.ref_cache_records(self.h))
        off = np.zeros(self.lines + 1, np.uint32)
        pa = np.zeros(n); pb = np.zeros(n)
        sl = np.zeros(n, np.uint16); rg = np.zeros(n, np.uint16)
        self.ref.L.ref_cache_export(self.h, _ptr(off, _u32p), _ptr(pa, _dp), _ptr(pb, _dp),
                                    _ptr(sl, _u16p), _ptr(rg, _u16p))
        return off, pa, pb, sl, rg

    def cache_bytes(self):
        return int(self.ref.L.ref_cache_bytes(self.h))

    def trace_line(self, line, theta):
        n = self.ref.L.ref_trace_line(self.h, line, theta, _ptr(self._out, _u32p), self._out.size, None, None)
        return self._out[:n].copy()

    def project(self, field):
        f = np.ascontiguousarray(field, float)
        out = np.zeros((self.views, self.lines))
        self.ref.check(self.ref.L.ref_project_binary(self.h, _ptr(f, _dp), _ptr(out, _dp)))
        return out

    def project_length(self, field):
        f = np.ascontiguousarray(field, float)
        out = np.zeros((self.views, self.lines))
        self.ref.check(self.ref.L.ref_project_length(self.h, _ptr(f, _dp), _ptr(out, _dp)))
        return out

    def reconstruct(self, proj, init=None, beta=0.4, tolerance=1e-6, max_sweeps=100, f_init=1.0, p_floor=0.0):
        p = np.ascontiguousarray(proj, float)
        out = np.zeros(self.cells)
        report = np.zeros(6)
        residuals = np.zeros(max_sweeps)
        crossed = np.zeros(self.cells, np.uint8)
        i = None if init is None else np.ascontiguousarray(init, float)
        self.ref.check(self.ref.L.ref_reconstruct(self.h, _ptr(p, _dp), _ptr(i, _dp), beta, tolerance, max_sweeps,
                                                  f_init, p_floor, _ptr(out, _dp), _ptr(report, _dp),
                                                  _ptr(residuals, _dp), _ptr(crossed, _u8p)))
        sweeps = int(report[0])
        rep = dict(sweeps=sweeps, converged=bool(report[1]), all_zero_data=bool(report[2]), seconds=report[3],
                   zero_measurement_skips=int(report[4]), factor_clamps=int(report[5]),
                   sweep_residuals=residuals[:sweeps].copy() if tolerance > 0 else np.zeros(0),
                   crossed=crossed)
        return out, rep


def ref_thetas(views, span=360.0):
    """View angles i*span/p (solver.cpp:101,116 uses norm360(view*360/p))."""
    step = span / views
    return np.array([view * step for view in range(views)], dtype=np.float64)
