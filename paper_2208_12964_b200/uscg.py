"""Python mirror of the reference's reconstruction API over the uscg_b200 C ABI.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/uscg/*.hpp) so that code and tests written
against ``uscg::`` read the same here:

====================================  ======================================================
reference (C++)                       here
====================================  ======================================================
``GridSpec`` grid.hpp:21-44            :class:`GridSpec` (+ ``ring_counts``, ``n_slices``)
``ScanGeometry`` scan.hpp:21-41        :class:`ScanGeometry` (+ ``detector``, ``view_angles``)
``Tracer`` tracer.hpp:85-105           :class:`Tracer` (device-resident first-view cache)
``FirstViewCache`` tracer.hpp:18-39    :meth:`Tracer.cache`
``Field`` / ``ProjectionSet``          :class:`Field` / :class:`ProjectionSet`
``SolverConfig`` / ``ReconReport``     :class:`SolverConfig` / :class:`ReconReport`
``reconstruct`` solver.hpp:78-79       :func:`reconstruct`
``reconstruct_from`` solver.hpp:82-83  :func:`reconstruct_from`
``generate_projections`` phantom.hpp   :func:`generate_projections` (Binary, LengthWeighted)
``field_to_cartesian`` phantom.hpp:56  :func:`field_to_cartesian`
``uspg_to_cg_map`` grid.hpp:84         :func:`uspg_to_cg_map`
====================================  ======================================================

``std::invalid_argument`` surfaces as :class:`InvalidArgument` (a ValueError)
and ``std::domain_error`` as :class:`DomainError` (an ArithmeticError).

Every compute call runs the CUDA kernels of ``lib/libuscg_b200.so``; there is
no CPU fallback. Without the library or without an sm_100 device the calls
raise :class:`NoDevice` / ``OSError``.
"""
from __future__ import annotations

import atexit
import ctypes as C
import enum
import os
import weakref
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np

from . import _build

# ---------------------------------------------------------------------------
# errors
# ---------------------------------------------------------------------------


class UscgError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class DomainError(ArithmeticError):
    """std::domain_error in the reference."""


class NoDevice(UscgError):
    """No usable sm_100 device: the path has no CPU fallback."""


DEVICE_POINTERS = 1
LAYOUT_INTERLEAVED = 2
MODEL_LENGTH = 4  # uscg_project: ForwardModel::LengthWeighted
UPDATE_POWER = 8  # uscg_reconstruct: (m/p)^beta update (extension; the reference is linear)

# ---------------------------------------------------------------------------
# ctypes structures (include/uscg_b200.h)
# ---------------------------------------------------------------------------
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_u16p = C.POINTER(C.c_uint16)
_u8p = C.POINTER(C.c_uint8)


class _Grid(C.Structure):
    _fields_ = [("n_rings", C.c_int32), ("ring_spacing", C.c_double), ("n_slices", C.c_int32),
                ("slice_height", C.c_double), ("volume", C.c_int32), ("ring_counts", _u32p)]


class _Scan(C.Structure):
    _fields_ = [("detector", C.c_int32), ("source", C.c_double * 3), ("detector_center", C.c_double * 3),
                ("det_u", C.c_int32), ("det_v", C.c_int32), ("spacing_u", C.c_double),
                ("spacing_v", C.c_double), ("views", C.c_int32), ("view_angles_deg", _dp)]


class _Cfg(C.Structure):
    _fields_ = [("beta", C.c_double), ("tolerance", C.c_double), ("max_sweeps", C.c_int32),
                ("f_init", C.c_double), ("p_floor", C.c_double)]


class _Report(C.Structure):
    _fields_ = [("sweeps", C.c_int32), ("converged", C.c_int32), ("all_zero_data", C.c_int32),
                ("seconds", C.c_double), ("zero_measurement_skips", C.c_uint64),
                ("factor_clamps", C.c_uint64), ("updates", C.c_uint64), ("sweep_residuals", _dp),
                ("crossed", _u8p)]


class _Cart(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("voxel", C.c_double),
                ("origin", C.c_double * 3)]


class _Info(C.Structure):
    _fields_ = [("lines", C.c_int32), ("views", C.c_int32), ("n_rings", C.c_int32), ("n_slices", C.c_int32),
                ("records", C.c_uint64), ("cells_per_slice", C.c_uint64), ("cell_count", C.c_uint64),
                ("cache_bytes", C.c_uint64), ("max_line_records", C.c_int32), ("max_line_cells", C.c_int32),
                ("cells_per_sweep", C.c_uint64), ("chords_per_sweep", C.c_uint64), ("levels", C.c_int32),
                ("generator_ms", C.c_double), ("executor", C.c_int32), ("wave_requirements", C.c_uint64),
                ("wave_build_s", C.c_double), ("executor_bytes", C.c_uint64), ("wave_ctas", C.c_int32)]


EXPORTS = [
    "uscg_last_error", "uscg_version", "uscg_launch_count", "uscg_ctx_create", "uscg_ctx_destroy",
    "uscg_ctx_set_stream", "uscg_ctx_synchronize", "uscg_first_view_rays", "uscg_tracer_create",
    "uscg_tracer_create_from_rays", "uscg_tracer_import_cache", "uscg_tracer_destroy",
    "uscg_tracer_get_info", "uscg_tracer_export_cache", "uscg_trace_line", "uscg_trace_counts",
    "uscg_trace_checksums", "uscg_tracer_export_schedule", "uscg_tracer_copy_cache",
    "uscg_tracer_import_cache_keys",
    "uscg_tracer_build_schedule", "uscg_tracer_export_successors", "uscg_reconstruct_batch", "uscg_problem_stride", "uscg_project", "uscg_reconstruct",
    "uscg_resample", "uscg_uspg_to_cg_map", "uscg_diag_math", "uscg_schedule_build", "uscg_image_metrics",
    "uscg_cartesian_like", "uscg_csystem_create", "uscg_csystem_info", "uscg_csystem_export",
    "uscg_csystem_reconstruct", "uscg_csystem_destroy", "uscg_tracer_length_system", "uscg_tracer_export_wave",
    "uscg_cartesian_to_field", "uscg_image_sharpness", "uscg_intensity_profile",
]

_lib = None


def library_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load lib/libuscg_b200.so (building it in-tree when nvcc is available)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if not os.path.exists(path) or _build._stale():
        if not build_if_missing:
            raise OSError(f"{path} is missing: build it with `python -m paper_2208_12964_b200._build`")
        _build.build()
    L = C.CDLL(path)
    vp = C.c_void_p
    L.uscg_last_error.restype = C.c_char_p
    L.uscg_version.restype = C.c_char_p
    L.uscg_launch_count.restype = C.c_uint64
    L.uscg_ctx_create.argtypes = [C.c_int32, C.POINTER(vp)]
    L.uscg_ctx_destroy.argtypes = [vp]
    L.uscg_ctx_set_stream.argtypes = [vp, vp]
    L.uscg_ctx_synchronize.argtypes = [vp]
    L.uscg_first_view_rays.argtypes = [C.POINTER(_Scan), _dp, _dp]
    L.uscg_tracer_create.argtypes = [vp, C.POINTER(_Grid), C.POINTER(_Scan), C.c_int32, C.POINTER(vp)]
    L.uscg_tracer_create_from_rays.argtypes = [vp, C.POINTER(_Grid), C.c_int32, _dp, _dp, C.c_int32, _dp,
                                               C.POINTER(vp)]
    L.uscg_tracer_import_cache.argtypes = [vp, C.POINTER(_Grid), C.c_int32, _u32p, C.c_uint64, _dp, _dp, _u16p,
                                           _u16p, C.c_int32, _dp, C.POINTER(vp)]
    L.uscg_tracer_destroy.argtypes = [vp]
    L.uscg_tracer_copy_cache.argtypes = [vp, vp, vp, vp, vp, C.c_uint32]
    L.uscg_tracer_import_cache_keys.argtypes = [vp, C.POINTER(_Grid), C.c_int32, vp, C.c_uint64, vp, vp, vp,
                                                C.c_int32, _dp, C.c_uint32, C.POINTER(vp)]
    L.uscg_tracer_get_info.argtypes = [vp, C.POINTER(_Info)]
    L.uscg_tracer_export_wave.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _u32p, _u32p, _u32p]
    L.uscg_tracer_export_cache.argtypes = [vp, _u32p, _dp, _dp, _u16p, _u16p]
    L.uscg_trace_line.argtypes = [vp, C.c_int32, C.c_double, _u32p, C.c_int64, C.POINTER(C.c_int64)]
    L.uscg_trace_counts.argtypes = [vp, _u32p]
    L.uscg_trace_checksums.argtypes = [vp, C.c_int32, C.c_int32, vp, vp, C.c_uint32]
    L.uscg_tracer_build_schedule.argtypes = [vp]
    L.uscg_tracer_export_successors.argtypes = [vp, C.POINTER(C.c_uint64), _u32p, _u32p]
    L.uscg_tracer_export_schedule.argtypes = [vp, C.POINTER(C.c_int32), _u32p, _u32p, C.POINTER(C.c_uint64), _u32p,
                                              _u32p, _u32p, _u32p, _u32p]
    L.uscg_problem_stride.argtypes = [C.c_int32]
    L.uscg_problem_stride.restype = C.c_int32
    L.uscg_project.argtypes = [vp, vp, C.c_int32, vp, C.c_uint32]
    L.uscg_reconstruct.argtypes = [vp, vp, C.c_int32, C.POINTER(_Cfg), vp, C.c_int32, C.POINTER(_Report),
                                   C.c_uint32]
    L.uscg_reconstruct_batch.argtypes = [vp, C.c_int32, C.POINTER(vp), C.c_int32, C.POINTER(_Cfg), C.POINTER(vp),
                                         C.c_int32, C.POINTER(_Report), C.c_uint32]
    L.uscg_resample.argtypes = [vp, C.POINTER(_Grid), vp, C.c_int32, C.c_int32, vp, C.c_uint32]
    L.uscg_uspg_to_cg_map.argtypes = [vp, C.c_int32, _u32p]
    L.uscg_cartesian_like.argtypes = [C.POINTER(_Grid), C.POINTER(_Cart)]
    L.uscg_csystem_create.argtypes = [vp, C.POINTER(_Cart), C.POINTER(_Scan), C.c_int32, C.POINTER(vp)]
    L.uscg_tracer_length_system.argtypes = [vp, C.POINTER(vp)]
    L.uscg_csystem_info.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_int32), _dp]
    L.uscg_csystem_export.argtypes = [vp, _u32p, _u32p, _fp]
    L.uscg_csystem_reconstruct.argtypes = [vp, vp, C.POINTER(_Cfg), vp, _dp, C.c_uint32]
    L.uscg_csystem_destroy.argtypes = [vp]
    L.uscg_image_metrics.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, _dp, _dp,
                                     _dp, C.c_uint32]
    L.uscg_cartesian_to_field.argtypes = [vp, C.POINTER(_Grid), vp, C.c_int32, C.c_int32, vp, C.c_uint32]
    L.uscg_image_sharpness.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_int32, _dp, C.c_uint32]
    L.uscg_intensity_profile.argtypes = [_fp, C.c_int32, C.c_int32, C.c_int32, _dp]
    L.uscg_diag_math.argtypes = [vp, C.c_int32, _dp, _dp, _dp]
    L.uscg_schedule_build.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p, C.c_uint64, _u32p, _u32p,
                                      _u32p, _u32p, _u32p, C.POINTER(C.c_uint64), _u32p]
    for name in EXPORTS:
        if name not in ("uscg_last_error", "uscg_version", "uscg_launch_count", "uscg_problem_stride"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().uscg_last_error().decode()
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 2:
        raise DomainError(msg)
    if rc == 4:
        raise NoDevice(msg)
    raise UscgError(f"uscg_b200 error {rc}: {msg}")


def launch_count() -> int:
    return int(load().uscg_launch_count())


def problem_stride(problems: int) -> int:
    return int(load().uscg_problem_stride(problems))


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------


class Context:
    """Device + stream (uscg_ctx). One per device is plenty."""

    def __init__(self, device: int = 0):
        L = load()
        h = C.c_void_p()
        _check(L.uscg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        _check(load().uscg_ctx_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def synchronize(self) -> None:
        _check(load().uscg_ctx_synchronize(self.h))

    def close(self) -> None:
        h, self.h = getattr(self, "h", None), None
        if h and _lib is not None:
            _lib.uscg_ctx_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None
_live_tracers: "weakref.WeakSet" = weakref.WeakSet()


@atexit.register
def _release_all() -> None:
    """Free device state while the library is still loaded: tracers first,
    then the default context (module teardown order is otherwise arbitrary)."""
    global _default_ctx
    for t in list(_live_tracers):
        t.close()
    if _default_ctx is not None:
        _default_ctx.close()
        _default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---------------------------------------------------------------------------
# grid / scan
# ---------------------------------------------------------------------------


class GridMode(enum.Enum):
    Slice2D = 0
    Volume3D = 1


@dataclass
class GridSpec:
    """GridSpec (grid.hpp:21-44). ``n`` is the image size: n/2 rings and, in 3D
    by default, n slices. Generalized seams: ``ring_counts`` (per-ring sector
    counts, None = the reference 4(2k-1) law) and ``n_slices``."""

    n: int = 0
    ring_spacing: float = 0.0
    slice_height: float = 0.0
    mode: GridMode = GridMode.Slice2D
    ring_counts: Optional[np.ndarray] = None
    n_slices: Optional[int] = None

    @staticmethod
    def square_2d(n: int) -> "GridSpec":
        return GridSpec(n, 2.0 / n, 2.0 / n, GridMode.Slice2D)

    @staticmethod
    def cube_3d(n: int) -> "GridSpec":
        return GridSpec(n, 2.0 / n, 2.0 / n, GridMode.Volume3D)

    def rings(self) -> int:
        return self.n // 2

    def slices(self) -> int:
        if self.mode != GridMode.Volume3D:
            return 1
        return self.n if self.n_slices is None else int(self.n_slices)

    def radius(self) -> float:
        return 0.5 * self.n * self.ring_spacing

    def counts(self) -> np.ndarray:
        if self.ring_counts is not None:
            return np.asarray(self.ring_counts, dtype=np.uint32)
        k = np.arange(1, self.rings() + 1)
        return (4 * (2 * k - 1)).astype(np.uint32)

    def cells_per_slice(self) -> int:
        return int(self.counts().astype(np.int64).sum())

    def cell_count(self) -> int:
        return self.cells_per_slice() * self.slices()

    def is_reference_law(self) -> bool:
        return self.ring_counts is None

    def _c(self):
        cnt = None if self.ring_counts is None else np.ascontiguousarray(self.ring_counts, dtype=np.uint32)
        g = _Grid(self.rings(), float(self.ring_spacing), self.slices(), float(self.slice_height),
                  1 if self.mode == GridMode.Volume3D else 0,
                  cnt.ctypes.data_as(_u32p) if cnt is not None else None)
        return g, cnt  # keep cnt alive with the struct


def ring_counts_m1(n_rings: int) -> np.ndarray:
    """BASELINE.json sector law: ring i (0-based) has round(2*pi*(i+0.5)) cells."""
    i = np.arange(n_rings, dtype=np.float64)
    return np.floor(2.0 * np.pi * (i + 0.5) + 0.5).astype(np.uint32)


class Detector(enum.IntEnum):
    Flat = 0
    Arc = 1
    Parallel = 2


@dataclass
class ScanGeometry:
    """ScanGeometry (scan.hpp:21-41) + detector kind and view-angle list."""

    source: Sequence[float] = (0.0, 0.0, 0.0)
    detector_center: Sequence[float] = (0.0, 0.0, 0.0)
    det_u: int = 1
    det_v: int = 1
    spacing_u: float = 0.0
    spacing_v: float = 0.0
    views: int = 1
    detector: Detector = Detector.Flat
    view_angles: Optional[np.ndarray] = None

    def step_deg(self) -> float:
        return 360.0 / self.views

    def lines(self) -> int:
        return self.det_u * self.det_v

    def thetas(self) -> np.ndarray:
        if self.view_angles is not None:
            return np.asarray(self.view_angles, dtype=np.float64)
        step = self.step_deg()
        return np.array([v * step for v in range(self.views)], dtype=np.float64)

    def _c(self):
        ang = None if self.view_angles is None else np.ascontiguousarray(self.view_angles, dtype=np.float64)
        s = _Scan(int(self.detector), (C.c_double * 3)(*[float(x) for x in self.source]),
                  (C.c_double * 3)(*[float(x) for x in self.detector_center]), int(self.det_u), int(self.det_v),
                  float(self.spacing_u), float(self.spacing_v), int(self.views),
                  ang.ctypes.data_as(_dp) if ang is not None else None)
        return s, ang

    def first_view_rays(self):
        """line_endpoints for every line of the first view, (lines, 3) x 2."""
        s, keep = self._c()
        src = np.zeros((self.lines(), 3))
        det = np.zeros((self.lines(), 3))
        _check(load().uscg_first_view_rays(C.byref(s), src.ctypes.data_as(_dp), det.ctypes.data_as(_dp)))
        return src, det


# ---------------------------------------------------------------------------
# tracer
# ---------------------------------------------------------------------------


@dataclass
class FirstViewCache:
    offsets: np.ndarray
    phi_a: np.ndarray
    phi_b: np.ndarray
    slice: np.ndarray
    ring: np.ndarray

    def line_count(self) -> int:
        return self.offsets.size - 1

    def record_count(self) -> int:
        return self.phi_a.size

    def byte_size(self) -> int:
        """Reference accounting (24-byte SegmentRecord + u32 offsets)."""
        return self.record_count() * 24 + self.offsets.size * 4


class Tracer:
    """Tracer (tracer.hpp:85-105): owns the device-resident first-view cache
    built by the K1 generator kernels, and traces any (line, view) on the
    device. ``from_rays`` and ``from_cache`` are the two other constructors of
    the C ABI (explicit rays; adopt an existing FirstViewCache)."""

    def __init__(self, geom: ScanGeometry, spec: GridSpec, quarter_symmetry: bool = False, threads: int = 1,
                 ctx: Optional[Context] = None, _handle=None):
        self.ctx = ctx or default_context()
        self.geom = geom
        self.spec = spec
        if _handle is not None:
            self.h = _handle
        else:
            g, keep1 = spec._c()
            s, keep2 = geom._c()
            h = C.c_void_p()
            _check(load().uscg_tracer_create(self.ctx.h, C.byref(g), C.byref(s), int(bool(quarter_symmetry)),
                                             C.byref(h)))
            self.h = h
        self._info = None
        _live_tracers.add(self)

    @classmethod
    def from_rays(cls, spec: GridSpec, src, det, views: int, view_angles=None, geom: Optional[ScanGeometry] = None,
                  ctx: Optional[Context] = None) -> "Tracer":
        ctx = ctx or default_context()
        src = np.ascontiguousarray(src, dtype=np.float64)
        det = np.ascontiguousarray(det, dtype=np.float64)
        ang = None if view_angles is None else np.ascontiguousarray(view_angles, dtype=np.float64)
        g, keep = spec._c()
        h = C.c_void_p()
        _check(load().uscg_tracer_create_from_rays(ctx.h, C.byref(g), src.shape[0], src.ctypes.data_as(_dp),
                                                   det.ctypes.data_as(_dp), views,
                                                   ang.ctypes.data_as(_dp) if ang is not None else None,
                                                   C.byref(h)))
        if geom is None:
            geom = ScanGeometry(det_u=src.shape[0], views=views, view_angles=ang)
        return cls(geom, spec, ctx=ctx, _handle=h)

    @classmethod
    def from_cache(cls, spec: GridSpec, cache: FirstViewCache, views: int, view_angles=None,
                   geom: Optional[ScanGeometry] = None, ctx: Optional[Context] = None) -> "Tracer":
        ctx = ctx or default_context()
        off = np.ascontiguousarray(cache.offsets, dtype=np.uint32)
        pa = np.ascontiguousarray(cache.phi_a, dtype=np.float64)
        pb = np.ascontiguousarray(cache.phi_b, dtype=np.float64)
        sl = np.ascontiguousarray(cache.slice, dtype=np.uint16)
        rg = np.ascontiguousarray(cache.ring, dtype=np.uint16)
        ang = None if view_angles is None else np.ascontiguousarray(view_angles, dtype=np.float64)
        g, keep = spec._c()
        h = C.c_void_p()
        _check(load().uscg_tracer_import_cache(ctx.h, C.byref(g), off.size - 1, off.ctypes.data_as(_u32p), pa.size,
                                               pa.ctypes.data_as(_dp), pb.ctypes.data_as(_dp),
                                               sl.ctypes.data_as(_u16p), rg.ctypes.data_as(_u16p), views,
                                               ang.ctypes.data_as(_dp) if ang is not None else None, C.byref(h)))
        if geom is None:
            geom = ScanGeometry(det_u=off.size - 1, views=views, view_angles=ang)
        return cls(geom, spec, ctx=ctx, _handle=h)

    def copy_cache(self, device: bool = True):
        """The record store in the device layout as torch tensors (on this
        tracer's GPU, or the host): offsets (lines+1) and keys (records) as
        int32 bit patterns of the u32 values, phi_a / phi_b float64."""
        import torch
        inf = self.info()
        where = torch.device("cuda", self.ctx.device) if device else torch.device("cpu")
        off = torch.empty(inf["lines"] + 1, dtype=torch.int32, device=where)
        pa = torch.empty(max(inf["records"], 1), dtype=torch.float64, device=where)
        pb = torch.empty_like(pa)
        key = torch.empty(max(inf["records"], 1), dtype=torch.int32, device=where)
        _check(load().uscg_tracer_copy_cache(self.h, off.data_ptr(), pa.data_ptr(), pb.data_ptr(), key.data_ptr(),
                                             DEVICE_POINTERS if device else 0))
        R = inf["records"]
        return off, pa[:R], pb[:R], key[:R]

    @classmethod
    def from_key_cache(cls, spec: GridSpec, offsets, phi_a, phi_b, keys, views: int, view_angles=None,
                       geom: Optional[ScanGeometry] = None, ctx: Optional[Context] = None) -> "Tracer":
        """Import a record store in the device layout (torch tensors, CUDA or CPU)."""
        ctx = ctx or default_context()
        dev = offsets.is_cuda
        ang = None if view_angles is None else np.ascontiguousarray(view_angles, dtype=np.float64)
        g, keep = spec._c()
        h = C.c_void_p()
        _check(load().uscg_tracer_import_cache_keys(ctx.h, C.byref(g), int(offsets.numel()) - 1, offsets.data_ptr(),
                                                    int(phi_a.numel()), phi_a.data_ptr(), phi_b.data_ptr(),
                                                    keys.data_ptr(), views,
                                                    ang.ctypes.data_as(_dp) if ang is not None else None,
                                                    DEVICE_POINTERS if dev else 0, C.byref(h)))
        if geom is None:
            geom = ScanGeometry(det_u=int(offsets.numel()) - 1, views=views, view_angles=ang)
        return cls(geom, spec, ctx=ctx, _handle=h)

    def close(self) -> None:
        h, self.h = getattr(self, "h", None), None
        if h and _lib is not None:
            _lib.uscg_tracer_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- introspection -------------------------------------------------------
    def info(self) -> dict:
        i = _Info()
        _check(load().uscg_tracer_get_info(self.h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in _Info._fields_}

    def cache(self) -> FirstViewCache:
        inf = self.info()
        n, L = inf["records"], inf["lines"]
        off = np.zeros(L + 1, np.uint32)
        pa = np.zeros(n); pb = np.zeros(n)
        sl = np.zeros(n, np.uint16); rg = np.zeros(n, np.uint16)
        _check(load().uscg_tracer_export_cache(self.h, off.ctypes.data_as(_u32p), pa.ctypes.data_as(_dp),
                                               pb.ctypes.data_as(_dp), sl.ctypes.data_as(_u16p),
                                               rg.ctypes.data_as(_u16p)))
        return FirstViewCache(off, pa, pb, sl, rg)

    def trace_line(self, line: int, theta_deg: float) -> np.ndarray:
        """Tracer::trace_line: deduplicated active cells, reference emission order."""
        inf = self.info()
        cap = inf["max_line_cells"] + inf["max_line_records"] + 1
        out = np.zeros(cap, np.uint32)
        n = C.c_int64()
        _check(load().uscg_trace_line(self.h, int(line), float(theta_deg), out.ctypes.data_as(_u32p), cap,
                                      C.byref(n)))
        return out[: n.value].copy()

    def trace_counts(self) -> np.ndarray:
        inf = self.info()
        out = np.zeros(inf["views"] * inf["lines"], np.uint32)
        _check(load().uscg_trace_counts(self.h, out.ctypes.data_as(_u32p)))
        return out.reshape(inf["views"], inf["lines"])

    def trace_checksums(self, view0: int = 0, nviews: Optional[int] = None):
        """Rotated reuse: (|active|, sum of active cell indices) of every line of
        views [view0, view0 + nviews), each shaped (nviews, lines)."""
        inf = self.info()
        nviews = inf["views"] - view0 if nviews is None else nviews
        counts = np.zeros(nviews * inf["lines"], np.uint32)
        sums = np.zeros(nviews * inf["lines"], np.uint64)
        _check(load().uscg_trace_checksums(self.h, int(view0), int(nviews), counts.ctypes.data, sums.ctypes.data, 0))
        return counts.reshape(nviews, inf["lines"]), sums.reshape(nviews, inf["lines"])

    def schedule(self) -> dict:
        """The dataflow executor's run schedule: run, runs, levels, order,
        level_off, pred_off, preds, npred_x, succ_off, succs (numpy u32 arrays)."""
        L = load()
        run, runs, levels, npr = C.c_int32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        _check(L.uscg_tracer_export_schedule(self.h, C.byref(run), C.byref(runs), C.byref(levels), C.byref(npr),
                                             None, None, None, None, None))
        R, V, P = runs.value, levels.value, npr.value
        out = {k: np.zeros(n, np.uint32) for k, n in (("order", R), ("level_off", V + 1), ("pred_off", R + 1),
                                                      ("preds", max(P, 1)), ("npred_x", R))}
        _check(L.uscg_tracer_export_schedule(self.h, C.byref(run), C.byref(runs), C.byref(levels), C.byref(npr),
                                             *[out[k].ctypes.data_as(_u32p) for k in
                                               ("order", "level_off", "pred_off", "preds", "npred_x")]))
        out["preds"] = out["preds"][:P]
        ns = C.c_uint64()
        _check(L.uscg_tracer_export_successors(self.h, C.byref(ns), None, None))
        out["succ_off"] = np.zeros(R + 1, np.uint32)
        out["succs"] = np.zeros(max(ns.value, 1), np.uint32)
        _check(L.uscg_tracer_export_successors(self.h, C.byref(ns), out["succ_off"].ctypes.data_as(_u32p),
                                               out["succs"].ctypes.data_as(_u32p)))
        out["succs"] = out["succs"][:ns.value]
        out.update(run=run.value, runs=R, levels=V)
        return out

    def wave_arrays(self) -> dict:
        """The wave executor's derived arrays (diagnostics): entries (n, 2) u32,
        dep_off (units + 1) and deps (n, 2) u32."""
        L = load()
        ne, nd = C.c_uint64(), C.c_uint64()
        _check(L.uscg_tracer_export_wave(self.h, C.byref(ne), C.byref(nd), None, None, None))
        inf = self.info()
        ent = np.zeros((max(ne.value, 1), 2), np.uint32)
        off = np.zeros(inf["views"] * inf["lines"] + 1, np.uint32)
        deps = np.zeros((max(nd.value, 1), 2), np.uint32)
        _check(L.uscg_tracer_export_wave(self.h, C.byref(ne), C.byref(nd), ent.ctypes.data_as(_u32p),
                                         off.ctypes.data_as(_u32p), deps.ctypes.data_as(_u32p)))
        return {"entries": ent[: ne.value], "dep_off": off, "deps": deps[: nd.value]}

    def build_schedule(self) -> int:
        _check(load().uscg_tracer_build_schedule(self.h))
        return self.info()["levels"]


# ---------------------------------------------------------------------------
# solver types
# ---------------------------------------------------------------------------


@dataclass
class Field:
    spec: GridSpec
    values: np.ndarray

    @staticmethod
    def constant(spec: GridSpec, value: float) -> "Field":
        return Field(spec, np.full(spec.cell_count(), float(value)))


@dataclass
class ProjectionSet:
    geometry: ScanGeometry
    data: np.ndarray  # (views, lines) or flat view-major

    def at(self, view: int, line: int) -> float:
        return float(np.asarray(self.data).reshape(-1)[view * self.geometry.lines() + line])


@dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:34-41). ``update``: "linear" is the reference's
    1 - beta (1 - m/p) (solver.cpp:41); "power" selects the multiplicative
    (m/p)^beta form (USCG_UPDATE_POWER, an extension without a reference
    counterpart)."""
    beta: float = 0.4
    tolerance: float = 1e-6
    max_sweeps: int = 100
    f_init: float = 1.0
    p_floor: float = 0.0
    update: str = "linear"

    def _flags(self) -> int:
        if self.update not in ("linear", "power"):
            raise InvalidArgument(f"unknown update form {self.update!r}")
        return UPDATE_POWER if self.update == "power" else 0


@dataclass
class ReconReport:
    sweep_residuals: list = dc_field(default_factory=list)
    sweeps: int = 0
    converged: bool = False
    all_zero_data: bool = False
    seconds: float = 0.0
    zero_measurement_skips: int = 0
    factor_clamps: int = 0
    updates: int = 0
    crossed: Optional[np.ndarray] = None


@dataclass
class ReconResult:
    field: Field
    report: ReconReport


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _validate_field(field_values: np.ndarray, spec: GridSpec):
    if field_values.size != spec.cell_count():
        raise InvalidArgument("field length does not match its grid")


def generate_projections(field: Field, geom: ScanGeometry, model: str = "binary",
                         tracer: Optional[Tracer] = None) -> ProjectionSet:
    """generate_projections (phantom.hpp:51-52) on the device: model "binary"
    (phantom.cpp:182-211) or "length" / "lengthweighted" (phantom.cpp:213-269)."""
    m = model.lower().replace("_", "").replace("-", "")
    if m not in ("binary", "length", "lengthweighted"):
        raise InvalidArgument(f"unknown forward model {model!r}")
    vals = np.ascontiguousarray(field.values, dtype=np.float32).reshape(-1)
    _validate_field(vals, field.spec)
    if tracer is None or m != "binary":
        # the reference's length-weighted model walks the geometry itself and
        # takes no tracer (phantom.cpp:213-269); here it runs on a tracer's rays
        tracer = Tracer(geom, field.spec, False)
    out = project_stack(tracer, vals[None, :], model="binary" if m == "binary" else "length")
    return ProjectionSet(geom, out[0].astype(np.float64))


def project_stack(tracer: Tracer, fields: np.ndarray, model: str = "binary") -> np.ndarray:
    """Projections of S independent fields sharing one tracer:
    fields (S, cell_count) -> (S, views, lines), float32. model "binary" or
    "length" (length-weighted; needs a tracer built from a geometry or rays)."""
    f = np.ascontiguousarray(fields, dtype=np.float32)
    S = f.shape[0]
    inf = tracer.info()
    out = np.zeros((S, inf["views"], inf["lines"]), np.float32)
    flags = MODEL_LENGTH if model == "length" else 0
    _check(load().uscg_project(tracer.h, _ptr(f), S, _ptr(out), flags))
    return out


def _run(proj_data: np.ndarray, init: Optional[np.ndarray], cfg: SolverConfig, tracer: Tracer, S: int,
         with_crossed: bool = True):
    inf = tracer.info()
    p = np.ascontiguousarray(proj_data, dtype=np.float32).reshape(S, -1)
    if p.shape[1] != inf["views"] * inf["lines"]:
        raise InvalidArgument(f"projection data size does not match geometry: got {p.shape[1]}, "
                              f"expected {inf['views'] * inf['lines']}")
    cells = inf["cell_count"]
    if init is None:
        fld = np.zeros((S, cells), np.float32)
        from_init = 0
    else:
        fld = np.array(init, dtype=np.float32, copy=True).reshape(S, cells)
        from_init = 1
    reps = (_Report * S)()
    resid = [np.zeros(cfg.max_sweeps) for _ in range(S)]
    crossed = [np.zeros(cells, np.uint8) for _ in range(S)] if with_crossed else None
    for i in range(S):
        reps[i].sweep_residuals = resid[i].ctypes.data_as(_dp)
        reps[i].crossed = crossed[i].ctypes.data_as(_u8p) if with_crossed else None
    c = _Cfg(cfg.beta, cfg.tolerance, cfg.max_sweeps, cfg.f_init, cfg.p_floor)
    _check(load().uscg_reconstruct(tracer.h, _ptr(p), S, C.byref(c), _ptr(fld), from_init, reps, cfg._flags()))
    out = []
    for i in range(S):
        r = reps[i]
        rep = ReconReport(
            sweep_residuals=list(resid[i][: r.sweeps]) if cfg.tolerance > 0 else [],
            sweeps=r.sweeps, converged=bool(r.converged), all_zero_data=bool(r.all_zero_data),
            seconds=r.seconds, zero_measurement_skips=int(r.zero_measurement_skips),
            factor_clamps=int(r.factor_clamps), updates=int(r.updates),
            crossed=crossed[i] if with_crossed else None)
        out.append((fld[i], rep))
    return out


def reconstruct(proj: ProjectionSet, spec: GridSpec, cfg: SolverConfig, tracer: Tracer) -> ReconResult:
    """reconstruct (solver.cpp:166-169): start from cfg.f_init everywhere."""
    (f, rep), = _run(np.asarray(proj.data), None, cfg, tracer, 1)
    return ReconResult(Field(spec, f.astype(np.float64)), rep)


def reconstruct_from(proj: ProjectionSet, init: Field, cfg: SolverConfig, tracer: Tracer) -> ReconResult:
    """reconstruct_from (solver.cpp:171-177): start from `init` (must be > 0)."""
    vals = np.asarray(init.values, dtype=np.float64)
    if not np.all(vals > 0):
        raise InvalidArgument("initial field must be strictly positive")
    (f, rep), = _run(np.asarray(proj.data), vals, cfg, tracer, 1)
    return ReconResult(Field(init.spec, f.astype(np.float64)), rep)


def reconstruct_stack(projections: np.ndarray, cfg: SolverConfig, tracer: Tracer,
                      init: Optional[np.ndarray] = None, with_crossed: bool = False):
    """S independent reconstructions sharing one tracer (the 2D slice stack):
    projections (S, views, lines) -> list of (field (cell_count,), ReconReport)."""
    S = projections.shape[0]
    return _run(projections, init, cfg, tracer, S, with_crossed)


def reconstruct_batch(stacks, cfg: SolverConfig, tracer: Tracer, inits=None):
    """reconstruct_stack over several independent stacks (each (S, views,
    lines)) in one call, their host transfers overlapped with the neighbouring
    stacks' solves (uscg_reconstruct_batch); returns one list of fields
    (S, cell_count) per stack. Host buffers are pinned (torch) when torch is
    importable, so the copies can overlap."""
    inf = tracer.info()
    cells, units = inf["cell_count"], inf["views"] * inf["lines"]
    B = len(stacks)
    if B == 0:
        return []
    S = int(np.asarray(stacks[0]).shape[0])
    try:
        import torch
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).pin_memory()  # noqa: E731
        host = lambda t: t.numpy()  # noqa: E731
    except Exception:  # pragma: no cover - torch is part of the image
        pin = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
        host = lambda t: t  # noqa: E731
    projs, flds = [], []
    for b in range(B):
        p = np.asarray(stacks[b], dtype=np.float32).reshape(S, -1)
        if p.shape[1] != units:
            raise InvalidArgument(f"projection data size does not match geometry: got {p.shape[1]}, "
                                  f"expected {units}")
        projs.append(pin(p))
        flds.append(pin(np.zeros((S, cells), np.float32) if inits is None
                        else np.asarray(inits[b], np.float32).reshape(S, cells)))
    pp = (C.c_void_p * B)(*[C.c_void_p(host(x).ctypes.data) for x in projs])
    ff = (C.c_void_p * B)(*[C.c_void_p(host(x).ctypes.data) for x in flds])
    c = _Cfg(cfg.beta, cfg.tolerance, cfg.max_sweeps, cfg.f_init, cfg.p_floor)
    _check(load().uscg_reconstruct_batch(tracer.h, B, pp, S, C.byref(c), ff, 0 if inits is None else 1, None,
                                         cfg._flags()))
    return [host(f).copy() for f in flds]


def field_to_cartesian(field: Field, npix: Optional[int] = None, ctx: Optional[Context] = None) -> np.ndarray:
    """field_to_cartesian (phantom.cpp:149-163): (slices, npix, npix), row 0 at the bottom.
    Reference law with npix = n: the one-to-one permutation; otherwise the
    bin-point rule at pixel centres."""
    ctx = ctx or default_context()
    spec = field.spec
    npix = spec.n if npix is None else npix
    vals = np.ascontiguousarray(field.values, dtype=np.float32).reshape(-1)
    _validate_field(vals, spec)
    return resample_stack(spec, vals[None, :], npix, ctx)[0]


def resample_stack(spec: GridSpec, fields: np.ndarray, npix: int, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    f = np.ascontiguousarray(fields, dtype=np.float32)
    S = f.shape[0]
    out = np.zeros((S, spec.slices(), npix, npix), np.float32)
    g, keep = spec._c()
    _check(load().uscg_resample(ctx.h, C.byref(g), _ptr(f), S, npix, _ptr(out), 0))
    return out


def cartesian_to_field(slices, spec: GridSpec, ctx: Optional[Context] = None) -> Field:
    """cartesian_to_field (phantom.hpp:59, phantom.cpp:165-180): the inverse
    of field_to_cartesian for the reference law. slices: (slices, n, n)
    rasters, row 0 at the bottom. Raises InvalidArgument, as the reference,
    when the slice count or shape does not match the grid."""
    ctx = ctx or default_context()
    im = np.ascontiguousarray(slices, dtype=np.float32)
    if im.ndim == 2:
        im = im[None]
    if im.ndim != 3 or im.shape[0] != spec.slices():
        raise InvalidArgument("slice count does not match the grid")
    if im.shape[1] != im.shape[2]:
        raise InvalidArgument("slice shape does not match the grid")
    out = np.zeros(spec.cell_count(), np.float32)
    g, keep = spec._c()
    _check(load().uscg_cartesian_to_field(ctx.h, C.byref(g), _ptr(im), 1, im.shape[1], _ptr(out), 0))
    return Field(spec, out)


def sharpness(image, ctx: Optional[Context] = None):
    """uscg::sharpness (metrics.cpp:138-152): mean central-difference gradient
    magnitude of one (rows, cols) raster; a (slices, rows, cols) stack gives one
    value per slice."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(image, dtype=np.float32)
    one = a.ndim == 2
    if one:
        a = a[None]
    if a.ndim != 3:
        raise InvalidArgument("sharpness needs (rows, cols) or (slices, rows, cols) rasters")
    out = np.zeros(a.shape[0])
    _check(load().uscg_image_sharpness(ctx.h, _ptr(a), a.shape[0], a.shape[1], a.shape[2],
                                       out.ctypes.data_as(_dp), 0))
    return float(out[0]) if one else out


def intensity_profile(image, row: int) -> np.ndarray:
    """uscg::intensity_profile (metrics.cpp:154-159): row `row` of a (rows, cols)
    raster as float64; InvalidArgument when the row is out of range."""
    a = np.ascontiguousarray(image, dtype=np.float32)
    if a.ndim != 2:
        raise InvalidArgument("intensity_profile needs one (rows, cols) raster")
    out = np.zeros(a.shape[1])
    _check(load().uscg_intensity_profile(a.ctypes.data_as(_fp), a.shape[0], a.shape[1], int(row),
                                         out.ctypes.data_as(_dp)))
    return out


def image_metrics(ref, test, shared_range: bool = False, dynamic_range: float = -1.0, ssim: bool = True,
                  ctx: Optional[Context] = None) -> dict:
    """Per-slice mae / rmse / ssim of two (slices, rows, cols) raster stacks on
    the device (metrics.cpp:35-60,105-136); shared_range: one ssim dynamic range
    from the whole reference stack (ssim_volume, metrics.cpp:186-199)."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(ref, dtype=np.float32)
    b = np.ascontiguousarray(test, dtype=np.float32)
    if a.ndim == 2:
        a, b = a[None], b[None]
    if a.shape != b.shape:
        raise InvalidArgument("image shapes differ")
    S, rows, cols = a.shape
    mae_o, rmse_o, ssim_o = np.zeros(S), np.zeros(S), np.zeros(S)
    _check(load().uscg_image_metrics(ctx.h, _ptr(a), _ptr(b), S, rows, cols, int(bool(shared_range)),
                                     float(dynamic_range), mae_o.ctypes.data_as(_dp), rmse_o.ctypes.data_as(_dp),
                                     ssim_o.ctypes.data_as(_dp) if ssim else None, 0))
    out = {"mae": mae_o, "rmse": rmse_o}
    if ssim:
        out["ssim"] = ssim_o
    return out


def rmse(ref, test) -> float:
    """uscg::rmse(Image, Image) (metrics.cpp:42-50,57-60)."""
    return float(image_metrics(ref, test, ssim=False)["rmse"][0])


def mae(ref, test) -> float:
    """uscg::mae(Image, Image) (metrics.cpp:35-41,52-55)."""
    return float(image_metrics(ref, test, ssim=False)["mae"][0])


def ssim(ref, test, dynamic_range: float = -1.0) -> float:
    """uscg::ssim (metrics.cpp:105-136): 8x8 windows, stride 1."""
    return float(image_metrics(ref, test, dynamic_range=dynamic_range)["ssim"][0])


def rmse_volume(ref, test) -> float:
    """uscg::rmse_volume (metrics.cpp:178-184): mean of per-slice rmse."""
    return float(image_metrics(ref, test, ssim=False)["rmse"].mean())


def mae_volume(ref, test) -> float:
    """uscg::mae_volume (metrics.cpp:170-176)."""
    return float(image_metrics(ref, test, ssim=False)["mae"].mean())


def ssim_volume(ref, test) -> float:
    """uscg::ssim_volume (metrics.cpp:186-199): per-slice ssim with the dynamic
    range of the whole reference stack, averaged."""
    return float(image_metrics(ref, test, shared_range=True)["ssim"].mean())


class CartesianSystem:
    """The paper's Cartesian baseline on the device (proj/include/uscg/siddon.hpp):
    CartesianSpec::like(spec), precompute_cartesian_system(geom, cspec) and
    cartesian_mart_stored (stored=True) / cartesian_mart_otf (stored=False)."""

    def __init__(self, spec: GridSpec, geom: ScanGeometry, stored: bool = True, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        self._ctx = ctx
        g, keep_g = spec._c()
        self.cart = _Cart()
        _check(load().uscg_cartesian_like(C.byref(g), C.byref(self.cart)))
        sc, keep_s = geom._c()
        h = C.c_void_p()
        _check(load().uscg_csystem_create(ctx.h, C.byref(self.cart), C.byref(sc), int(bool(stored)), C.byref(h)))
        self.h = h.value
        self.geom, self.stored = geom, bool(stored)
        self.voxels = self.cart.nx * self.cart.ny * self.cart.nz

    def info(self) -> dict:
        e, b, lv, ms = C.c_uint64(), C.c_uint64(), C.c_int32(), C.c_double()
        _check(load().uscg_csystem_info(self.h, C.byref(e), C.byref(b), C.byref(lv), C.byref(ms)))
        return {"entries": e.value, "device_bytes": b.value, "levels": lv.value, "precompute_ms": ms.value}

    def export(self):
        """(offsets u32 [views*lines+1], voxel indices u32, lengths f32)"""
        inf = self.info()
        rows = self.geom.views * self.geom.lines()
        off = np.zeros(rows + 1, np.uint32)
        idx = np.zeros(inf["entries"], np.uint32)
        w = np.zeros(inf["entries"], np.float32)
        _check(load().uscg_csystem_export(self.h, off.ctypes.data_as(_u32p), idx.ctypes.data_as(_u32p),
                                          w.ctypes.data_as(_fp)))
        return off, idx, w

    def reconstruct(self, proj, cfg: SolverConfig):
        """(field f32 [voxels], device seconds) after cfg.max_sweeps sweeps"""
        p = np.ascontiguousarray(proj, dtype=np.float32).reshape(-1)
        if p.size != self.geom.views * self.geom.lines():
            raise InvalidArgument("projection data size does not match geometry")
        out = np.zeros(self.voxels, np.float32)
        sec = C.c_double()
        c = _Cfg(cfg.beta, cfg.tolerance, cfg.max_sweeps, cfg.f_init, cfg.p_floor)
        _check(load().uscg_csystem_reconstruct(self.h, _ptr(p), C.byref(c), _ptr(out), C.byref(sec), 0))
        return out, sec.value

    def close(self) -> None:
        h, self.h = getattr(self, "h", None), None
        if h and _lib is not None:
            _lib.uscg_csystem_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LengthSystem(CartesianSystem):
    """The polar grid's own (voxel index, chord length) lists (the pieces of
    the LengthWeighted model, phantom.cpp:213-269, a cell's pieces merged) for
    every (view, line) of the tracer's scan, with the reference's weighted row
    action (weighted_update, siddon.cpp:141-154) on the USPG / USCG field:
    export() -> (offsets, cell indices, lengths); reconstruct(proj, cfg) ->
    (field f32 [cell_count], device seconds)."""

    def __init__(self, tracer: "Tracer"):
        h = C.c_void_p()
        _check(load().uscg_tracer_length_system(tracer.h, C.byref(h)))
        self.h = h.value
        self._tracer = tracer  # the system uses the tracer's context
        self.geom, self.stored = tracer.geom, True
        self.voxels = tracer.spec.cell_count()


def uspg_to_cg_map(n: int, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    out = np.zeros(max(n, 0) * max(n, 0), np.uint32)
    _check(load().uscg_uspg_to_cg_map(ctx.h, n, out.ctypes.data_as(_u32p)))
    return out


def diag_math(x, y, ctx: Optional[Context] = None) -> np.ndarray:
    """Device math of the generator: columns atan2 (the generator's quick form
    with its fallback), hypot (correctly rounded), azimuth_deg, libdevice
    atan2, the double-double atan2 alone — for parity tests."""
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    out = np.zeros((x.size, 5))
    _check(load().uscg_diag_math(ctx.h, x.size, x.ctypes.data_as(_dp), y.ctypes.data_as(_dp),
                                 out.ctypes.data_as(_dp)))
    return out


def schedule_build(supports, cell_count: int, lines_per_view: Optional[int] = None, run: int = 1):
    """The MART dependency schedule (host C++, no device needed) from explicit
    supports in sweep order, grouped into runs of `run` consecutive lines of a
    view: dict(levels, order, level_off, pred_off, preds, npred_x) per run."""
    n = len(supports)
    lpv = n if lines_per_view is None else int(lines_per_view)
    pos = np.zeros(n + 1, np.uint32)
    pos[1:] = np.cumsum([len(s) for s in supports])
    idx = np.ascontiguousarray(np.concatenate([np.asarray(s, np.uint32) for s in supports])
                               if n else np.zeros(0, np.uint32), dtype=np.uint32)
    runs = n // max(run, 1) if n else 0
    order = np.zeros(max(runs, 1), np.uint32)
    level_off = np.zeros(runs + 1, np.uint32)
    levels = np.zeros(1, np.uint32)
    pred_off = np.zeros(runs + 1, np.uint32)
    preds = np.zeros(max(int(pos[-1]), 1), np.uint32)
    npred_x = np.zeros(max(runs, 1), np.uint32)
    npreds = C.c_uint64()
    _check(load().uscg_schedule_build(n, lpv, run, pos.ctypes.data_as(_u32p), idx.ctypes.data_as(_u32p), cell_count,
                                      order.ctypes.data_as(_u32p), level_off.ctypes.data_as(_u32p),
                                      levels.ctypes.data_as(_u32p), pred_off.ctypes.data_as(_u32p),
                                      preds.ctypes.data_as(_u32p), C.byref(npreds), npred_x.ctypes.data_as(_u32p)))
    L = int(levels[0])
    return dict(levels=L, order=order[:runs], level_off=level_off[:L + 1], pred_off=pred_off,
                preds=preds[:npreds.value], npred_x=npred_x[:runs])
