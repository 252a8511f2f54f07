"""B200-native USPG/USCG Sp-MART hot path (arXiv 2208.12964).

The product is ``lib/libuscg_b200.so``: hand-written sm_100a CUDA kernels behind
the C ABI declared in ``include/uscg_b200.h``. :mod:`.uscg` mirrors the
reference library's reconstruction API on top of that ABI.
"""
from .uscg import (  # noqa: F401
    CartesianSystem, LengthSystem, Context, cartesian_to_field, intensity_profile, sharpness, Detector, DomainError, Field, FirstViewCache, GridMode, GridSpec, InvalidArgument, NoDevice,
    ProjectionSet, ReconReport, ReconResult, ScanGeometry, SolverConfig, Tracer, field_to_cartesian,
    generate_projections, image_metrics, launch_count, load, mae, mae_volume, problem_stride, project_stack,
    reconstruct, reconstruct_batch, reconstruct_from, reconstruct_stack, resample_stack, ring_counts_m1, rmse, rmse_volume, ssim,
    ssim_volume, uspg_to_cg_map,
)

__all__ = [
    "cartesian_to_field", "intensity_profile", "sharpness", "CartesianSystem", "LengthSystem", "Context", "Detector", "DomainError", "Field", "FirstViewCache", "GridMode", "GridSpec", "InvalidArgument",
    "NoDevice", "ProjectionSet", "ReconReport", "ReconResult", "ScanGeometry", "SolverConfig", "Tracer",
    "field_to_cartesian", "generate_projections", "image_metrics", "launch_count", "load", "mae", "mae_volume",
    "problem_stride", "project_stack", "reconstruct", "reconstruct_batch", "reconstruct_from", "reconstruct_stack", "resample_stack",
    "ring_counts_m1", "rmse", "rmse_volume", "ssim", "ssim_volume", "uspg_to_cg_map",
]
