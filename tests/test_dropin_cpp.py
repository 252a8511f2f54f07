"""The C++ drop-in (include/uscg_b200.hpp), compiled and run as a reference
caller would after switching namespace uscg -> uscg_b200:
Tracer(geom, spec, quarter) -> reconstruct -> field_to_cartesian on the
snippet's cone-beam geometry, against the unmodified reference library
(oracle/_ref) on the same projections: counters exact, field and rasters
within the fp32 tolerance; invalid input throws std::invalid_argument
(solver.hpp:78-83, solver.cpp:55-61)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_matches_reference(ub, ref, tmp_path):
    exe = tmp_path / "dropin_cpp"
    lib = os.path.join(ROOT, "paper_2208_12964_b200", "lib")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "dropin_cpp.cpp"), "-o", str(exe), "-L", lib, "-luscg_b200",
                    f"-Wl,-rpath,{lib}"], check=True)
    sweeps = 4
    out = str(tmp_path / "run")
    subprocess.run([str(exe), out, str(sweeps)], check=True, timeout=600)
    n, views, det = 64, 70, 101
    proj = np.fromfile(out + ".proj").reshape(views, det * det)
    field = np.fromfile(out + ".field")
    img = np.fromfile(out + ".img").reshape(n, n, n)
    s, upd, skips, clamps, threw, nimg = open(out + ".rep").read().split()
    rt = ref.tracer(n, True, (-3, 0, 0), (10, 0, 0), det, det, 0.092, 0.13, views, True)
    want, wrep = rt.reconstruct(proj, beta=0.4, tolerance=0, max_sweeps=sweeps)
    assert int(s) == wrep["sweeps"] == sweeps
    assert int(skips) == wrep["zero_measurement_skips"] and int(clamps) == wrep["factor_clamps"]
    assert int(threw) == 1 and int(nimg) == n
    assert (np.abs(field - want) / want).max() <= 1e-4
    want_img = ref.field_to_cartesian(n, True, field.astype(np.float32).astype(np.float64))
    assert np.array_equal(img, want_img)  # the permutation moves fp32 values unchanged
    # cartesian_to_field, sharpness, intensity_profile, rmse, ssim, mae, area_average
    back = np.fromfile(out + ".back")
    assert np.array_equal(back, ref.cartesian_to_field(n, True, img))
    extra = np.fromfile(out + ".extra")
    a, b = img[31], img[32]
    assert abs(extra[0] - ref.sharpness(b)) <= 1e-12 * ref.sharpness(b)
    assert abs(extra[1] - ref.rmse(a, b)) <= 1e-12 * ref.rmse(a, b)
    assert abs(extra[2] - ref.ssim(a, b)) <= 1e-9
    assert abs(extra[3] - np.abs(a - b).mean()) <= 1e-12 * np.abs(a - b).mean()
    assert abs(extra[4] - b.mean()) <= 1e-12 * abs(b.mean())
    assert np.array_equal(extra[5:], ref.intensity_profile(b, 10))
    # U = every non-skipped line's |active| per sweep (TraceScratch::cells,
    # tracer.cpp:200), sampled against the reference's own trace_line
    spec = ub.GridSpec.cube_3d(n)
    geom = ub.ScanGeometry(source=(-3, 0, 0), detector_center=(10, 0, 0), det_u=det, det_v=det, spacing_u=0.092,
                           spacing_v=0.13, views=views)
    counts = ub.Tracer(geom, spec, True).trace_counts()
    rng = np.random.default_rng(0)
    for v, l in zip(rng.integers(0, views, 200), rng.integers(0, det * det, 200)):
        assert counts[v, l] == rt.trace_line(int(l), v * 360.0 / views).size
    assert int(upd) == int(counts[proj != 0].sum()) * sweeps
