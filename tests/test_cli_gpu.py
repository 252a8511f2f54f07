"""The CLI pipeline on the device: phantom -> project
-> reconstruct -> map -> metrics with the reference's file formats, the same
steps and checks as the reference's pipeline test (proj/tests/test_io_cli.cpp:
163-231). Where the step is exact the reference library's own output is the
oracle: the phantom field and its Cartesian companion (bytes and sidecars);
projections agree to fp32 rounding; the reconstruction closes on its data.

The tolerance here is 1e-6, not the reference test's 1e-9: an fp32 field
cannot move by less than ~1e-7 relative per sweep."""
import os
import subprocess

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _cli(*args):
    from paper_2208_12964_b200 import _build
    _build.build()
    r = subprocess.run([_build.CLI, *map(str, args)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return r


def _meta(path):
    out = {}
    for line in open(str(path) + ".meta"):
        k, v = line.rstrip("\n").split(" = ", 1)
        out[k] = v
    return out


@pytest.fixture
def rio():
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("reference library not built")
    return oracle.RefIO(oracle.Ref())


def test_cli_pipeline(ub, ref, rio, tmp_path):
    n = 16
    rng = np.random.default_rng(11)
    raw = rng.uniform(0.2, 3.0, n * n).astype(np.float32)
    raw.tofile(tmp_path / "raw.bin")
    _cli("phantom", "--kind", "raw-volume", "--raw", tmp_path / "raw.bin", "--raw-mode", "2d", "--n", n,
         "--out", tmp_path / "truth.fld")
    assert (tmp_path / "truth.cg.pgm").exists()

    # the reference's bytes for the same phantom: cartesian_to_field, its
    # companion raster (field_to_cartesian), identical sidecars
    m = ref.uspg_to_cg_map(n)
    field = raw.astype(np.float64)[m]
    echo = {"provenance": "phantom raw-volume", "config.kind": "raw-volume", "config.n": str(n),
            "config.ring_spacing": "0.125", "config.slice_height": "0.125", "config.raw": str(tmp_path / "raw.bin"),
            "config.threads": "1", "config.seed": "0", "clipped_negative": "false"}
    rio.write_field(tmp_path / "ref_truth.fld", n, 0.125, 0.125, False, field, echo)
    assert open(tmp_path / "truth.fld", "rb").read() == open(tmp_path / "ref_truth.fld", "rb").read()
    assert _meta(tmp_path / "truth.fld") == _meta(tmp_path / "ref_truth.fld")
    img = ref.field_to_cartesian(n, False, field).reshape(n, n)
    rio.write_pgm16(tmp_path / "ref_truth.cg.pgm", img, float(field.min()), float(field.max()),
                    {**echo, "slice": "0", "slices": "1"})
    assert open(tmp_path / "truth.cg.pgm", "rb").read() == open(tmp_path / "ref_truth.cg.pgm", "rb").read()
    assert _meta(tmp_path / "truth.cg.pgm") == _meta(tmp_path / "ref_truth.cg.pgm")

    geo = ["--views", 20, "--det-u", 21, "--spacing-u", 0.2, "--source", "-8,0", "--center", "8,0"]
    _cli("project", "--field", tmp_path / "truth.fld", *geo, "--out", tmp_path / "data.prj")
    side = _meta(tmp_path / "data.prj")
    assert side["grid_n"] == str(n) and side["config.model"] == "binary" and side["type"] == "projections"
    data = np.fromfile(tmp_path / "data.prj", np.float32, offset=40).astype(np.float64)
    rt = ref.tracer(n, False, (-8, 0, 0), (8, 0, 0), 21, 1, 0.2, 0.0, 20, False)
    want = rt.project(field).reshape(-1)
    np.testing.assert_allclose(data, want, rtol=1e-6, atol=1e-6)

    _cli("reconstruct", "--proj", tmp_path / "data.prj", "--n", n, "--beta", 1.0, "--tol", 1e-6, "--sweeps", 20000,
         "--out", tmp_path / "recon.fld", "--report", tmp_path / "recon.report.txt")
    assert (tmp_path / "recon.report.txt").exists()
    rs = _meta(tmp_path / "recon.fld")
    assert rs["config.beta"] == "1" and rs["converged"] == "true"
    report = dict(line.rstrip("\n").split(" = ", 1) for line in open(tmp_path / "recon.report.txt"))
    assert report["all_zero_data"] == "false" and int(report["crossed_cells"]) > 0

    # map + metrics identity: the mapped phantom equals its companion raster
    _cli("map", "--field", tmp_path / "truth.fld", "--out", tmp_path / "mapped.pgm")
    assert open(tmp_path / "mapped.pgm", "rb").read() == open(tmp_path / "truth.cg.pgm", "rb").read()
    _cli("metrics", "--ref", tmp_path / "truth.cg.pgm", "--test", tmp_path / "mapped.pgm", "--out",
         tmp_path / "id.txt")
    vals = dict(line.rstrip("\n").split(" = ", 1) for line in open(tmp_path / "id.txt"))
    assert float(vals["ssim"]) == 1.0 and float(vals["rmse"]) == 0.0

    # closure: the reconstruction reproduces its measurements
    _cli("project", "--field", tmp_path / "recon.fld", *geo, "--out", tmp_path / "redata.prj")
    re = np.fromfile(tmp_path / "redata.prj", np.float32, offset=40).astype(np.float64)
    nz = data != 0
    assert np.abs(re[nz] / data[nz] - 1.0).max() <= 1e-4


def test_cli_metrics_match_reference(ub, ref, rio, tmp_path):
    """metrics on two rasters: mae / rmse / ssim on the device, area averages
    and sharpness on the host, against the reference library."""
    rng = np.random.default_rng(5)
    a = rng.uniform(0, 1, (24, 20))
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
    rio.write_pgm16(tmp_path / "a.pgm", a, 0.0, 1.0)
    rio.write_pgm16(tmp_path / "b.pgm", b, 0.0, 1.0)
    r = _cli("metrics", "--ref", tmp_path / "a.pgm", "--test", tmp_path / "b.pgm", "--profile-row", 3)
    vals = dict(line.split(" = ", 1) for line in r.stdout.strip().splitlines())
    ia, ib = rio.read_pgm16(tmp_path / "a.pgm"), rio.read_pgm16(tmp_path / "b.pgm")
    assert abs(float(vals["rmse"]) - ref.rmse(ia, ib)) <= 1e-6 * ref.rmse(ia, ib)
    assert abs(float(vals["ssim"]) - ref.ssim(ia, ib)) <= 1e-6
    assert abs(float(vals["area_average.ref"]) - ia.mean()) <= 1e-12
    assert vals["profile.row"] == "3"
