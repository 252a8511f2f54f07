"""The C-ABI library (CPU checks, no GPU): it loads, exports every symbol
include/uscg_b200.h declares, fails loudly (no CPU fallback) without a
device, and its host-only entry points behave like the reference."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from conftest import has_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "uscg_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(uscg_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol(ub):
    lib = ub.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/uscg_b200.h but not exported"
    assert set(ub.uscg.EXPORTS) <= set(syms)
    assert b"sm_100a" in lib.uscg_version()


def test_library_is_sm100a_code(ub):
    """The .so carries sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ub.uscg.library_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device(ub):
    with pytest.raises(ub.NoDevice):
        ub.Context(0)


def test_problem_stride(ub):
    # chunks of up to 8 problems; S_pad is a multiple of the chunk width
    assert ub.problem_stride(1) == 1
    assert ub.problem_stride(3) == 4
    assert ub.problem_stride(8) == 8
    assert ub.problem_stride(37) == 40
    assert ub.problem_stride(128) == 128


def test_first_view_rays_flat_matches_reference_formula(ub, orc):
    """uscg_first_view_rays (host) == ScanGeometry::detector_position
    (proj/src/scan.cpp:27-36), restated in the oracle, bit for bit."""
    geom = ub.ScanGeometry(source=(-3, 0.25, 0.1), detector_center=(10, -0.5, 0.2), det_u=17, det_v=9,
                           spacing_u=0.1, spacing_v=0.13, views=5)
    s, d = geom.first_view_rays()
    os_, od = orc.rays_flat((-3, 0.25, 0.1), (10, -0.5, 0.2), 17, 9, 0.1, 0.13)
    assert np.array_equal(s, os_) and np.array_equal(d, od)


def test_first_view_rays_arc_and_parallel_match_restatement(ub, orc):
    geom = ub.ScanGeometry(source=(-3, 0, 0), detector_center=(1.5, 0, 0), det_u=64, spacing_u=0.6,
                           views=4, detector=ub.Detector.Arc)
    s, d = geom.first_view_rays()
    os_, od = orc.rays_arc((-3, 0, 0), (1.5, 0, 0), 64, 0.6)
    assert np.array_equal(s, os_) and np.array_equal(d, od)
    geom = ub.ScanGeometry(source=(-2, 0, 0), detector_center=(2, 0, 0), det_u=32, spacing_u=1 / 16, views=4,
                           detector=ub.Detector.Parallel)
    s, d = geom.first_view_rays()
    os_, od = orc.rays_parallel(32, 1 / 16, 2.0)
    assert np.array_equal(s, os_) and np.array_equal(d, od)


def test_scan_validation_errors(ub):
    """ScanGeometry::validate (proj/src/scan.cpp:9-24) -> InvalidArgument."""
    good = dict(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=5, spacing_u=0.1, views=3)
    for bad in (dict(views=0), dict(det_u=0), dict(spacing_u=0.0), dict(det_v=3, spacing_v=0.0),
                dict(detector_center=(-8, 0, 0))):
        with pytest.raises(ub.InvalidArgument):
            ub.ScanGeometry(**{**good, **bad}).first_view_rays()


def test_uspg_to_cg_map_rejects_odd_without_device(ub):
    if has_gpu():
        pytest.skip("device path tested in test_gpu_parity")
    with pytest.raises((ub.DomainError, ub.NoDevice)):
        ub.uspg_to_cg_map(5)


def test_header_compiles_as_c_and_cpp(tmp_path):
    for lang, comp in (("c", "gcc"), ("cpp", "g++")):
        src = tmp_path / f"t.{lang}"
        src.write_text('#include "uscg_b200.h"\nint main(void){uscg_grid g; (void)g; return 0;}\n')
        r = os.system(f"{comp} -I{ROOT}/include -c {src} -o {tmp_path}/t_{lang}.o")
        assert r == 0


def test_cpp_mirror_header_compiles(tmp_path):
    """include/uscg_b200.hpp (the C++ mirror of the reference API) compiles
    and links against the library."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "uscg_b200.hpp"\n'
                   'int main(){ auto s = uscg_b200::GridSpec::square_2d(16);'
                   ' return s.rings() == 8 ? 0 : 1; }\n')
    lib = os.path.join(ROOT, "paper_2208_12964_b200", "lib")
    r = os.system(f"g++ -std=c++17 -I{ROOT}/include {src} -L{lib} -luscg_b200 -Wl,-rpath,{lib} "
                  f"-o {tmp_path}/t && {tmp_path}/t")
    assert r == 0
