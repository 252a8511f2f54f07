"""File formats and the CLI drop-in, on the CPU.

include/uscg_b200_io.hpp writes the reference's .fld / .prj / .pgm files and
their .meta sidecars; every file it writes is compared byte for byte with the
reference's own writer (proj/src/io.cpp, built into oracle/_ref), and each
side reads the other's files. The CLI binary's argument and I/O error paths
(exit codes of proj/src/cli.cpp:523-543) need no GPU.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_dp = C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def hio(tmp_path_factory):
    """tests/io_harness.cpp (our header behind a C ABI), built with g++."""
    out = tmp_path_factory.mktemp("io") / "libio_harness.so"
    cxx = os.environ.get("CXX", "g++")
    subprocess.run([cxx, "-std=c++17", "-O2", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "io_harness.cpp"), "-o", str(out), "-Wl,--exclude-libs,ALL"],
                   check=True)
    L = C.CDLL(str(out))
    sp = C.POINTER(C.c_char_p)
    L.io_write_field.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_int, _dp, sp, sp, C.c_int,
                                 C.c_char_p, C.c_int]
    L.io_read_field.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, C.c_longlong, C.c_char_p,
                                C.c_int]
    L.io_write_projections.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp,
                                       _dp, sp, sp, C.c_int, C.c_char_p, C.c_int]
    L.io_read_projections.argtypes = [C.c_char_p, C.POINTER(C.c_int), _dp, _dp, C.c_longlong, C.c_char_p, C.c_int]
    L.io_write_pgm16.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp, C.c_double, C.c_double, sp, sp, C.c_int,
                                 C.c_char_p, C.c_int]
    L.io_read_pgm16.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, C.c_longlong, C.c_char_p,
                                C.c_int]
    return L


@pytest.fixture(scope="module")
def rio():
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("reference library not built")
    return oracle.RefIO(oracle.Ref())


def _kv(side):
    return oracle._kv(side)


def _call(fn, *args):
    err = C.create_string_buffer(512)
    rc = fn(*args, err, 512)
    return rc, err.value.decode()


def _ptr(a):
    return a.ctypes.data_as(_dp)


def _same_files(a, b):
    assert open(a, "rb").read() == open(b, "rb").read(), (a, b)
    assert open(str(a) + ".meta", "rb").read() == open(str(b) + ".meta", "rb").read()


SIDE = {"provenance": "reconstruct from data.prj", "config.beta": "1", "config.threads": "1"}


@pytest.mark.parametrize("n,volume,r,h", [(16, False, 0.125, 0.125), (8, True, 0.25, 0.1), (6, False, 2 / 6, 2 / 6)])
def test_field_file_bytes_match_reference(hio, rio, tmp_path, n, volume, r, h):
    rng = np.random.default_rng(n)
    cells = n * n * (n if volume else 1)
    vals = rng.uniform(0, 3, cells).astype(np.float32).astype(np.float64)
    ours, ref = tmp_path / "ours.fld", tmp_path / "ref.fld"
    rc, err = _call(hio.io_write_field, str(ours).encode(), n, r, h, int(volume), _ptr(vals), *_kv(SIDE))
    assert rc == 0, err
    rio.write_field(ref, n, r, h, volume, vals, SIDE)
    _same_files(ours, ref)
    out = np.zeros(cells)
    nn, sl = C.c_int(), C.c_int()
    rc, err = _call(hio.io_read_field, str(ref).encode(), C.byref(nn), C.byref(sl), _ptr(out), cells)
    assert rc == 0, err
    assert nn.value == n and sl.value == (n if volume else 1)
    assert np.array_equal(out, vals)


def test_projection_file_bytes_match_reference(hio, rio, tmp_path):
    rng = np.random.default_rng(7)
    views, du, dv = 6, 9, 3
    data = rng.uniform(0, 5, views * du * dv).astype(np.float32).astype(np.float64)
    src, ctr = np.array([-3.0, 0.0, 0.1]), np.array([10.0, 0.5, 0.0])
    ours, ref = tmp_path / "ours.prj", tmp_path / "ref.prj"
    rc, err = _call(hio.io_write_projections, str(ours).encode(), views, du, dv, 0.1, 0.3, _ptr(src), _ptr(ctr),
                    _ptr(data), *_kv(SIDE))
    assert rc == 0, err
    rio.write_projections(ref, views, du, dv, 0.1, 0.3, src, ctr, data, SIDE)
    _same_files(ours, ref)
    dims = (C.c_int * 3)()
    geom = np.zeros(8)
    back = np.zeros(data.size)
    rc, err = _call(hio.io_read_projections, str(ref).encode(), dims, _ptr(geom), _ptr(back), back.size)
    assert rc == 0, err
    assert list(dims) == [views, du, dv] and np.array_equal(back, data)
    assert np.array_equal(geom, [0.1, 0.3, -3.0, 0.0, 0.1, 10.0, 0.5, 0.0])


@pytest.mark.parametrize("shape,window", [((5, 7), (0.0, 2.5)), ((16, 16), (-1.0, 1.0)), ((1, 3), (0.2, 0.3))])
def test_pgm16_bytes_match_reference(hio, rio, tmp_path, shape, window):
    rng = np.random.default_rng(shape[0])
    img = rng.uniform(window[0] - 0.2, window[1] + 0.2, shape)  # clamps at both ends
    ours, ref = tmp_path / "ours.pgm", tmp_path / "ref.pgm"
    rc, err = _call(hio.io_write_pgm16, str(ours).encode(), shape[0], shape[1], _ptr(img), window[0], window[1],
                    *_kv({"slice": "0", "slices": "1"}))
    assert rc == 0, err
    rio.write_pgm16(ref, img, window[0], window[1], {"slice": "0", "slices": "1"})
    _same_files(ours, ref)
    rows, cols = C.c_int(), C.c_int()
    back = np.zeros(img.size)
    rc, err = _call(hio.io_read_pgm16, str(ref).encode(), C.byref(rows), C.byref(cols), _ptr(back), back.size)
    assert rc == 0, err
    assert (rows.value, cols.value) == shape
    assert np.array_equal(back.reshape(shape), rio.read_pgm16(ours))


def test_format_errors_follow_the_reference(hio, rio, tmp_path):
    vals = np.ones(16)
    good = tmp_path / "f.fld"
    rio.write_field(good, 4, 0.5, 0.5, False, vals, {})
    raw = open(good, "rb").read()
    bad = tmp_path / "t.fld"
    open(bad, "wb").write(raw[:30])
    open(str(bad) + ".meta", "w").write(open(str(good) + ".meta").read())
    out = np.zeros(16)
    nn, sl = C.c_int(), C.c_int()
    rc, err = _call(hio.io_read_field, str(bad).encode(), C.byref(nn), C.byref(sl), _ptr(out), 16)
    assert rc == 1 and "truncated at byte" in err
    open(bad, "wb").write(b"USCGPRJ\0" + raw[8:])
    rc, err = _call(hio.io_read_field, str(bad).encode(), C.byref(nn), C.byref(sl), _ptr(out), 16)
    assert rc == 1 and "magic mismatch at byte 0" in err
    # negative measurement: ProjectionSet::validate
    data = np.array([1.0, -1.0])
    rc, err = _call(hio.io_write_projections, str(tmp_path / "p.prj").encode(), 1, 2, 1, 0.1, 0.1,
                    _ptr(np.zeros(3)), _ptr(np.array([1.0, 0, 0])), _ptr(data), *_kv({}))
    assert rc == 2 and "negative measurement" in err


def _cli(*args):
    from paper_2208_12964_b200 import _build
    _build.build()
    return subprocess.run([_build.CLI, *args], capture_output=True, text=True)


def test_cli_error_paths(tmp_path):
    """cli.cpp:523-543 exit codes; these paths never reach the device."""
    assert _cli("no-such-command").returncode == 1
    r = _cli("reconstruct", "--out", str(tmp_path / "x.fld"))
    assert r.returncode == 1 and "--proj is required" in r.stderr
    r = _cli("map", "--field", str(tmp_path / "missing.fld"), "--out", str(tmp_path / "m.pgm"))
    assert r.returncode == 1 and "cannot open" in r.stderr
    r = _cli("project", "--field", "a.fld", "--bogus", "1", "--out", "b.prj")
    assert r.returncode == 1 and "unknown option" in r.stderr
    r = _cli("phantom", "--kind", "shepp-logan-2d", "--n", "16", "--out", str(tmp_path / "p.fld"))
    assert r.returncode == 1 and "--table" in r.stderr
