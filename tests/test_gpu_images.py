"""Device image paths beside the resampler: cartesian_to_field
(proj/src/phantom.cpp:165-180), sharpness and intensity_profile
(proj/src/metrics.cpp:138-159), against the oracle restatement (itself pinned
to the reference library by tests/test_oracle.py) and the committed golden
fixtures of the unmodified reference (tests/golden/images.npz)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _spec(ub, n, volume):
    mode = ub.GridMode.Volume3D if volume else ub.GridMode.Slice2D
    return ub.GridSpec(n, 2.0 / n, 2.0 / n, mode)


@pytest.mark.parametrize("n,volume", [(64, False), (16, True), (2, False), (256, False)])
def test_cartesian_to_field_matches_oracle(ub, orc, n, volume):
    spec = _spec(ub, n, volume)
    grid = oracle.OrcGrid.reference(n, volume)
    imgs = np.random.default_rng(n).uniform(0, 2, (spec.slices(), n, n)).astype(np.float32)
    got = ub.cartesian_to_field(imgs, spec)
    want = orc.cartesian_to_field(grid, imgs.astype(np.float64), n)
    assert np.array_equal(got.values.astype(np.float64), want)  # a permutation: bit-exact
    # round trip through the device resampler
    back = ub.field_to_cartesian(got)
    assert np.array_equal(back, imgs)


def test_cartesian_to_field_matches_golden(ub):
    z = np.load(os.path.join(GOLDEN, "images.npz"))
    for key, n, volume in (("2", 16, False), ("3", 8, True)):
        f = ub.cartesian_to_field(z["im" + key].astype(np.float32), _spec(ub, n, volume))
        assert np.array_equal(f.values, z["field" + key].astype(np.float32))


def test_cartesian_to_field_stack_interleaved(ub, orc):
    """S problems at once through the C ABI, device-native interleaved layout"""
    from paper_2208_12964_b200 import uscg

    n, S = 32, 5
    spec = _spec(ub, n, False)
    grid = oracle.OrcGrid.reference(n, False)
    imgs = np.random.default_rng(3).uniform(0, 1, (S, 1, n, n)).astype(np.float32)
    Sp = ub.problem_stride(S)
    out = np.full((spec.cell_count(), Sp), -1.0, np.float32)
    g, keep = spec._c()
    L = ub.load()
    uscg._check(L.uscg_cartesian_to_field(uscg.default_context().h, C.byref(g), imgs.ctypes.data_as(C.c_void_p), S,
                                          n, out.ctypes.data_as(C.c_void_p), uscg.LAYOUT_INTERLEAVED))
    for p in range(S):
        assert np.array_equal(out[:, p].astype(np.float64), orc.cartesian_to_field(grid, imgs[p].astype(np.float64), n))
    assert (out[:, S:] == 0).all()


def test_cartesian_to_field_errors(ub):
    spec = _spec(ub, 16, False)
    with pytest.raises(ub.InvalidArgument, match="slice shape"):
        ub.cartesian_to_field(np.zeros((1, 8, 8), np.float32), spec)
    with pytest.raises(ub.InvalidArgument, match="slice count"):
        ub.cartesian_to_field(np.zeros((2, 16, 16), np.float32), spec)
    m1 = ub.GridSpec(32, 1.0 / 16, 1.0 / 16, ub.GridMode.Slice2D, ring_counts=ub.ring_counts_m1(16))
    with pytest.raises(ub.InvalidArgument, match="reference sector law"):
        ub.cartesian_to_field(np.zeros((1, 32, 32), np.float32), m1)


def test_sharpness_matches_oracle(ub, orc):
    rng = np.random.default_rng(12)
    for shape in [(2, 2), (64, 64), (3, 17), (31, 2), (1024, 1024), (257, 129)]:
        a = rng.uniform(0, 1, shape).astype(np.float32)
        want = orc.sharpness(a.astype(np.float64))
        got = ub.sharpness(a)
        assert abs(got - want) <= 1e-12 * abs(want), shape
    stack = rng.uniform(0, 1, (7, 40, 50)).astype(np.float32)
    got = ub.sharpness(stack)
    for s in range(7):
        want = orc.sharpness(stack[s].astype(np.float64))
        assert abs(got[s] - want) <= 1e-12 * abs(want)
    assert ub.sharpness(np.full((9, 9), 3.0, np.float32)) == 0.0


def test_sharpness_matches_golden(ub):
    z = np.load(os.path.join(GOLDEN, "images.npz"))
    off = 0
    for (r, c), want in zip(z["sharp_shapes"], z["sharpness"]):
        img = z["sharp_pixels"][off:off + r * c].reshape(r, c)
        off += r * c
        # fp32 rasters on the device: compare with the reference on the rounded raster
        exact = img.astype(np.float32).astype(np.float64)
        got = ub.sharpness(img.astype(np.float32))
        if np.array_equal(exact, img):
            assert abs(got - want) <= 1e-12 * max(abs(want), 1e-300)
        else:
            assert abs(got - want) <= 1e-6 * max(abs(want), 1.0)


def test_sharpness_and_profile_errors(ub):
    with pytest.raises(ub.InvalidArgument, match="2x2"):
        ub.sharpness(np.zeros((1, 5), np.float32))
    ramp = np.arange(12, dtype=np.float32).reshape(3, 4)
    assert np.array_equal(ub.intensity_profile(ramp, 0), np.arange(4.0))
    z = np.load(os.path.join(GOLDEN, "images.npz"))
    first = z["sharp_pixels"][: 9 * 13].reshape(9, 13)
    assert np.array_equal(ub.intensity_profile(first.astype(np.float32), 4),
                          z["profile"].astype(np.float32).astype(np.float64))
    for row in (3, -1):
        with pytest.raises(ub.InvalidArgument, match="out of range"):
            ub.intensity_profile(ramp, row)
