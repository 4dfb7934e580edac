"""Hand-computed pins for the oracle's depth key (O3.7, reading R13) and SH
view direction (O3.8, reading R18) -- VERDICT r1 "What's weak" #1.

* Depth key (R13, "sorts them globally"): the camera-frame
  DISTANCE ||x_c|| of mu at mu's own shutter time t*_0.  The cases are built so
  that the plausible mistakes give other numbers: view-space z instead of the
  distance, the pose at t = 0 (or t = 1) instead of t*_0.
* SH direction (R18): d = normalize(mu - c(t*_0)).  A Gaussian
  with only band-1 coefficients has the closed-form colour
  0.5 + sum_b c_b Y_b(d), Y_1 = -C1 y, Y_2 = C1 z, Y_3 = -C1 x,
  C1 = sqrt(3 / (4 pi)) (the real SH basis of 3DGS, R19); a flipped direction
  (c - mu) flips every band-1 term.

Rolling shutter: a pure x-translation of the camera leaves y_c and z_c of any
point unchanged, so its row v = fy y_c / z_c + cy -- and with it the shutter
time t* = v / H (top-to-bottom, R16) -- are known in closed form.
"""
import math

import numpy as np
import pytest

import scenegen as S

C1 = math.sqrt(3.0 / (4.0 * math.pi))


def _one(mu, sh1=None, deg=0):
    nc = (deg + 1) ** 2
    sh = np.zeros((1, nc, 3), np.float32)
    if sh1 is not None:
        for b in range(1, 4):
            sh[0, b, :] = sh1[b - 1]
    # small, round Gaussian (every sigma point valid), identity rotation
    return S.Scene(np.asarray([mu], np.float32), np.asarray([[1, 0, 0, 0]], np.float32),
                   np.full((1, 3), 0.01, np.float32), np.full(1, 0.9, np.float32), sh, deg)


def _pinhole(c0, c1=None, shutter="global"):
    c1 = c0 if c1 is None else c1
    return S.Camera("pinhole", 100, 100, 100.0, 100.0, 50.0, 50.0, shutter=shutter,
                    q_c2w=((1, 0, 0, 0), (1, 0, 0, 0)), c_w=(tuple(c0), tuple(c1)))


def test_depth_key_is_distance_global(orc):
    """c = (1,2,3), mu = (4,6,15): x_c = (3,4,12), distance 13 (view-space z
    would be 12)."""
    p = orc.preprocess(_one((4.0, 6.0, 15.0)), _pinhole((1.0, 2.0, 3.0)), S.RenderOptions())
    assert p["reason"][0] == 0
    assert p["depth"][0] == pytest.approx(13.0, rel=0, abs=1e-6)  # fp32 inputs are exact here


def test_depth_key_rolling_shutter_own_time(orc):
    """c(t) = (t, 0, 0), mu = (0.5, 1, 4): v = 100 * 1/4 + 50 = 75 for every
    t, so t*_0 = 0.75 and x_c = (0.5 - 0.75, 1, 4):
    depth = sqrt(0.0625 + 1 + 16) = sqrt(17.0625).  Pose at t = 0 would give
    sqrt(17.25), at t = 1 sqrt(17.25), view-space z would give 4."""
    cam = _pinhole((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), shutter="top_to_bottom")
    p = orc.preprocess(_one((0.5, 1.0, 4.0)), cam, S.RenderOptions())
    assert p["reason"][0] == 0
    assert p["t0"][0] == pytest.approx(0.75, abs=1e-12)
    # (vy is the UT mean, not g(mu): it carries the O(s^2) UT bias -- not asserted here)
    assert p["depth"][0] == pytest.approx(math.sqrt(17.0625), abs=1e-9)
    assert abs(p["depth"][0] - math.sqrt(17.25)) > 1e-3


def test_depth_key_rolling_shutter_off_axis_bottom_to_top(orc):
    """bottom-to-top shutter (t = 1 - v/H), c(t) = (2t, 0, 0) + (0, 0, -1),
    mu = (3, -1, 4): x_c(t) = (3 - 2t, -1, 5), v = 100 (-1/5) + 50 = 30,
    t*_0 = 1 - 0.3 = 0.7, depth = sqrt(1.6^2 + 1 + 25)."""
    cam = _pinhole((0.0, 0.0, -1.0), (2.0, 0.0, -1.0), shutter="bottom_to_top")
    p = orc.preprocess(_one((3.0, -1.0, 4.0)), cam, S.RenderOptions())
    assert p["reason"][0] == 0
    assert p["t0"][0] == pytest.approx(0.7, abs=1e-12)
    assert p["depth"][0] == pytest.approx(math.sqrt(1.6 ** 2 + 1 + 25), abs=1e-9)


def _band1_rgb(d, sh1):
    """closed-form colour: 0.5 + sum_b c_b Y_b(d) per channel (clamped >= 0)."""
    x, y, z = d
    Y = (-C1 * y, C1 * z, -C1 * x)
    return [max(0.0, 0.5 + sum(sh1[b][ch] * Y[b] for b in range(3))) for ch in range(3)]


def test_sh_band1_direction_global(orc):
    """c = (1,2,3), mu = c + (2,3,6): d = (2,3,6)/7.  Only band-1 coefficients
    set (one basis function per channel)."""
    sh1 = [(0.5, 0.0, 0.0), (0.0, 0.5, 0.0), (0.0, 0.0, 0.5)]
    p = orc.preprocess(_one((3.0, 5.0, 9.0), sh1, deg=1), _pinhole((1.0, 2.0, 3.0)), S.RenderOptions())
    assert p["reason"][0] == 0
    want = _band1_rgb((2 / 7, 3 / 7, 6 / 7), sh1)
    assert want == pytest.approx([0.5 - 0.5 * C1 * 3 / 7, 0.5 + 0.5 * C1 * 6 / 7, 0.5 - 0.5 * C1 * 2 / 7])
    np.testing.assert_allclose(p["rgb"][0], want, rtol=0, atol=1e-12)
    flipped = _band1_rgb((-2 / 7, -3 / 7, -6 / 7), sh1)
    assert np.abs(np.asarray(flipped) - p["rgb"][0]).max() > 0.1


def test_sh_band1_direction_rolling_shutter(orc):
    """The SH direction is taken at mu's own shutter time: c(t) = (t,0,0),
    mu = (0.5, 1, 4), t*_0 = 0.75 -> d = (-0.25, 1, 4)/sqrt(17.0625)."""
    sh1 = [(0.7, 0.0, 0.0), (0.0, 0.7, 0.0), (0.0, 0.0, 0.7)]
    cam = _pinhole((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), shutter="top_to_bottom")
    p = orc.preprocess(_one((0.5, 1.0, 4.0), sh1, deg=1), cam, S.RenderOptions())
    n = math.sqrt(17.0625)
    want = _band1_rgb((-0.25 / n, 1 / n, 4 / n), sh1)
    np.testing.assert_allclose(p["rgb"][0], want, rtol=0, atol=1e-7)  # (mu in fp32: 0.5, 1, 4 exact)
    at0 = _band1_rgb((0.5 / math.sqrt(17.25), 1 / math.sqrt(17.25), 4 / math.sqrt(17.25)), sh1)
    assert abs(at0[2] - p["rgb"][0][2]) > 1e-2  # the t = 0 pose is distinguishable


def test_sh_band1_clamp(orc):
    """A band-1 term below -0.5 is clamped to 0 (reading R19)."""
    sh1 = [(0.0, 0.0, 0.0), (-2.0, 0.0, 0.0), (0.0, 0.0, 0.0)]  # red: 0.5 - 2 C1 z, z = 6/7
    p = orc.preprocess(_one((3.0, 5.0, 9.0), sh1, deg=1), _pinhole((1.0, 2.0, 3.0)), S.RenderOptions())
    assert p["rgb"][0][0] == 0.0
    assert p["rgb"][0][1] == pytest.approx(0.5, abs=1e-12)
