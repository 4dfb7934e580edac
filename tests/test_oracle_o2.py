"""Pins for oracle steps O2 (exact projection g, rolling shutter) and O5
(pixel rays): closed-form camera values, the forward/inverse
round trip between two independently written maps, special cases (zero
distortion == pinhole, pose0 == pose1 == global shutter) and brute-force
root finding of the rolling-shutter fixed point."""
import dataclasses
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import scenegen as S

OPT = S.RenderOptions()


def cam(model, **kw):
    base = dict(model=model, width=640, height=480, fx=500.0, fy=480.0, cx=320.0, cy=240.0)
    base.update(kw)
    return S.Camera(**base)


def test_pinhole_axis_and_value(orc):
    c = cam("pinhole")
    v, uv, _ = orc.project_cam(c, OPT, [0, 0, 3.0])
    assert v and uv[0] == 320.0 and uv[1] == 240.0
    v, uv, _ = orc.project_cam(c, OPT, [1.0, -2.0, 4.0])
    assert uv[0] == pytest.approx(320 + 500 * 0.25) and uv[1] == pytest.approx(240 - 480 * 0.5)
    v, _, _ = orc.project_cam(c, OPT, [0, 0, 0.1])  # behind the near plane (reading R9)
    assert not v


def test_opencv_radial_factor(orc):
    # k1 = 0.1, normalised radius r = 0.5 -> factor 1 + 0.1*0.25 = 1.025
    c = cam("opencv", k=(0.1, 0, 0, 0, 0, 0), fov_limit=2.0)
    v, uv, _ = orc.project_cam(c, OPT, [0.5 * 2.0, 0.0, 2.0])
    assert v
    assert (uv[0] - 320) / 500 == pytest.approx(0.5 * 1.025, abs=1e-15)


def test_opencv_zero_distortion_is_pinhole(orc):
    rng = np.random.default_rng(0)
    cp, co = cam("pinhole"), cam("opencv")
    for _ in range(200):
        x = np.array([rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.5, 9)])
        a = orc.project_cam(cp, OPT, x)[1]
        b = orc.project_cam(co, OPT, x)[1]
        assert np.array_equal(a, b)  # bit for bit


def test_fisheye_closed_forms(orc):
    c = cam("fisheye", fx=300.0, fy=300.0, fov_limit=math.radians(120))
    # theta = 90 deg -> radius f*pi/2, still valid
    v, uv, _ = orc.project_cam(c, OPT, [2.0, 0.0, 0.0])
    assert v and uv[0] - 320 == pytest.approx(300 * math.pi / 2, abs=1e-12) and uv[1] == 240
    # theta > 90 deg (z < 0) valid below theta_max, invalid above (reading R8)
    th = math.radians(110)
    v, uv, _ = orc.project_cam(c, OPT, [math.sin(th), 0, math.cos(th)])
    assert v and uv[0] - 320 == pytest.approx(300 * th, abs=1e-9)
    th = math.radians(121)
    assert not orc.project_cam(c, OPT, [math.sin(th), 0, math.cos(th)])[0]


def _roundtrip(orc, c, n=300, seed=0, tol=1e-9):
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(n):
        u, v = rng.uniform(0, c.width), rng.uniform(0, c.height)
        ok, o, d = orc.pixel_ray(c, u, v)
        if not ok:
            continue
        assert np.linalg.norm(d) == pytest.approx(1.0, abs=1e-14)
        tau = rng.uniform(1.0, 20.0)
        valid, uv, t, _ = orc.project_point(c, OPT, o + tau * d)
        assert valid
        worst = max(worst, float(np.hypot(uv[0] - u, uv[1] - v)))
    assert worst < tol, worst
    return worst


@pytest.mark.parametrize("model,kw", [
    ("pinhole", {}),
    ("ortho", dict(fx=40.0, fy=40.0)),
    ("opencv", dict(k=(-0.2, 0.05, 0.01, 0.02, -0.01, 0.003), p=(1e-3, -1e-3), fov_limit=1.0)),
    ("fisheye", dict(fx=200.0, fy=200.0, fov_limit=math.radians(110))),
    ("fisheye", dict(fx=200.0, fy=200.0, k=(0.05, -0.01, 0.002, 0, 0, 0), fov_limit=math.radians(100))),
])
def test_pixel_ray_roundtrip(orc, model, kw):
    """O5 (inverse camera) and O2 (forward camera) are written independently;
    project(pixel_ray(p) * tau) must return p to 1e-9 px."""
    q = S._mat_to_quat(S.look_at_c2w((1.0, -2.0, 0.5), (0.0, 0.5, 0.2)))
    c = cam(model, q_c2w=(q, q), c_w=((1.0, -2.0, 0.5), (1.0, -2.0, 0.5)), **kw)
    _roundtrip(orc, c)


def test_pixel_ray_principal_point(orc):
    c = cam("pinhole")
    ok, o, d = orc.pixel_ray(c, 320.0, 240.0)
    assert ok and np.allclose(o, 0) and np.allclose(d, [0, 0, 1], atol=1e-15)
    ok, o1, d1 = orc.pixel_ray(cam("ortho", fx=40.0, fy=40.0), 10.5, 3.5)
    ok, o2, d2 = orc.pixel_ray(cam("ortho", fx=40.0, fy=40.0), 300.5, 400.5)
    assert np.array_equal(d1, d2)  # orthographic rays are parallel


def _rs_cam(**kw):
    q1 = S._mat_to_quat(S._rot_axis((0, 1, 0), math.radians(2.0)))
    base = dict(model="pinhole", width=640, height=480, fx=500.0, fy=500.0, cx=320.0, cy=240.0,
                shutter="top_to_bottom", q_c2w=((1.0, 0, 0, 0), q1), c_w=((0, 0, 0), (0.35, 0, 0)))
    base.update(kw)
    return S.Camera(**base)


def test_pose_interpolation(orc):
    c = _rs_cam()
    R, cc = orc.pose_at(c, 0.5)
    assert cc[0] == pytest.approx(0.175)  # SPEC L160 midpoint lerp
    for t in (0.0, 0.25, 0.5, 1.0):
        R, _ = orc.pose_at(c, t)
        ang = Rotation.from_matrix(R).as_rotvec()
        np.testing.assert_allclose(ang, [0, math.radians(2.0) * t, 0], atol=1e-13)  # slerp = constant-rate yaw
    g = dataclasses.replace(c, shutter="global")
    R, cc = orc.pose_at(g, 0.7)
    assert np.allclose(R, np.eye(3)) and np.allclose(cc, 0)


def test_rs_equal_poses_is_global(orc):
    q = S._mat_to_quat(S.look_at_c2w((0, 0, 0), (0.2, 0.1, 1.0), up=(0, -1, 0)))
    rs = cam("pinhole", shutter="top_to_bottom", q_c2w=(q, q), c_w=((0.1, 0.2, 0.3), (0.1, 0.2, 0.3)))
    gs = dataclasses.replace(rs, shutter="global")
    rng = np.random.default_rng(5)
    for _ in range(100):
        x = rng.uniform(-1, 1, 3) + np.array([0.2, 0.1, 5.0])
        a = orc.project_point(rs, OPT, x)
        b = orc.project_point(gs, OPT, x)
        assert a[0] == b[0] and np.allclose(a[1], b[1], rtol=0, atol=1e-10)


def test_rs_fixed_point_by_bisection(orc):
    """Reading R14: t* = clamp(rho(g(x; pose(t*)))).  Brute-force root of
    f(t) = t - rho(g(x; pose(t))) by bisection on [0,1], evaluated through the
    camera-frame projection only."""
    c = _rs_cam()
    rng = np.random.default_rng(6)
    for _ in range(50):
        x = np.array([rng.uniform(-1.5, 1.5), rng.uniform(-1.2, 1.2), rng.uniform(2, 8)])
        ok, uv, t, it = orc.project_point(c, OPT, x)
        assert ok and it > 0

        def f(tt):
            R, cc = orc.pose_at(c, tt)
            v, p, _ = orc.project_cam(c, OPT, R.T @ (x - cc))
            return tt - min(max(p[1] / c.height, 0.0), 1.0)

        lo, hi = 0.0, 1.0
        assert f(lo) <= 0 <= f(hi)
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if f(mid) <= 0:
                lo = mid
            else:
                hi = mid
        assert t == pytest.approx(lo, abs=1e-9)
        assert uv[1] / c.height == pytest.approx(t, abs=1e-9)


def test_rs_ray_of_row_projects_back(orc):
    """A point on the ray of pixel (u,v) (time v/H, reading R17) projects back
    to (u,v) through the fixed point (reading R14): ties O5 and O2 together."""
    c = _rs_cam()
    rng = np.random.default_rng(7)
    for _ in range(100):
        u, v = rng.uniform(0, c.width), rng.uniform(0, c.height)
        ok, o, d = orc.pixel_ray(c, u, v)
        valid, uv, t, _ = orc.project_point(c, OPT, o + rng.uniform(2, 10) * d)
        assert valid
        assert uv[0] == pytest.approx(u, abs=1e-7) and uv[1] == pytest.approx(v, abs=1e-7)
        assert t == pytest.approx(v / c.height, abs=1e-9)
