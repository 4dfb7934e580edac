"""Pins for O8, the projection-quality comparison (PAPER Supp. C, L522-588;
reading R31): UT vs EWA vs Monte Carlo, KL divergences.

* the counter-based normal generator: a Python re-implementation of its spec
  (splitmix64 + Box-Muller) reproduces it exactly; moments of 3e5 draws;
* KL(N0 || N1) against numerical integration on a grid, KL(N || N) = 0;
* ORTHO camera (affine): UT and EWA both equal the analytic image of the
  Gaussian, and the Monte-Carlo moments equal the affine image of the
  generator's own sample moments (numpy);
* RS camera: RS-aware UT tracks the RS-aware MC reference much better than the
  RS-unaware EWA (the paper's central qualitative claim, Fig. 10/12).
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import scenegen as S

MASK = (1 << 64) - 1


def _mix(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def _normal3_py(seed, gid, s):
    u = [((_mix(seed ^ _mix((gid << 24) ^ (s << 2) ^ k)) >> 11) + 0.5) / 9007199254740992.0 for k in range(4)]
    r0, r1 = math.sqrt(-2 * math.log(u[0])), math.sqrt(-2 * math.log(u[2]))
    return np.array([r0 * math.cos(2 * math.pi * u[1]), r0 * math.sin(2 * math.pi * u[1]), r1 * math.cos(2 * math.pi * u[3])])


def test_generator_spec_and_moments(orc):
    for seed, gid, s in [(0, 0, 0), (1, 5, 7), (123456789, 2999999, 499), (2 ** 63 + 5, 17, 3)]:
        np.testing.assert_allclose(orc.normal3(seed, gid, s), _normal3_py(seed, gid, s), rtol=0, atol=1e-14)
    z = np.array([orc.normal3(7, g, s) for g in range(200) for s in range(500)])
    assert np.abs(z.mean(0)).max() < 0.01
    np.testing.assert_allclose(np.cov(z.T), np.eye(3), atol=0.012)


def test_kl_closed_form(orc):
    rng = np.random.default_rng(3)
    g = np.array([1.0, -2.0, 2.0, 0.3, 1.5])
    assert abs(orc.kl2(g, g)) < 1e-15
    for _ in range(5):
        def rand_g():
            A = rng.normal(size=(2, 2))
            C = A @ A.T + 0.5 * np.eye(2)
            return np.array([rng.normal(), rng.normal(), C[0, 0], C[0, 1], C[1, 1]])
        g0, g1 = rand_g(), rand_g()

        def pdf(g, X, Y):
            C = np.array([[g[2], g[3]], [g[3], g[4]]])
            Ci = np.linalg.inv(C)
            dx, dy = X - g[0], Y - g[1]
            q = Ci[0, 0] * dx * dx + 2 * Ci[0, 1] * dx * dy + Ci[1, 1] * dy * dy
            return np.exp(-0.5 * q) / (2 * np.pi * math.sqrt(np.linalg.det(C)))
        xs = np.linspace(g0[0] - 9 * math.sqrt(g0[2]), g0[0] + 9 * math.sqrt(g0[2]), 1501)
        ys = np.linspace(g0[1] - 9 * math.sqrt(g0[4]), g0[1] + 9 * math.sqrt(g0[4]), 1501)
        X, Y = np.meshgrid(xs, ys)
        p, q = pdf(g0, X, Y), pdf(g1, X, Y)
        integrand = np.where(p > 1e-300, p * (np.log(np.maximum(p, 1e-300)) - np.log(np.maximum(q, 1e-300))), 0.0)
        num = integrand.sum() * (xs[1] - xs[0]) * (ys[1] - ys[0])
        assert orc.kl2(g0, g1) == pytest.approx(num, rel=2e-4, abs=1e-7)


def test_ortho_affine_exact(orc):
    """ORTHO: g is affine, so UT = EWA = the exact image and MC = the affine
    image of the generator's sample moments."""
    rng = np.random.default_rng(9)
    n = 12
    means = np.column_stack([rng.uniform(-0.5, 0.5, (n, 2)), rng.uniform(3, 5, n)]).astype(np.float32)
    q = rng.standard_normal((n, 4)).astype(np.float32)
    s = np.exp(rng.uniform(math.log(0.03), math.log(0.3), (n, 3))).astype(np.float32)
    sc = S.Scene(means, q, s, np.full(n, 0.9, np.float32), np.zeros((n, 1, 3), np.float32), 0)
    cam = S.Camera("ortho", 64, 64, 32.0, 32.0, 32.0, 32.0)
    out = orc.projection_quality(sc, cam, S.RenderOptions(), n_mc=300, seed=11)
    F = np.diag([32.0, 32.0])
    for i in range(n):
        assert out["valid"][i] == 1
        Rg = Rotation.from_quat(np.roll(q[i].astype(np.float64) / np.linalg.norm(q[i]), -1)).as_matrix()
        L = F @ (Rg @ np.diag(s[i].astype(np.float64)))[:2]        # 2x3 affine map of z
        m = np.array([32 + 32 * float(means[i, 0]), 32 + 32 * float(means[i, 1])])
        C = L @ L.T
        exact = np.array([m[0], m[1], C[0, 0], C[0, 1], C[1, 1]])
        np.testing.assert_allclose(out["ut"][i], exact, rtol=1e-10, atol=1e-9)
        np.testing.assert_allclose(out["ewa"][i], exact, rtol=1e-6, atol=1e-6)  # (central differences)
        z = np.array([_normal3_py(11, i, k) for k in range(300)])
        y = z @ L.T
        mu_s = y.mean(0)
        cov_s = (y - mu_s).T @ (y - mu_s) / 300
        mc = np.array([m[0] + mu_s[0], m[1] + mu_s[1], cov_s[0, 0], cov_s[0, 1], cov_s[1, 1]])
        np.testing.assert_allclose(out["mc"][i], mc, rtol=1e-9, atol=1e-9)


def test_rs_ut_beats_rs_unaware_ewa(orc):
    scene, cam = S.tiny(2, "rs", n=64)
    out = orc.projection_quality(scene, cam, S.RenderOptions(), n_mc=500, seed=3)
    v = out["valid"] == 1
    assert v.sum() > 40
    kl_ut, kl_ewa = np.median(out["kl_ut"][v]), np.median(out["kl_ewa"][v])
    print(f"RS: median KL UT {kl_ut:.2e}  EWA {kl_ewa:.2e}")
    assert kl_ut < 0.05 and kl_ewa > 3 * kl_ut
