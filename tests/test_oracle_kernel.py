"""Pins for the generalized Gaussian kernels of degree n (PAPER Supp. A,
L454-462; reading R29 in DESIGN.md): rho = exp(-(1/2) lambda_n d^n),
lambda_n = r^2 / r^n, r = 3.

* closed forms: n = 2 is the Gaussian exp(-d^2/2) (Eq. 1); the response at
  d = r = 3 is exp(-4.5) for every n (the paper's normalisation);
  log rho_n / log rho_2 = (d/3)^(n-2);
* the opacity-aware extent (Alg. 1 l.3) of degree n: sigma rho_n(k2) = alpha_min;
* ORTHO single Gaussian: alpha(pixel) = sigma exp(-(1/2) lambda_n q^(n/2)) with
  q = D^T A^-1 D the projected marginal's quadratic form (numpy), i.e. the
  3D max response along the ray (the maximiser of a decreasing function of
  the Mahalanobis distance is Eq. 11's tau_max);
* ORTHO: binned == brute force bit for bit for n = 3, 4, 8 (the degree-n
  extent contains the alpha >= alpha_min set).
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import scenegen as S

DEGREES = [1, 2, 3, 4, 5, 8]


@pytest.mark.parametrize("n", DEGREES)
def test_kernel_closed_forms(orc, n):
    assert orc.kernel_lambda(n) == pytest.approx(3.0 ** (2 - n), rel=1e-15)
    assert orc.kernel_response(9.0, n) == pytest.approx(math.exp(-4.5), rel=1e-14)
    for d in (0.3, 1.0, 2.0, 4.5):
        if n == 2:
            assert orc.kernel_response(d * d, n) == pytest.approx(math.exp(-0.5 * d * d), rel=1e-15)
        ratio = math.log(orc.kernel_response(d * d, n)) / (-0.5 * d * d)
        assert ratio == pytest.approx((d / 3.0) ** (n - 2), rel=1e-12)
    assert orc.kernel_response(0.0, n) == 1.0


@pytest.mark.parametrize("n", DEGREES)
def test_extent_level(orc, n):
    scene, cam = S.tiny(2, "pinhole", n=64)
    opt = S.RenderOptions(kernel_degree=n)
    p = orc.preprocess(scene, cam, opt)
    ok = p["reason"] == 0
    assert ok.sum() > 10
    sig = scene.opacities[ok].astype(np.float64)
    resp = np.array([orc.kernel_response(k2, n) for k2 in p["k2"][ok]])
    np.testing.assert_allclose(sig * resp, opt.alpha_min, rtol=1e-12)


@pytest.mark.parametrize("n", [3, 4, 8])
def test_ortho_marginal_identity_degree_n(orc, n):
    rng = np.random.default_rng(31 + n)
    opt = S.RenderOptions(kernel_degree=n)
    cam = S.Camera("ortho", 64, 64, 32.0, 32.0, 32.0, 32.0)
    F = np.diag([32.0, 32.0])
    lam = 3.0 ** (2 - n)
    for _ in range(8):
        mu = np.array([[rng.uniform(-0.6, 0.6), rng.uniform(-0.6, 0.6), 4.0]], np.float32)
        q = rng.standard_normal((1, 4)).astype(np.float32)
        s = np.exp(rng.uniform(math.log(0.03), math.log(0.25), (1, 3))).astype(np.float32)
        sig = np.float32(rng.uniform(0.2, 0.99))
        sc = S.Scene(mu, q, s, np.array([sig], np.float32), np.zeros((1, 1, 3), np.float32), 0)
        r = orc.render(sc, cam, opt)
        Rg = Rotation.from_quat(np.roll(q[0].astype(np.float64) / np.linalg.norm(q[0]), -1)).as_matrix()
        Sig = Rg @ np.diag(s[0].astype(np.float64) ** 2) @ Rg.T
        Ai = np.linalg.inv(F @ Sig[:2, :2] @ F)
        jj, ii = np.mgrid[0:64, 0:64]
        m64 = mu[0].astype(np.float64)
        D = np.stack([ii + 0.5 - (32 + 32 * m64[0]), jj + 0.5 - (32 + 32 * m64[1])], -1)
        qf = np.einsum("hwi,ij,hwj->hw", D, Ai, D)
        al = np.minimum(float(sig) * np.exp(-0.5 * lam * qf ** (0.5 * n)), opt.alpha_max)
        exp = np.where(al >= opt.alpha_min, al, 0.0)
        keep = np.abs(al - opt.alpha_min) > 1e-9
        assert (exp[keep] > 0).sum() > 4
        np.testing.assert_allclose(r["alpha"][keep], exp[keep], atol=1e-6)


@pytest.mark.parametrize("n", [3, 4, 8])
def test_ortho_binned_equals_brute_degree_n(orc, n):
    opt = S.RenderOptions(kernel_degree=n)
    for seed in range(6):
        sc, cam = S.tiny(seed, "ortho")
        a = orc.render(sc, cam, opt)
        b = orc.render(sc, cam, opt, brute=True)
        assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["alpha"], b["alpha"])


def test_degree_changes_footprint(orc):
    """Higher degree: denser core, narrower fall-off (Fig. 8): the extent level
    k2 shrinks with n for sigma well above alpha_min... and alpha at d < 3 rises."""
    assert orc.kernel_response(4.0, 8) > orc.kernel_response(4.0, 4) > orc.kernel_response(4.0, 2)
    assert orc.kernel_response(16.0, 8) < orc.kernel_response(16.0, 4) < orc.kernel_response(16.0, 2)
