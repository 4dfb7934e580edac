"""Pins for oracle steps O5/O6 (Eq. 11 max response, Eq. 5 compositing) and
the end-to-end render:

* Eq. 11 vs golden-section maximisation of rho(o + tau d) with Sigma^-1 from
  numpy (independent of the canonical-space form), SPEC worked values;
* compositing worked values (tests/golden/compositing.json) rendered through
  the full pipeline with an ORTHO camera whose rays pass exactly through mu;
* conservation sum(alpha_i T_i) + T = 1, T in [0,1], alpha <= 1 - T_min;
* ORTHO: binned render == brute force bit for bit (UT ellipse is the exact
  silhouette of an affine image); per-pixel alpha == the Gaussian marginal
  sigma exp(-1/2 D^T (F P R^T Sigma R P^T F)^-1 D);
* perspective / fisheye / RS: coverage misses are reported.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import scenegen as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
C0 = 0.28209479177387814


def _golden_section(f, a, b, tol=1e-13):
    g = (math.sqrt(5) - 1) / 2
    c, d = b - g * (b - a), a + g * (b - a)
    while b - a > tol:
        if f(c) > f(d):
            b, d = d, c
            c = b - g * (b - a)
        else:
            a, c = c, d
            d = a + g * (b - a)
    return 0.5 * (a + b)


def test_max_response_golden(orc):
    g = json.load(open(os.path.join(GOLD, "response.json")))
    for c in g["tau_max"]:
        w2, tau = orc.max_response([0, 0, 0], np.eye(3), [1, 1, 1], c["o"], c["d"])
        assert tau == pytest.approx(c["tau"], abs=1e-14)
    for c in g["alpha"]:
        w2, tau = orc.max_response([0, 0, 0], np.eye(3), [1, 1, 1], c["o"], c["d"])
        assert c["sigma"] * math.exp(-0.5 * w2) == pytest.approx(c["alpha"], abs=1e-15)


def test_max_response_vs_line_search(orc):
    """Eq. 11 against a direct 1-D maximisation of the Eq. 1 response along the
    ray with Sigma^-1 = inv(R S S^T R^T) from scipy/numpy."""
    rng = np.random.default_rng(21)
    for _ in range(200):
        mu = rng.uniform(-2, 2, 3)
        q = rng.standard_normal(4)
        s = np.exp(rng.uniform(-3, 0, 3))
        R = Rotation.from_quat(np.roll(q / np.linalg.norm(q), -1)).as_matrix()
        Si = np.linalg.inv(R @ np.diag(s * s) @ R.T)
        o = rng.uniform(-8, 8, 3)
        d = mu - o + rng.normal(0, 0.3, 3)
        d /= np.linalg.norm(d)
        w2, tau = orc.max_response(mu, orc.quat_to_rot(q), s, o, d)

        def rho(t):
            x = o + t * d - mu
            return -0.5 * x @ Si @ x

        t_ls = _golden_section(rho, -50, 50)
        assert tau == pytest.approx(t_ls, abs=1e-6 * max(1, abs(t_ls)))
        assert w2 == pytest.approx(-2 * rho(tau), rel=1e-9, abs=1e-12)
        assert -2 * rho(t_ls) >= w2 - 1e-9 * max(1, w2)


def test_max_response_rigid_invariance(orc):
    rng = np.random.default_rng(22)
    for _ in range(50):
        mu, o = rng.uniform(-2, 2, 3), rng.uniform(-5, 5, 3)
        q = rng.standard_normal(4)
        s = np.exp(rng.uniform(-2, 0, 3))
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        R = orc.quat_to_rot(q)
        w2, tau = orc.max_response(mu, R, s, o, d)
        T = Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
        t = rng.uniform(-3, 3, 3)
        w2b, taub = orc.max_response(T @ mu + t, T @ R, s, T @ o + t, T @ d)
        assert w2b == pytest.approx(w2, rel=1e-9, abs=1e-10)
        assert taub == pytest.approx(tau, rel=1e-9, abs=1e-10)


def _hit_scene(hits, px=(5, 7), fx=32.0):
    """Gaussians centred on the ray of pixel px of an ORTHO camera (rays pass
    exactly through mu, so alpha = sigma), colours set through the SH DC term."""
    u, v = px[0] + 0.5, px[1] + 0.5
    x, y = (u - 32.0) / fx, (v - 32.0) / fx
    n = len(hits)
    mu = np.array([[x, y, 3.0 + i] for i in range(n)], np.float32).reshape(n, 3)
    sh = np.zeros((n, 1, 3), np.float32)
    for i, h in enumerate(hits):
        for c in range(3):
            sh[i, 0, c] = (0.5 / C0) if h["rgb"][c] == 1 else (-1.0 / C0)
    sc = S.Scene(mu, np.tile(np.array([[1, 0, 0, 0]], np.float32), (n, 1)).reshape(n, 4),
                 np.full((n, 3), 0.05, np.float32), np.array([h["alpha"] for h in hits], np.float32).reshape(n), sh, 0)
    cam = S.Camera("ortho", 64, 64, fx, fx, 32.0, 32.0)
    return sc, cam


def test_compositing_golden(orc):
    g = json.load(open(os.path.join(GOLD, "compositing.json")))
    for c in g["cases"]:
        if not c["hits"]:
            sc, cam = _hit_scene([{"alpha": 0.5, "rgb": [1, 1, 1]}])
            sc.means[:, 2] = -3.0  # behind the camera: no hit
        else:
            sc, cam = _hit_scene(c["hits"])
        r = orc.render(sc, cam, S.RenderOptions())
        np.testing.assert_allclose(r["rgb"][7, 5], c["rgb"], atol=1e-7)
        assert 1 - r["alpha"][7, 5] == pytest.approx(c["T"], abs=1e-7)


def _tiny_scenes():
    for variant in S.TINY_VARIANTS:
        for seed in range(8):
            yield variant, seed


def test_invariants_tiny(orc):
    """Conservation: with every colour = 1 and black background,
    rgb = sum alpha_i T_i = 1 - T = alpha; T in [0,1]; alpha <= 1 - T_min."""
    opt = S.RenderOptions()
    for variant, seed in _tiny_scenes():
        sc, cam = S.tiny(seed, variant)
        sc.sh[:, 0, :] = 0.5 / C0
        r = orc.render(sc, cam, opt)
        a = r["alpha"]
        assert np.all(a >= 0) and np.all(a <= 1 - opt.transmittance_min + 1e-7)
        for c in range(3):
            np.testing.assert_allclose(r["rgb"][..., c], a, atol=2e-7)
        assert np.all(np.isfinite(r["depth"]))


def test_ortho_binned_equals_brute(orc):
    """UT is exact for affine cameras and the dilated ellipse contains the
    alpha >= alpha_min set, so binning misses nothing: bit-identical images."""
    opt = S.RenderOptions()
    for seed in range(16):
        sc, cam = S.tiny(seed, "ortho")
        a = orc.render(sc, cam, opt)
        b = orc.render(sc, cam, opt, brute=True)
        assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["alpha"], b["alpha"])
        assert np.array_equal(a["depth"], b["depth"])


@pytest.mark.parametrize("tile_cull", [0, 1])
def test_ortho_marginal_identity(orc, tile_cull):
    """Single Gaussian, ORTHO camera: alpha(pixel) = min(alpha_max,
    sigma exp(-1/2 D^T A^-1 D)) with A = F P R^T Sigma R P^T F (the projected
    marginal), wherever that value is >= alpha_min, else 0."""
    rng = np.random.default_rng(23)
    opt = S.RenderOptions(tile_cull=tile_cull)
    cam = S.Camera("ortho", 64, 64, 32.0, 32.0, 32.0, 32.0)
    F = np.diag([32.0, 32.0])
    for _ in range(10):
        mu = np.array([[rng.uniform(-0.6, 0.6), rng.uniform(-0.6, 0.6), 4.0]], np.float32)
        q = rng.standard_normal((1, 4)).astype(np.float32)
        s = np.exp(rng.uniform(math.log(0.03), math.log(0.25), (1, 3))).astype(np.float32)
        sig = np.float32(rng.uniform(0.2, 0.99))
        sc = S.Scene(mu, q, s, np.array([sig], np.float32), np.zeros((1, 1, 3), np.float32), 0)
        r = orc.render(sc, cam, opt)
        Rg = Rotation.from_quat(np.roll(q[0].astype(np.float64) / np.linalg.norm(q[0]), -1)).as_matrix()
        Sig = Rg @ np.diag(s[0].astype(np.float64) ** 2) @ Rg.T
        A = F @ Sig[:2, :2] @ F
        Ai = np.linalg.inv(A)
        jj, ii = np.mgrid[0:64, 0:64]
        D = np.stack([ii + 0.5 - (32 + 32 * mu[0, 0]), jj + 0.5 - (32 + 32 * mu[0, 1])], -1)
        al = float(sig) * np.exp(-0.5 * np.einsum("hwi,ij,hwj->hw", D, Ai, D))
        al = np.minimum(al, opt.alpha_max)
        exp = np.where(al >= opt.alpha_min, al, 0.0)
        keep = np.abs(al - opt.alpha_min) > 1e-9
        np.testing.assert_allclose(r["alpha"][keep], exp[keep], atol=1e-6)


@pytest.mark.parametrize("variant", ["pinhole", "opencv", "fisheye", "rs"])
def test_coverage_misses_reported(orc, variant):
    """under nonlinear projection the UT footprint may under-cover.
    Report the binned-vs-brute difference; it must stay small on tiny scenes."""
    opt = S.RenderOptions()
    worst = 0.0
    for seed in range(8):
        sc, cam = S.tiny(seed, variant)
        a = orc.render(sc, cam, opt)
        b = orc.render(sc, cam, opt, brute=True)
        worst = max(worst, float(np.abs(a["rgb"] - b["rgb"]).max()))
    print(f"{variant}: max |binned - brute| = {worst:.3e}")
    assert worst < 0.05
