"""Pins for oracle step O3 (UT estimate Eq. 9-10, extent, tiles) and O4.

* affine cameras: UT is exact (moment matching), so v_mu and
  Sigma' - b I equal the linear image of (mu, Sigma), computed here with scipy
  rotations for random alpha/beta/kappa;
* nonlinear cameras: Sigma' - b I -> J Sigma J^T with O(s^2) relative error as
  s -> 0 (J = central-difference Jacobian);
* extent: the corrected SPEC values (tests/golden/extent.json);
* ellipse-tile test: brute-force dense sampling of the square;
* tile lists: sorted by (depth, index), a permutation of the kept pairs.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import scenegen as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _scene(mu, q, s, sig=0.9, deg=0):
    n = len(mu)
    sh = np.zeros((n, (deg + 1) ** 2, 3), np.float32)
    return S.Scene(np.asarray(mu, np.float32), np.asarray(q, np.float32), np.asarray(s, np.float32),
                   np.full(n, sig, np.float32), sh, deg)


def _ortho_cam(rng):
    eye = rng.uniform(-1, 1, 3)
    tgt = eye + np.array([0.3, 0.2, 1.0]) + rng.uniform(-0.2, 0.2, 3)
    q = S._mat_to_quat(S.look_at_c2w(eye, tgt, up=(0.1, -1.0, 0.0)))
    return S.Camera("ortho", 256, 256, 41.0, 37.0, 128.3, 127.1, q_c2w=(q, q), c_w=(tuple(eye), tuple(eye)))


def test_ut_exact_for_affine_camera(orc):
    """ORTHO: v_mu = F P R^T (mu - c) + (cx,cy), Sigma' - bI = F P R^T Sigma R P^T F
    exactly for any alpha, beta, kappa with 3+lambda > 0."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        cam = _ortho_cam(rng)
        a, b, k = rng.uniform(0.5, 1.8), rng.uniform(-0.5, 3.0), rng.uniform(0, 2)
        opt = S.RenderOptions(ut_alpha=a, ut_beta=b, ut_kappa=k)
        Rc = Rotation.from_quat(np.roll(cam.q_c2w[0], -1)).as_matrix()
        c = np.array(cam.c_w[0])
        n = 50
        mu_c = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(3, 6, n)], 1)
        mu = (Rc @ mu_c.T).T + c
        q = rng.standard_normal((n, 4))
        s = np.exp(rng.uniform(math.log(0.01), math.log(0.2), (n, 3)))
        sc = _scene(mu, q, s)
        p = orc.preprocess(sc, cam, opt)
        F = np.diag([cam.fx, cam.fy])
        for i in range(n):
            assert p["reason"][i] in (0, 5, 6)
            m = sc.means[i].astype(np.float64)
            Rg = Rotation.from_quat(np.roll(sc.rotations[i].astype(np.float64), -1)).as_matrix()
            Sig = Rg @ np.diag(sc.scales[i].astype(np.float64) ** 2) @ Rg.T
            A = F @ Rc.T[:2, :]
            v_exp = A @ (m - c) + np.array([cam.cx, cam.cy])
            cov_exp = A @ Sig @ A.T
            assert p["vx"][i] == pytest.approx(v_exp[0], abs=1e-10)
            assert p["vy"][i] == pytest.approx(v_exp[1], abs=1e-10)
            cov = np.array([[p["cxx"][i], p["cxy"][i]], [p["cxy"][i], p["cyy"][i]]]) - opt.cov2d_dilation * np.eye(2)
            np.testing.assert_allclose(cov, cov_exp, rtol=1e-10, atol=1e-11)


@pytest.mark.parametrize("model", ["pinhole", "fisheye", "opencv"])
def test_ut_linearisation_limit(orc, model):
    """Nonlinear g: UT covariance converges to J Sigma J^T with the absolute
    error O(s^4), i.e. the relative error falls ~4x per halving of s."""
    kw = dict(fov_limit=math.radians(100)) if model == "fisheye" else {}
    if model == "opencv":
        kw = dict(k=(-0.2, 0.05, 0, 0, 0, 0), p=(1e-3, -1e-3), fov_limit=1.2)
    cam = S.Camera(model, 800, 600, 300.0, 310.0, 400.0, 300.0, **kw)
    opt = S.RenderOptions(cov2d_dilation=0.0)
    mu = np.array([[0.9, -0.4, 2.5]])
    q = np.array([[0.3, 0.8, -0.2, 0.4]])
    Rg = Rotation.from_quat(np.roll(q[0] / np.linalg.norm(q[0]), -1)).as_matrix()
    base = np.array([0.04, 0.02, 0.01])

    def g(x):
        v, uv, _, _ = orc.project_point(cam, opt, x)
        return uv

    h = 1e-6
    J = np.stack([(g(mu[0] + h * e) - g(mu[0] - h * e)) / (2 * h) for e in np.eye(3)], 1)
    errs = []
    for f in (1.0, 0.5, 0.25, 0.125):
        s = base * f
        p = orc.preprocess(_scene(mu, q, [s]), cam, opt)
        cov = np.array([[p["cxx"][0], p["cxy"][0]], [p["cxy"][0], p["cyy"][0]]])
        Sig = Rg @ np.diag(s.astype(np.float32).astype(np.float64) ** 2) @ Rg.T
        ref = J @ Sig @ J.T
        errs.append(np.abs(cov - ref).max() / np.abs(ref).max())
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(r > 3.0 for r in ratios), (errs, ratios)


def test_extent_golden(orc):
    """Alg. 1 Extent: with an ORTHO camera, Sigma' is chosen exactly
    (Sigma' = F^2 s^2 + b); h must equal the corrected SPEC L340-341 values."""
    g = json.load(open(os.path.join(GOLD, "extent.json")))
    opt = S.RenderOptions()
    assert opt.alpha_min == g["alpha_min_f32"]
    cam = S.Camera("ortho", 64, 64, 1.0, 1.0, 32.0, 32.0)
    for c in g["cases"]:
        cxx, _, cyy = c["cov"]
        s = [math.sqrt(cxx - opt.cov2d_dilation), math.sqrt(cyy - opt.cov2d_dilation), 0.05]
        sc = _scene([[0.0, 0.0, 3.0]], [[1, 0, 0, 0]], [s], sig=c["sigma"])
        # float32 scales perturb Sigma' at 1e-8: compare at 1e-6
        p = orc.preprocess(sc, cam, opt)
        assert p["hx"][0] == pytest.approx(c["h"][0], abs=2e-6)
        assert p["hy"][0] == pytest.approx(c["h"][1], abs=2e-6)


def test_ellipse_tile_test_brute_force(orc):
    rng = np.random.default_rng(12)
    G = np.linspace(0, 16, 161)
    for _ in range(400):
        vx, vy = rng.uniform(-30, 46), rng.uniform(-30, 46)
        L = rng.uniform(0.3, 12, 2)
        th = rng.uniform(0, math.pi)
        Rm = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
        cov = Rm @ np.diag(L ** 2) @ Rm.T
        k2 = rng.uniform(0.5, 11)
        hit = orc.tile_hits_ellipse(vx, vy, cov[0, 0], cov[0, 1], cov[1, 1], k2, 0.0, 0.0, 16.0, 16.0)
        X, Y = np.meshgrid(G, G)
        D = np.stack([X.ravel() - vx, Y.ravel() - vy], 1)
        qv = np.einsum("ni,ij,nj->n", D, np.linalg.inv(cov), D)
        qmin = qv.min()
        if qmin <= k2 * (1 - 1e-3):
            assert hit
        if qmin > k2 * 1.05 + 0.05:
            assert not hit


def test_tile_spec_cases(orc):
    """a small conic in the middle of a tile -> 1 tile; on a
    4-tile corner -> 4 tiles; an invalid (behind-camera) Gaussian -> 0 tiles."""
    cam = S.Camera("ortho", 64, 64, 16.0, 16.0, 0.0, 0.0)
    opt = S.RenderOptions()
    mu = [[24 / 16, 24 / 16, 3.0], [32 / 16, 32 / 16, 3.0], [1.0, 1.0, -3.0]]
    sc = _scene(mu, [[1, 0, 0, 0]] * 3, [[0.05, 0.05, 0.05]] * 3)
    p = orc.preprocess(sc, cam, opt)
    assert list(p["tiles"]) == [1, 4, 0]
    assert p["reason"][2] == 3  # invalid sigma point


def test_tile_lists_order_and_permutation(orc):
    for variant in S.TINY_VARIANTS:
        for seed in range(4):
            sc, cam = S.tiny(seed, variant)
            opt = S.RenderOptions()
            p = orc.preprocess(sc, cam, opt)
            tiles, gids, ranges = orc.tile_lists(p, cam, opt)
            assert tiles.size == int(p["tiles"][p["reason"] == 0].sum())
            # sorted by (tile, fp32 depth key, gid) -- the 3DGS key (reading R13')
            key = list(zip(tiles, p["depth"][gids].astype(np.float32), gids))
            assert key == sorted(key)
            # each visible Gaussian appears exactly 'tiles' times, each pair once
            pairs = set(zip(tiles.tolist(), gids.tolist()))
            assert len(pairs) == tiles.size
            cnt = np.bincount(gids, minlength=sc.count)
            np.testing.assert_array_equal(cnt, np.where(p["reason"] == 0, p["tiles"], 0))
            for t in range(ranges.shape[0]):
                a, b = ranges[t]
                assert np.all(tiles[a:b] == t)


def test_tile_lists_fp32_key_ties_by_index(orc):
    """Two Gaussians whose fp64 depths differ but round to the same fp32 key
    are listed by index, not by the fp64 depth (reading R13': the sort key is
    the 3DGS (tile, float depth bits) key, ties by Gaussian index)."""
    sc, cam = S.tiny(0, "pinhole", n=2)
    x1 = np.nextafter(np.float32(0.1), np.float32(0))       # gid 1 nearer by ~2e-10 in fp64
    sc.means[:] = [[0.1, 0.1, 4.0], [x1, 0.1, 4.0]]
    sc.scales[:] = 0.05
    sc.rotations[:] = [1, 0, 0, 0]
    opt = S.RenderOptions()
    p = orc.preprocess(sc, cam, opt)
    assert np.all(p["reason"] == 0)
    assert p["depth"][1] < p["depth"][0] and np.float32(p["depth"][1]) == np.float32(p["depth"][0])
    tiles, gids, ranges = orc.tile_lists(p, cam, opt)
    for t in np.unique(tiles):
        a, b = ranges[t]
        assert list(gids[a:b]) == [0, 1]
    # distinct fp32 keys: the nearer one first
    sc.means[1, 2] = 3.9
    p = orc.preprocess(sc, cam, opt)
    tiles, gids, ranges = orc.tile_lists(p, cam, opt)
    a, b = ranges[tiles[0]]
    assert list(gids[a:b]) == [1, 0]


def test_aabb_mode_counts_rectangle(orc):
    sc, cam = S.tiny(3, "pinhole")
    opt = S.RenderOptions(tile_cull=0)
    p = orc.preprocess(sc, cam, opt)
    vis = p["reason"] == 0
    r = p["rect"][vis]
    np.testing.assert_array_equal(p["tiles"][vis], (r[:, 2] - r[:, 0] + 1) * (r[:, 3] - r[:, 1] + 1))
    pe = orc.preprocess(sc, cam, S.RenderOptions(tile_cull=1))
    assert np.all(pe["tiles"][vis] <= p["tiles"][vis])
