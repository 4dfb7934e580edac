"""Pins for oracle step O1 (UT weights, R(q), sigma points) and the SH basis.

Each test ties the oracle to something other than itself: printed constants
(SPEC worked examples in tests/golden/), textbook identities
(moment matching of Eq. 6-8, orthonormality of the real SH basis), or an
independent library (scipy's quaternion -> matrix).
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_ut_weights_golden(orc):
    g = json.load(open(os.path.join(GOLD, "ut_weights.json")))
    for c in g["cases"]:
        wm, ws, lam = orc.ut_weights(c["alpha"], c["beta"], c["kappa"])
        assert lam == pytest.approx(c["lambda"], abs=1e-15)
        np.testing.assert_allclose(wm, c["w_mu"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(ws, c["w_sigma"], rtol=0, atol=1e-15)
    for c in g["invalid"]:
        with pytest.raises(ValueError):
            orc.ut_weights(c["alpha"], c["beta"], c["kappa"])


def test_ut_weights_sum_to_one(orc):
    rng = np.random.default_rng(1)
    for _ in range(100):
        a, b, k = rng.uniform(0.3, 2.0), rng.uniform(-1, 3), rng.uniform(-1, 2)
        wm, ws, lam = orc.ut_weights(a, b, k)
        assert wm.sum() == pytest.approx(1.0, abs=1e-12)
        # Eq. 8: sum of w_sigma = 1 + (1 - alpha^2 + beta)
        assert ws.sum() == pytest.approx(1.0 + (1 - a * a + b), abs=1e-12)


def test_rotation_worked_values(orc):
    # identity, s=(1,2,3) -> diag(1,4,9); 90 deg about z, s=(2,1,1) -> diag(1,4,1)
    R = orc.quat_to_rot([1, 0, 0, 0])
    S = np.diag([1.0, 2.0, 3.0])
    np.testing.assert_allclose(R @ S @ S.T @ R.T, np.diag([1, 4, 9]), atol=1e-15)
    q = [math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)]
    R = orc.quat_to_rot(q)
    S = np.diag([2.0, 1.0, 1.0])
    np.testing.assert_allclose(R @ S @ S.T @ R.T, np.diag([1, 4, 1]), atol=1e-14)


def test_rotation_matches_scipy(orc):
    rng = np.random.default_rng(2)
    for _ in range(200):
        q = rng.standard_normal(4) * rng.uniform(0.1, 10)  # not normalised: oracle normalises (reading R1)
        R = orc.quat_to_rot(q)
        Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scipy is scalar-last
        np.testing.assert_allclose(R, Rs, atol=1e-13)
        np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-13)
        assert np.linalg.det(R) == pytest.approx(1.0, abs=1e-13)
    with pytest.raises(ValueError):
        orc.quat_to_rot([0, 0, 0, 0])


def test_sigma_points_worked_example(orc):
    # mu=0, Sigma=I, lambda=0 -> {0, +-sqrt3 e_j}
    X = orc.sigma_points([0, 0, 0], np.eye(3), [1, 1, 1], 0.0)
    r3 = math.sqrt(3)
    exp = np.array([[0, 0, 0], [r3, 0, 0], [0, r3, 0], [0, 0, r3], [-r3, 0, 0], [0, -r3, 0], [0, 0, -r3]])
    np.testing.assert_allclose(X, exp, atol=1e-15)


def test_sigma_points_moment_matching(orc):
    """UT moment matching: sum w_mu x = mu and
    sum w_sigma (x-mu)(x-mu)^T = Sigma = R S S^T R^T for any beta (x0 = mu),
    with Sigma built from scipy's rotation (independent of the oracle)."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        a, b, k = rng.uniform(0.4, 2.0), rng.uniform(-1, 3), rng.uniform(-0.5, 2)
        wm, ws, lam = orc.ut_weights(a, b, k)
        mu = rng.uniform(-5, 5, 3)
        q = rng.standard_normal(4)
        s = np.exp(rng.uniform(-4, 0, 3))
        R = orc.quat_to_rot(q)
        X = orc.sigma_points(mu, R, s, lam)
        Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
        Sigma = Rs @ np.diag(s * s) @ Rs.T
        np.testing.assert_allclose((wm[:, None] * X).sum(0), mu, atol=1e-12)
        D = X - mu
        cov = (ws[:, None, None] * D[:, :, None] * D[:, None, :]).sum(0)
        np.testing.assert_allclose(cov, Sigma, atol=1e-12 * max(1.0, np.abs(Sigma).max()))
        # translation equivariance
        X2 = orc.sigma_points(mu + 1.25, R, s, lam)
        np.testing.assert_allclose(X2, X + 1.25, atol=1e-12)


def _sphere_quadrature(n_theta=64, n_phi=128):
    """Gauss-Legendre in cos(theta) x uniform phi: exact for polynomials of
    degree < 2*n_theta on the sphere."""
    x, w = np.polynomial.legendre.leggauss(n_theta)
    phi = (np.arange(n_phi) + 0.5) * 2 * np.pi / n_phi
    ct = np.repeat(x, n_phi)
    st = np.sqrt(1 - ct * ct)
    ph = np.tile(phi, n_theta)
    d = np.stack([st * np.cos(ph), st * np.sin(ph), ct], 1)
    wt = np.repeat(w, n_phi) * (2 * np.pi / n_phi)
    return d, wt


def test_sh_basis_orthonormal(orc):
    """The 3DGS real SH basis (reading R19) is orthonormal on the sphere: a
    wrong constant, sign-insensitive typo or dropped term breaks <Y_i, Y_j> = delta_ij."""
    d, w = _sphere_quadrature(24, 48)
    Y = np.stack([orc.sh_basis(v) for v in d])
    G = (Y * w[:, None]).T @ Y
    np.testing.assert_allclose(G, np.eye(16), atol=1e-12)


def test_sh_degree_structure(orc):
    """Y_lm is a homogeneous harmonic polynomial of degree l: Y(-d) = (-1)^l Y(d)."""
    rng = np.random.default_rng(4)
    for _ in range(20):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        Y, Yn = orc.sh_basis(d), orc.sh_basis(-d)
        for l in range(4):
            sl = slice(l * l, (l + 1) * (l + 1))
            np.testing.assert_allclose(Yn[sl], (-1) ** l * Y[sl], atol=1e-14)
    assert orc.sh_basis([0, 0, 1])[0] == pytest.approx(0.28209479177387814, abs=0)
