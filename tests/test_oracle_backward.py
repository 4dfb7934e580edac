"""Pins for O7, the backward pass (PAPER Supp. B, L494-513; reading R30):

* central finite differences of the oracle's fp64 forward loss
  L = sum g_rgb.rgb + g_alpha alpha + g_depth depth (the derivative's
  definition) for mu, q, s, sigma and SH of the Gaussians that matter most,
  at two step sizes (a parameter whose two estimates disagree sits on a
  discontinuity -- alpha skip, termination, binning -- and is skipped);
* the loss reported by O7 equals the image-space loss of the O6 render;
* invariances: a global scale of q does not change the image, so
  dL/dq . q = 0; SH gradients are the colour gradient times Y_k (DC:
  Y_0 = 0.2821) wherever the colour is not clamped.
"""
import numpy as np
import pytest

import scenegen as S

C0 = 0.28209479177387814


def _grads(rng, cam):
    H, W = cam.height, cam.width
    return (rng.standard_normal((H, W, 3)).astype(np.float32), rng.standard_normal((H, W)).astype(np.float32),
            (0.1 * rng.standard_normal((H, W))).astype(np.float32))


@pytest.mark.parametrize("variant", ["pinhole", "fisheye", "opencv"])
def test_backward_loss_matches_render(orc, variant):
    scene, cam = S.tiny(3, variant, n=64, sh_degree=1)
    rng = np.random.default_rng(1)
    g = _grads(rng, cam)
    b = orc.backward(scene, cam, S.RenderOptions(), *g)
    r = orc.render(scene, cam, S.RenderOptions(), ambiguity=False)
    L = float((g[0].astype(np.float64) * r["rgb"]).sum() + (g[1] * r["alpha"].astype(np.float64)).sum()
              + (g[2] * r["depth"].astype(np.float64)).sum())
    assert b["loss"] == pytest.approx(L, rel=1e-5, abs=1e-3)


def _fd(orc, scene, cam, opt, g, field, i, comp, h):
    arr = getattr(scene, field)
    flat = arr.reshape(arr.shape[0], -1)
    p0 = flat[i, comp]
    hi, lo = np.float32(p0 + h), np.float32(p0 - h)
    flat[i, comp] = hi
    Lp = orc.backward(scene, cam, opt, *g)["loss"]
    flat[i, comp] = lo
    Lm = orc.backward(scene, cam, opt, *g)["loss"]
    flat[i, comp] = p0
    return (Lp - Lm) / (float(hi) - float(lo))


@pytest.mark.parametrize("variant,seed,deg,kdeg", [("pinhole", 0, 0, 2), ("fisheye", 1, 0, 2), ("opencv", 2, 0, 2),
                                                   ("pinhole", 4, 2, 2), ("rs", 5, 0, 2), ("pinhole", 6, 0, 4),
                                                   ("fisheye", 7, 0, 3)])
def test_backward_finite_differences(orc, variant, seed, deg, kdeg):
    """deg 0: every parameter.  deg > 0: the colour's view direction is held
    constant in the backward (reading R30), so mu is checked at deg 0 only."""
    scene, cam = S.tiny(seed, variant, n=48, sh_degree=deg)
    opt = S.RenderOptions(kernel_degree=kdeg)
    rng = np.random.default_rng(10 + seed)
    g = _grads(rng, cam)
    b = orc.backward(scene, cam, opt, *g)
    top = np.argsort(-np.abs(b["opacities"]))[:5]
    checked = tried = 0
    for i in top:
        for field, key, comps, h in (("means", "means", range(3) if deg == 0 else [], 2e-4),
                                     ("rotations", "rotations", range(4), 2e-4),
                                     ("scales", "scales", range(3), 2e-5), ("opacities", "opacities", [0], 2e-4),
                                     ("sh", "sh", [0, 1, 2] + ([3, 5, 13] if deg else []), 2e-3)):
            for c in comps:
                tried += 1
                f1 = _fd(orc, scene, cam, opt, g, field, i, c, h)
                f2 = _fd(orc, scene, cam, opt, g, field, i, c, h / 2)
                an = b[key].reshape(scene.count, -1)[i, c]
                scale = max(abs(an), abs(f2), 1e-2)
                if abs(f1 - f2) > 2e-3 * scale:
                    continue  # a discontinuity inside the step: not a smooth point
                checked += 1
                assert abs(an - f2) <= 1e-4 * scale, (field, i, c, an, f1, f2)  # (measured ~1e-8)
    assert checked >= 0.7 * tried, (checked, tried)


def test_backward_invariances(orc):
    scene, cam = S.tiny(5, "pinhole", n=64, sh_degree=2)
    opt = S.RenderOptions()
    g = _grads(np.random.default_rng(3), cam)
    b = orc.backward(scene, cam, opt, *g)
    q = scene.rotations.astype(np.float64)
    np.testing.assert_allclose((b["rotations"] * q).sum(1), 0.0, atol=1e-9 * (1 + np.abs(b["rotations"]).max()))
    p = orc.preprocess(scene, cam, opt)
    ok = (p["reason"] == 0)[:, None] & (p["rgb"] > 0)
    np.testing.assert_allclose(b["sh"][:, 0, :][ok], C0 * b["rgb"][ok], rtol=1e-12, atol=1e-15)
    assert np.all(b["sh"][:, 0, :][~ok] == 0)
    # Gaussians that touch no pixel have zero gradients
    dead = p["reason"] != 0
    assert np.all(b["means"][dead] == 0) and np.all(b["opacities"][dead] == 0)
