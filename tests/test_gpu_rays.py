"""GPU: the pixel-ray table (a5, PAPER L116 r(tau) = o + tau d) and the
per-block affine lattice that K5's candidate masks are built on
(k5_blend.cu entry_mask): for every 8x8 block, every valid pixel's fp32 ray
offsets (a, b) lie within rho of a00 + ax x + ay y (resp. b), rho as
recorded.  The masks are conservative only if this holds, so it is checked
on every camera model, ragged image edges included, and at the bench
resolution; the lattice must also be tight (rho far below a pixel step) for
the masks to cull anything.  Results of the masks themselves: images are
bitwise those of a build without them (tools/ab_compare.py)."""
import numpy as np
import pytest

import scenegen as S

pytestmark = pytest.mark.gpu


def _lattice_check(r, cam, label, global_shutter=True, tight=False):
    from paper_2412_12507_b200 import gut
    r.render(cam, S.RenderOptions())
    rays, fit = gut.gut_debug_copy_stage(r.ctx, gut.STAGE_RAYS)
    nt = rays.shape[0]
    assert fit.shape == (nt, 4, 8)
    cx, ry = np.meshgrid(np.arange(8), np.arange(8))  # [ry, cx]
    worst, n_blocks, loose = 0.0, 0, 0
    for b in range(4):
        x = 8 * (b & 1) + cx
        y = 8 * (b >> 1) + ry
        idx = 32 * ((x >> 3) | ((y >> 2) << 1)) + 8 * (y & 3) + (x & 7)  # rays_kernel layout
        v = rays[:, idx, :]                      # [nt, 8, 8, 4]
        valid = v[..., 2] > 0
        f = fit[:, b, :].astype(np.float64)      # [nt, 8]
        has = valid.any(axis=(1, 2))
        for comp, off in ((0, 0), (1, 4)):
            pred = (f[:, off, None, None] + f[:, off + 1, None, None] * cx[None] + f[:, off + 2, None, None] * ry[None])
            res = np.abs(v[..., comp].astype(np.float64) - pred)
            rho = f[:, off + 3]
            if global_shutter:
                assert np.isfinite(rho[has]).all(), f"{label}: block {b} without a lattice"
            ok = np.where(valid, res <= rho[:, None, None], True)
            assert ok.all(), f"{label}: block {b} comp {comp}: {(~ok).sum()} pixels off their lattice"
            full = valid.all(axis=(1, 2)) & np.isfinite(rho)
            step = np.abs(f[:, off + 1]) + np.abs(f[:, off + 2])
            if full.any():
                rel = rho[full] / step[full]
                worst = max(worst, float(rel.max()))
                loose += int((rel > 0.05).sum())
            n_blocks += int(has.sum())
    print(f"{label}: {n_blocks} blocks, worst rho / pixel step {worst:.2e}")
    # tight at the configs' focal lengths (the tiny 64 px-focal cameras bend
    # visibly within 8 px): the lattice error is a small fraction of a pixel step
    if tight:
        assert loose == 0, f"{label}: {loose} full blocks with rho above 5% of a pixel step"


@pytest.mark.parametrize("variant", ["pinhole", "ortho", "opencv", "fisheye"])
def test_ray_lattice_tiny(variant):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import gut
    scene, cam = S.tiny(3, variant, n=64, size=70)  # 70 px: ragged tiles at both edges
    r = gut.Renderer(scene)
    _lattice_check(r, cam, f"tiny {variant}")
    r.close()


@pytest.mark.parametrize("config", ["multiview", "mipnerf360", "scannetpp"])
def test_ray_lattice_full_resolution(config):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import gut
    scene = S.make_scene(config, n=2000)
    cam = S.make_views(config)[1]
    r = gut.Renderer(scene, max_wh=(cam.width, cam.height))
    _lattice_check(r, cam, config, tight=True)
    r.close()
