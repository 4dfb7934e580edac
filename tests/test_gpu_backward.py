"""GPU parity of the backward pass (K6, PAPER Supp. B; reading R30) through
the C ABI against the fp64 oracle O7 on the same seeded inputs.  Upstream
gradients are random; at pixels the oracle marks ambiguous (alpha-skip /
termination bands, order ties, binning / cull ambiguity) they are set to 0
on both sides, so both differentiate the same function.  Per-Gaussian
gradients are compared per field: |gpu - oracle| <= 2e-3 |oracle| + 2e-4
max|oracle| (fp32 terms over many pixels, summed in 32.32 fixed point)."""
import dataclasses

import numpy as np
import pytest

import scenegen as S
from gpu_common import pixel_mask

pytestmark = pytest.mark.gpu

FIELDS = ("means", "rotations", "scales", "opacities", "sh", "rgb")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import build
    build.build()


def _run(scene, cam, opt=None, seed=0, label=""):
    import torch
    from oracle import oracle as O
    from paper_2412_12507_b200 import gut
    opt = opt or S.RenderOptions()
    o = O.render(scene, cam, opt)
    mask = pixel_mask(o["diag"], cam)
    rng = np.random.default_rng(seed)
    H, W = cam.height, cam.width
    g_rgb = rng.standard_normal((H, W, 3)).astype(np.float32) * mask[..., None]
    g_a = rng.standard_normal((H, W)).astype(np.float32) * mask
    g_d = (0.1 * rng.standard_normal((H, W))).astype(np.float32) * mask
    ob = O.backward(scene, cam, opt, g_rgb, g_a, g_d)
    r = gut.Renderer(scene, max_wh=(max(W, 16), max(H, 16)))
    out = r.render(cam, opt)[:3]
    dev = out[0].device
    gb = r.backward(cam, opt, out, torch.from_numpy(g_rgb).to(dev), torch.from_numpy(g_a).to(dev),
                    torch.from_numpy(g_d).to(dev))
    torch.cuda.synchronize()
    worst = 0.0
    for f in FIELDS:
        a = gb[f].cpu().numpy().astype(np.float64).reshape(scene.count, -1)
        b = ob[f].reshape(scene.count, -1)
        scale = np.abs(b).max() + 1e-12
        err = np.abs(a - b) / (2e-3 * np.abs(b) + 2e-4 * scale)
        worst = max(worst, float(err.max(initial=0)))
        i = np.unravel_index(np.argmax(err), err.shape) if err.size else None
        print(f"{label} {f}: max |d| {np.abs(a - b).max(initial=0):.3e} (max |g| {scale:.3e}) ratio {err.max(initial=0):.3f}"
              + (f" at {i}: gpu {a[i]:.6e} oracle {b[i]:.6e}" if i is not None else ""))
    # densification statistic (reading R32): |dL/dmu| / (distance / 2)
    p = O.preprocess(scene, cam, opt)
    cen = np.array([O.pose_at(cam, t)[1] for t in p["t0"]]) if cam.shutter != "global" else np.array(cam.c_w[0])
    dist = np.linalg.norm(scene.means.astype(np.float64) - cen, axis=-1)
    want = np.linalg.norm(ob["means"], axis=1) / (0.5 * dist)
    got = gb["densify"].cpu().numpy().astype(np.float64)
    ok = p["reason"] == 0
    np.testing.assert_allclose(got[ok], want[ok], rtol=5e-3, atol=2e-4 * want.max() + 1e-12)
    r.close()
    assert worst <= 1.0, label
    return gb, ob


@pytest.mark.parametrize("variant", ["pinhole", "fisheye", "opencv", "rs"])
@pytest.mark.parametrize("deg", [0, 3])
def test_tiny_backward(variant, deg):
    scene, cam = S.tiny(2, variant, n=96, sh_degree=deg)
    _run(scene, cam, seed=deg, label=f"{variant} deg {deg}")


@pytest.mark.parametrize("variant,kdeg", [("pinhole", 4), ("fisheye", 3), ("rs", 8)])
def test_tiny_backward_kernel_degree(variant, kdeg):
    scene, cam = S.tiny(3, variant, n=96, sh_degree=1)
    _run(scene, cam, S.RenderOptions(kernel_degree=kdeg), seed=kdeg, label=f"{variant} kernel degree {kdeg}")


def test_tiny_backward_ragged_dense():
    scene, cam = S.tiny(9, "pinhole", n=300, size=64, sh_degree=1)
    scene.scales[:] *= 1.5
    cam = dataclasses.replace(cam, width=70, height=50, cx=35.0, cy=25.0)
    _run(scene, cam, seed=5, label="ragged dense")


@pytest.mark.parametrize("config,n,factor,view", [("multiview", 60_000, 0.12, 5), ("scannetpp", 30_000, 0.12, 3),
                                                  ("waymo", 40_000, 0.1, 1)])
def test_reduced_config_backward(config, n, factor, view):
    scene = S.make_scene(config, n=n)
    cam = S.scaled_camera(S.make_views(config)[view], factor)
    _run(scene, cam, seed=7, label=f"{config} n={n}")


def test_backward_errors():
    import torch
    from paper_2412_12507_b200 import gut
    scene, cam = S.tiny(0, "pinhole", n=16)
    r = gut.Renderer(scene)
    out = r.render(cam)[:3]
    g = torch.zeros_like(out[0])
    with pytest.raises(gut.GutError) as e:   # camera differs from the last render
        r.backward(dataclasses.replace(cam, fx=cam.fx * 1.01), None, out, g)
    assert e.value.status == 1
    # empty scene: zero gradients, no error
    empty = scene.subset(np.zeros(0, np.int64))
    re_ = gut.Renderer(empty)
    oe = re_.render(cam)[:3]
    ge = re_.backward(cam, None, oe, torch.ones_like(oe[0]))
    assert all(v.numel() == 0 for v in ge.values())
    re_.close()
    for c2, o2 in ((S.tiny(0, "ortho", n=16)[1], None), (cam, S.RenderOptions(kbuffer=16))):
        out2 = r.render(c2, o2)[:3]
        with pytest.raises(gut.GutError) as e:
            r.backward(c2, o2, out2, torch.zeros_like(out2[0]))
        assert e.value.status == 2
    r.close()


def test_full_size_sampled_backward():
    """The bench frame (3M Gaussians, 1920x1080 fisheye, the launch
    configuration bench.py times for ours_forward_backward) with random upstream
    gradients on 24 sampled tiles (the 8 longest lists + 16 random ones), zero
    elsewhere and on ambiguous pixels: every per-Gaussian gradient against the
    fp64 oracle O7 (which skips zero-gradient pixels exactly)."""
    import torch
    from oracle import oracle as O
    from paper_2412_12507_b200 import gut
    scene = S.make_scene("multiview")
    cam = S.make_views("multiview")[0]
    opt = S.RenderOptions()
    r = gut.Renderer(scene, reserve_keys=int(scene.count * 12), max_wh=(cam.width, cam.height))
    out = r.render(cam, opt)[:3]
    ranges = r.stage(gut.STAGE_RANGES)
    tx, ty = cam.tiles
    lens = ranges[:, 1].astype(np.int64) - ranges[:, 0]
    rng = np.random.default_rng(7)
    longest = np.argsort(-lens)[:8]
    sub = np.sort(np.concatenate([longest, rng.choice(np.setdiff1d(np.arange(tx * ty), longest), 16,
                                                      replace=False)])).astype(np.int32)
    o = O.render(scene, cam, opt, tile_subset=sub)
    H, W = cam.height, cam.width
    sel = np.zeros((H, W), bool)
    for t in sub:
        sel[(t // tx) * 16:(t // tx) * 16 + 16, (t % tx) * 16:(t % tx) * 16 + 16] = True
    mask = sel & pixel_mask(o["diag"], cam)
    g_rgb = rng.standard_normal((H, W, 3)).astype(np.float32) * mask[..., None]
    g_a = rng.standard_normal((H, W)).astype(np.float32) * mask
    g_d = (0.1 * rng.standard_normal((H, W))).astype(np.float32) * mask
    dev = out[0].device
    gb = r.backward(cam, opt, out, torch.from_numpy(g_rgb).to(dev), torch.from_numpy(g_a).to(dev),
                    torch.from_numpy(g_d).to(dev))
    torch.cuda.synchronize()
    ob = O.backward(scene, cam, opt, g_rgb, g_a, g_d)
    touched = np.zeros(scene.count, bool)
    worst = 0.0
    for f in FIELDS:
        a = gb[f].cpu().numpy().astype(np.float64).reshape(scene.count, -1)
        b = ob[f].reshape(scene.count, -1)
        touched |= np.abs(b).max(1) > 0
        scale = np.abs(b).max() + 1e-12
        err = np.abs(a - b) / (2e-3 * np.abs(b) + 2e-4 * scale)
        worst = max(worst, float(err.max(initial=0)))
        print(f"full-size backward {f}: max |d| {np.abs(a - b).max(initial=0):.3e} (max |g| {scale:.3e}) "
              f"ratio {err.max(initial=0):.3f}")
    print(f"full-size backward: {int(touched.sum())} Gaussians with gradient, {int(mask.sum())} pixels")
    assert touched.sum() > 1000
    r.close()
    assert worst <= 1.0


@pytest.mark.parametrize("config,shutter_view", [("multiview", 1), ("waymo", 1)])
def test_backward_bitwise_reproducible(config, shutter_view):
    """The per-Gaussian sums accumulate in 32.32 fixed point (integer atomics
    commute): repeated backward passes of the same render -- thousands of
    warps adding to the same Gaussians in whatever order -- return bitwise
    identical gradients (multiview: global shutter; Waymo-shaped: rolling)."""
    import torch
    from paper_2412_12507_b200 import gut
    scene = S.make_scene(config, n=300_000)
    cam = S.scaled_camera(S.make_views(config)[shutter_view], 0.5)
    r = gut.Renderer(scene, max_wh=(cam.width, cam.height))
    out = r.render(cam)[:3]
    gen = torch.Generator(device="cuda").manual_seed(3)
    g_rgb = torch.randn(out[0].shape, device="cuda", generator=gen)
    g_a = torch.randn(out[1].shape, device="cuda", generator=gen)
    g_d = 0.1 * torch.randn(out[2].shape, device="cuda", generator=gen)
    runs = [r.backward(cam, S.RenderOptions(), out, g_rgb, g_a, g_d) for _ in range(3)]
    torch.cuda.synchronize()
    for f in FIELDS + ("densify",):
        assert torch.isfinite(runs[0][f]).all(), f
        for k in (1, 2):
            assert torch.equal(runs[0][f], runs[k][f]), f"{config} {f}: run {k} differs"
    assert runs[0]["means"].abs().max() > 0
    r.close()
