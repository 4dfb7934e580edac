"""GPU parity: the sm_100a path (through the C ABI) against the fp64 oracle on
the same seeded inputs.  Stage by stage (K1 projection, K2/K3/K4 binning,
sort and ranges, K5 blend on the GPU's own lists) and end to end, on the
tiny config and its camera variants (ragged edges: 64x64 -> 4x4 tiles; 70x50
-> partial tiles), on reduced-N / reduced-resolution versions of the large
configs (several tiles, ragged tails), and at full size on sampled tiles."""
import dataclasses
import math

import numpy as np
import pytest

import scenegen as S
from gpu_common import (ALPHA_BAND, TERM_BAND, TOL_ALPHA, TOL_DEPTH_REL, TOL_RGB, assert_images_close, gpu_lists, gpu_render, pixel_mask)

pytestmark = pytest.mark.gpu

OPT = S.RenderOptions()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import build
    build.build()


def _proj_parity(scene, cam, g, o_proj, opt=OPT):
    gp = g["proj"]
    vis_g = gp["tiles"] > 0
    vis_o = o_proj["reason"] == 0
    amb = (o_proj["cull_ambig"] != 0) | (o_proj["bin_ambig"] != 0)
    # culling identical outside the ambiguity set
    bad = (vis_g != vis_o) & ~amb
    assert not bad.any(), np.nonzero(bad)[0][:10]
    both = vis_g & vis_o & ~amb
    # tile counts bit-exact outside the 1e-3 px band
    np.testing.assert_array_equal(gp["tiles"][both], o_proj["tiles"][both])
    # binning geometry: mean and extent edges within half the 1e-3 px band,
    # covariance within 1e-3 relative (fp32 pixel coordinates)
    # (the debug record is fp32: add its own representation error, 2 ulp, for
    # the "wide" Gaussians whose fp64 ellipse sits far from the image)
    # Relative term 2e-6 * extent: R(q) and s are formed from the fp32 inputs on
    # the GPU, so sigma points differ from the fp64 oracle's by ~1e-7 relative,
    # which the projection of edge-on Gaussians grazing the near plane (extents
    # of 10^4 px) amplifies; their tile sets still match bit for bit (above).
    hx_o, hy_o = o_proj["hx"][both], o_proj["hy"][both]
    for v, h_o in (("vx", hx_o), ("vy", hy_o)):
        tol = 5e-4 + 2e-6 * h_o + 2 * np.spacing(np.abs(gp[v][both]).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(gp[v][both] - o_proj[v][both]) < tol), v
    for f, h in (("cxx", "hx"), ("cyy", "hy")):
        rel = np.abs(gp[f][both] - o_proj[f][both]) / np.abs(o_proj[f][both])
        assert rel.max(initial=0) < 1e-3, f
        hg = np.sqrt(gp["k2"][both].astype(np.float64) * gp[f][both])
        assert np.all(np.abs(hg - o_proj[h][both]) < 5e-4 + 2e-6 * o_proj[h][both]), h
    sc = np.sqrt(o_proj["cxx"][both] * o_proj["cyy"][both])
    assert (np.abs(gp["cxy"][both] - o_proj["cxy"][both]) / sc).max(initial=0) < 1e-3
    rel = np.abs(gp["depth"][both] - o_proj["depth"][both]) / o_proj["depth"][both]
    assert rel.max(initial=0) < 2e-6
    assert np.abs(gp["rgb"][both] - o_proj["rgb"][both]).max(initial=0) < 1e-5
    np.testing.assert_array_equal(gp["rect"][both].astype(np.int32), o_proj["rect"][both])
    return int(both.sum()), int(amb.sum())


def _sort_parity(scene, cam, g):
    """K2-K4 on the GPU's own K1 output: the sorted pairs are exactly the pairs
    implied by the GPU tile counts, ordered by (tile, fp32 depth, index)."""
    gp = g["proj"]
    pairs = g["sorted"]
    K = pairs.shape[0]
    assert K == int(gp["tiles"].sum()) == g["stats"]["n_keys"]
    tiles, gids = pairs[:, 0].astype(np.int64), pairs[:, 1].astype(np.int64)
    depth = gp["depth"][gids]
    order = np.lexsort((gids, depth, tiles))
    assert np.array_equal(order, np.arange(K)), "not sorted by (tile, depth, gid)"
    np.testing.assert_array_equal(np.bincount(gids, minlength=scene.count), gp["tiles"])
    assert len(set(zip(tiles.tolist(), gids.tolist()))) == K
    # each Gaussian's tiles lie in its rectangle
    r = gp["rect"][gids].astype(np.int64)
    tx, ty = tiles % cam.tiles[0], tiles // cam.tiles[0]
    assert np.all((tx >= r[:, 0]) & (tx <= r[:, 2]) & (ty >= r[:, 1]) & (ty <= r[:, 3]))
    # ranges
    ranges = g["ranges"]
    for t in range(ranges.shape[0]):
        a, b = ranges[t]
        assert np.all(tiles[a:b] == t)
        assert (b - a) == int((tiles == t).sum())
    # depth order of the visible Gaussians
    vis = np.nonzero(gp["tiles"] > 0)[0]
    exp = vis[np.lexsort((vis, gp["depth"][vis]))]
    np.testing.assert_array_equal(g["order"], exp)


def _tile_sets_match_oracle(g, o_proj, cam, opt):
    """For non-ambiguous Gaussians the GPU's (tile, gid) set equals the oracle's."""
    from oracle import oracle as O
    tiles_o, gids_o, _ = O.tile_lists(o_proj, cam, opt)
    amb = (o_proj["cull_ambig"] != 0) | (o_proj["bin_ambig"] != 0)
    so = set((int(t), int(i)) for t, i in zip(tiles_o, gids_o) if not amb[i])
    sg = set((int(t), int(i)) for t, i in g["sorted"] if not amb[i])
    assert so == sg, (len(so - sg), len(sg - so))


def _blend_parity(scene, cam, g, opt=OPT, max_excluded=0.01):
    """K5 isolated: oracle O6 on the GPU's own sorted lists."""
    from oracle import oracle as O
    proj = O.preprocess(scene, cam, opt)
    gids, ranges = gpu_lists(g, cam.tiles[0] * cam.tiles[1])
    rgb, alpha, depth, diag = O.composite(scene, proj, gids, ranges, cam, opt)
    o = dict(rgb=rgb, alpha=alpha, depth=depth)
    m = (diag["min_alpha_gap"] > ALPHA_BAND) & (diag["min_term_gap"] > TERM_BAND)
    return assert_images_close(g, o, m, f"blend {cam.model}/{cam.shutter}", max_excluded=max_excluded)


def _full_parity(scene, cam, opt=OPT, max_excluded=0.01, label=""):
    from oracle import oracle as O
    g = gpu_render(scene, cam, opt)
    o = O.render(scene, cam, opt)
    _proj_parity(scene, cam, g, o["proj"], opt)
    _sort_parity(scene, cam, g)
    _tile_sets_match_oracle(g, o["proj"], cam, opt)
    _blend_parity(scene, cam, g, opt, max_excluded=max_excluded)
    res = assert_images_close(g, o, pixel_mask(o["diag"], cam), label or f"e2e {cam.model}/{cam.shutter}",
                              max_excluded=max_excluded)
    # invariants on the GPU output
    T = 1 - g["alpha"]
    assert np.all(np.isfinite(g["rgb"])) and np.all(np.isfinite(g["depth"]))
    assert np.all(T >= 0) and np.all(T <= 1) and np.all(g["alpha"] <= 1 - opt.transmittance_min + 1e-6)
    return g, o, res


@pytest.mark.parametrize("variant", S.TINY_VARIANTS)
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_tiny_parity(variant, seed):
    scene, cam = S.tiny(seed, variant)
    _full_parity(scene, cam)


@pytest.mark.parametrize("variant", ["pinhole", "fisheye", "rs"])
def test_tiny_ragged_and_sh3(variant):
    """70x50 image (partial tiles on both edges), 200 Gaussians, SH degree 3."""
    scene, cam = S.tiny(7, variant, n=200, size=64, sh_degree=3)
    cam = dataclasses.replace(cam, width=70, height=50, cx=35.0, cy=25.0)
    _full_parity(scene, cam)


def test_tiny_aabb_mode():
    scene, cam = S.tiny(5, "pinhole", n=128)
    _full_parity(scene, cam, S.RenderOptions(tile_cull=0))


def test_nondefault_ut_params_and_background():
    scene, cam = S.tiny(6, "opencv", n=128)
    opt = S.RenderOptions(ut_alpha=0.8, ut_beta=1.0, ut_kappa=1.0, background=(0.2, 0.4, 0.6))
    _full_parity(scene, cam, opt)


@pytest.mark.parametrize("config,n,factor,view", [
    ("mipnerf360", 60_000, 0.25, 0),
    ("scannetpp", 40_000, 0.2, 3),
    ("waymo", 80_000, 0.15, 1),
    ("multiview", 100_000, 0.2, 5),
])
def test_reduced_configs(config, n, factor, view):
    """The large configs' recipes at reduced N and resolution (seconds for the
    oracle), spanning tens of tiles with ragged edges."""
    scene = S.make_scene(config, n=n)
    cam = S.scaled_camera(S.make_views(config)[view], factor)
    g, o, _ = _full_parity(scene, cam, max_excluded=0.02, label=f"{config} n={n} x{factor}")
    assert g["stats"]["n_keys"] > 0


CNT_NITEMS = 26  # csrc/launch.h: blend segment slots of the render (> n_tiles iff lists were split)


@pytest.mark.parametrize("seg,window", [(256, 1), (256, 3), (512, 2)])
@pytest.mark.parametrize("config,n,factor,view", [("multiview", 100_000, 0.2, 5), ("waymo", 2_000_000, 0.5, 1)])
def test_segmented_blend(config, n, factor, view, seg, window, monkeypatch):
    """K5's split-list machinery at short segments, so that most tiles span
    many segments: speculative passes, look-back, checkpointed re-runs,
    successor grants and the in-order combine against the oracle (the
    defaults only split the longest lists)."""
    monkeypatch.setenv("GUT_BLEND_SEG", str(seg))
    monkeypatch.setenv("GUT_BLEND_WINDOW", str(window))
    scene = S.make_scene(config, n=n)
    cam = S.scaled_camera(S.make_views(config)[view], factor)
    g = gpu_render(scene, cam)
    # K5 isolated (oracle O6 on the GPU's own lists): the dense full street
    # scene has more pixels inside the alpha / termination bands (all counted)
    _blend_parity(scene, cam, g, max_excluded=0.05 if config == "waymo" else 0.02)
    lens = g["ranges"][:, 1].astype(np.int64) - g["ranges"][:, 0]
    assert (lens > seg).sum() >= 4, "the case must split several tiles"
    assert int(g["counters"][CNT_NITEMS]) >= len(lens) + (lens > seg).sum(), "segments in effect"


@pytest.mark.parametrize("config,view", [("multiview", 0), ("waymo", 1), ("mipnerf360", 3), ("scannetpp", 5)])
def test_full_size_sampled_tiles(config, view):
    """Every BASELINE config at full size (multiview: configs[4] in the launch
    configuration bench.py times; waymo: 2M Gaussians, OpenCV + rolling
    shutter 1920x1280): 16 random tiles and the 8 longest lists (split into
    segments, re-runs) against the oracle."""
    from oracle import oracle as O
    scene = S.make_scene(config)
    cam = S.make_views(config)[view]
    g = gpu_render(scene, cam, reserve=int(scene.count * 12))
    tx, ty = cam.tiles
    rng = np.random.default_rng(0)
    lens = g["ranges"][:, 1].astype(np.int64) - g["ranges"][:, 0]
    longest = np.argsort(-lens)[:8]
    rest = np.setdiff1d(np.arange(tx * ty), longest)
    sub = np.sort(np.concatenate([longest, rng.choice(rest, 16, replace=False)])).astype(np.int32)
    o = O.render(scene, cam, OPT, tile_subset=sub)
    sampled = np.zeros((cam.height, cam.width), bool)
    for t in sub:
        x0, y0 = (t % tx) * 16, (t // tx) * 16
        sampled[y0:y0 + 16, x0:x0 + 16] = True
    mask = sampled & pixel_mask(o["diag"], cam)
    excluded = 1.0 - mask.sum() / sampled.sum()
    e_rgb = np.abs(g["rgb"] - o["rgb"]).max(-1)[mask].max()
    e_a = np.abs(g["alpha"] - o["alpha"])[mask].max()
    ref = np.abs(o["depth"])
    med = np.median(ref[sampled & (ref > 0)])
    e_d = (np.abs(g["depth"] - o["depth"]) / np.maximum(ref, 0.01 * med))[mask].max()
    print(f"full-size sampled {config}: rgb {e_rgb:.2e} alpha {e_a:.2e} depth_rel {e_d:.2e} "
          f"excluded {excluded:.4%} of {int(sampled.sum())} px; K={g['stats']['n_keys']}")
    # (ambiguity bands: alpha-skip, termination, order, binning, cull -- DESIGN §6)
    assert excluded <= 0.01, excluded
    assert e_rgb <= TOL_RGB and e_a <= TOL_ALPHA and e_d <= TOL_DEPTH_REL
    _proj_parity(scene, cam, g, o["proj"])


def test_edge_cases():
    """Empty scene, all-culled scene, a single Gaussian, Gaussians behind the camera."""
    scene, cam = S.tiny(0, "pinhole", n=8)
    empty = scene.subset(np.zeros(0, np.int64))
    g = gpu_render(empty, cam)
    assert np.all(g["alpha"] == 0) and g["stats"]["n_keys"] == 0
    behind = scene.subset(np.arange(8))
    behind.means[:, 2] = -3.0
    g = gpu_render(behind, cam)
    assert np.all(g["alpha"] == 0) and g["stats"]["n_visible"] == 0
    bad = scene.subset(np.arange(8))
    bad.scales[0] = 0.0
    bad.rotations[1] = 0.0
    bad.opacities[2] = 0.0
    bad.means[3, 0] = np.nan
    _full_parity(bad, cam)
    one = scene.subset(np.arange(1))
    _full_parity(one, cam)


def test_determinism_and_modes():
    """Bitwise-identical re-runs; capacity mode == sync mode; host outputs ==
    device outputs."""
    import torch
    from paper_2412_12507_b200 import gut
    scene = S.make_scene("multiview", n=50_000)
    cam = S.scaled_camera(S.make_views("multiview")[2], 0.3)
    a = gpu_render(scene, cam)
    b = gpu_render(scene, cam)
    c = gpu_render(scene, cam, reserve=2_000_000)
    for k in ("rgb", "alpha", "depth"):
        assert np.array_equal(a[k], b[k]) and np.array_equal(a[k], c[k])
    assert np.array_equal(a["sorted"], c["sorted"])
    r = gut.Renderer(scene)
    H, W = cam.height, cam.width
    hr = torch.empty((H, W, 3), pin_memory=True)
    ha = torch.empty((H, W), pin_memory=True)
    hd = torch.empty((H, W), pin_memory=True)
    o = gut.gut_outputs(hr.data_ptr(), ha.data_ptr(), hd.data_ptr(), 0, 0)
    gut.gut_render(r.ctx, r.scene, gut.make_camera(cam), gut.make_options(), o)
    torch.cuda.synchronize()
    assert np.array_equal(hr.numpy(), a["rgb"]) and np.array_equal(ha.numpy(), a["alpha"])
    r.close()


def test_invalid_arguments():
    from paper_2412_12507_b200 import gut
    scene, cam = S.tiny(0)
    r = gut.Renderer(scene)
    bad = dataclasses.replace(cam, model="fisheye", fov_limit=0.0)
    with pytest.raises(gut.GutError) as e:
        r.render(bad)
    assert e.value.status == 1 and "fov_limit" in str(e.value)
    with pytest.raises(gut.GutError):
        r.render(cam, S.RenderOptions(ut_alpha=0.0))
    with pytest.raises(gut.GutError) as e:
        r.render(dataclasses.replace(cam, model="ortho", shutter="top_to_bottom"))
    assert e.value.status == 2
    r.close()


def test_capacity_overflow_is_sticky():
    """A reserved render whose key count exceeds the reservation is reported by
    the next synchronising call (gut.h gut_workspace_reserve), even when the
    truncated render itself asked for no stats; the latch then clears."""
    import torch
    from paper_2412_12507_b200 import gut
    scene = S.make_scene("multiview", n=50_000)
    cam = S.scaled_camera(S.make_views("multiview")[2], 0.3)
    K = gpu_render(scene, cam)["stats"]["n_keys"]
    assert K > 1000
    r = gut.Renderer(scene, reserve_keys=K // 3, max_wh=(cam.width, cam.height))
    r.render(cam, stats=False)                      # truncated, no error possible here
    r.render(cam, stats=False)
    with pytest.raises(gut.GutError) as e:
        gut.gut_check(r.ctx)
    assert e.value.status == 4                      # GUT_E_CAPACITY
    gut.gut_check(r.ctx)                            # cleared
    r.render(cam, stats=False)
    with pytest.raises(gut.GutError) as e:          # a stats render reports earlier truncation too
        r.render(cam, stats=True)
    assert e.value.status == 4
    gut.gut_check(r.ctx)
    with pytest.raises(gut.GutError) as e:
        r.render(cam, timing=True, stats=False)
        gut.gut_timing_read(r.ctx)
    assert e.value.status == 4
    gut.gut_check(r.ctx)
    torch.cuda.synchronize()
    r.close()
    big = gut.Renderer(scene, reserve_keys=2 * K, max_wh=(cam.width, cam.height))
    big.render(cam, stats=False)
    gut.gut_check(big.ctx)                          # no overflow, no error
    big.close()


def test_4k_fisheye_sampled_tiles():
    """Scale beyond the configs: the bench scene's recipe (1M Gaussians) at
    3840x2160 fisheye (240 x 135 = 32,400 tiles: 15-bit tile ids, the two
    8-bit tile passes) -- 24 sampled tiles (the 8 longest lists + 16 random)
    against the oracle, and the sorted lists of those tiles bit-exact."""
    from oracle import oracle as O
    scene = S.make_scene("multiview", n=1_000_000)
    cam = S.scaled_camera(S.make_views("multiview")[3], 2.0)
    assert cam.width == 3840 and cam.height == 2160
    g = gpu_render(scene, cam, reserve=int(scene.count * 12))
    tx, ty = cam.tiles
    assert tx * ty > 1 << 14  # (15 significant tile-id bits)
    rng = np.random.default_rng(4)
    lens = g["ranges"][:, 1].astype(np.int64) - g["ranges"][:, 0]
    longest = np.argsort(-lens)[:8]
    sub = np.sort(np.concatenate([longest, rng.choice(np.setdiff1d(np.arange(tx * ty), longest), 16,
                                                      replace=False)])).astype(np.int32)
    o = O.render(scene, cam, OPT, tile_subset=sub)
    sampled = np.zeros((cam.height, cam.width), bool)
    for t in sub:
        sampled[(t // tx) * 16:(t // tx) * 16 + 16, (t % tx) * 16:(t % tx) * 16 + 16] = True
    mask = sampled & pixel_mask(o["diag"], cam)
    excluded = 1.0 - mask.sum() / sampled.sum()
    e_rgb = np.abs(g["rgb"] - o["rgb"]).max(-1)[mask].max()
    e_a = np.abs(g["alpha"] - o["alpha"])[mask].max()
    print(f"4k fisheye sampled: rgb {e_rgb:.2e} alpha {e_a:.2e} excluded {excluded:.4%}; K={g['stats']['n_keys']}")
    assert excluded <= 0.01 and e_rgb <= TOL_RGB and e_a <= TOL_ALPHA
    # the sampled tiles' lists equal the oracle's (tile, fp32 depth, index) order
    tiles_o, gids_o, ranges_o = O.tile_lists(O.preprocess(scene, cam, OPT), cam, OPT)
    amb = (o["proj"]["cull_ambig"] != 0) | (o["proj"]["bin_ambig"] != 0)
    pairs = g["sorted"]
    for t in sub:
        a, b = g["ranges"][t]
        lg = [int(x) for x in pairs[a:b, 1] if not amb[x]] if b > a else []
        ao, bo = ranges_o[t]
        lo = [int(x) for x in gids_o[ao:bo] if not amb[x]]
        assert lg == lo, t
