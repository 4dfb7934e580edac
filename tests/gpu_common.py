"""Shared helpers for the -m gpu parity tests: run the CUDA path through the
C ABI, run the oracle on the same seeded inputs, compare with the
north_star tolerances and the ambiguity masks of SURVEY §8(c).5."""
import numpy as np

import scenegen as S

# BASELINE.json north_star tolerances
TOL_RGB = 2e-4           # absolute, per fp32 RGB channel
TOL_ALPHA = 2e-4         # absolute
TOL_DEPTH_REL = 1e-3     # relative on depth
# ambiguity bands
ALPHA_BAND = 1e-5        # |alpha - alpha_min| <= band: the alpha-skip may flip
TERM_BAND = 2e-8         # |T' - T_min| <= band: the termination may flip
ORDER_BAND = 8 * 2 ** -23  # contributing depths within 8 fp32 ulps: order may swap


def gpu_render(scene, cam, opt=None, reserve=None, timing=False):
    import torch
    from paper_2412_12507_b200 import gut
    r = gut.Renderer(scene, reserve_keys=reserve, max_wh=(max(cam.width, 16), max(cam.height, 16)))
    rgb, alpha, depth, st = r.render(cam, opt, timing=timing)
    torch.cuda.synchronize()
    out = dict(rgb=rgb.cpu().numpy(), alpha=alpha.cpu().numpy(), depth=depth.cpu().numpy(), stats=st.as_dict(),
               proj=r.stage(gut.STAGE_PROJECT), sorted=r.stage(gut.STAGE_SORTED), ranges=r.stage(gut.STAGE_RANGES),
               order=r.stage(gut.STAGE_DEPTH_ORDER), counters=r.stage(gut.STAGE_COUNTERS))
    r.close()
    return out


def pixel_mask(diag):
    """True where the strict comparison applies."""
    m = (diag["min_alpha_gap"] > ALPHA_BAND) & (diag["min_term_gap"] > TERM_BAND)
    m &= diag["min_order_gap"] > ORDER_BAND
    m &= (diag["amb_bin"] == 0) & (diag["amb_cull"] == 0)
    return m


def compare_images(g, o, mask, label=""):
    """Returns (max abs rgb err, max abs alpha err, max rel depth err, excluded fraction)."""
    d_rgb = np.abs(g["rgb"] - o["rgb"]).max(-1)
    d_a = np.abs(g["alpha"] - o["alpha"])
    ref = np.abs(o["depth"])
    med = np.median(ref[ref > 0]) if np.any(ref > 0) else 1.0
    d_d = np.abs(g["depth"] - o["depth"]) / np.maximum(ref, 0.01 * med)
    e_rgb = float(d_rgb[mask].max()) if mask.any() else 0.0
    e_a = float(d_a[mask].max()) if mask.any() else 0.0
    e_d = float(d_d[mask].max()) if mask.any() else 0.0
    excl = 1.0 - float(mask.mean())
    return e_rgb, e_a, e_d, excl


def assert_images_close(g, o, mask, label="", max_excluded=0.01):
    e_rgb, e_a, e_d, excl = compare_images(g, o, mask, label)
    msg = f"{label}: rgb {e_rgb:.2e} alpha {e_a:.2e} depth_rel {e_d:.2e} excluded {excl:.4%}"
    print(msg)
    assert e_rgb <= TOL_RGB, msg
    assert e_a <= TOL_ALPHA, msg
    assert e_d <= TOL_DEPTH_REL, msg
    assert excl <= max_excluded, msg
    return e_rgb, e_a, e_d, excl


def gpu_lists(g, n_tiles):
    """GPU sorted pairs -> (gids, ranges[n_tiles,2]) in the oracle's format."""
    pairs = g["sorted"]
    gids = pairs[:, 1].astype(np.int32) if pairs.size else np.zeros(0, np.int32)
    ranges = g["ranges"].astype(np.int32).reshape(n_tiles, 2)
    return gids, ranges
