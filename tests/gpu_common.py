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
# |alpha - alpha_min| <= band: the alpha-skip may flip.  Near alpha_min the GPU
# alpha error is alpha_min |d omega^2| / 2: with the largest |d omega^2| implied
# by SURVEY App. B's worst |d alpha| (4.8e-6 at alpha ~ 0.5, i.e. |d omega^2|
# ~ 2e-5) that is ~4e-8, so 1e-6 keeps a 25x margin.
ALPHA_BAND = 1e-6
# |T' - T_min| <= band: the termination may flip.  T carries the relative error
# sum_i |d alpha_i| / (1 - alpha_i) of every earlier hit (~1e-4 relative with
# App. B's |d alpha| over 15-30 hits), i.e. ~1.4e-8 at T = T_min.
TERM_BAND = 2e-8
# order margin (oracle min_order_gap: the relative depth perturbation that could
# swap two contributing entries under the (fp32 depth key, index) order,
# reading R13').  Global shutter: K1 forms the depth in fp64 like the oracle
# (differences ~1e-16), so only keys within 1e-12 of a rounding boundary can
# differ.  Rolling shutter: the depth is taken at the centre's shutter time,
# solved to 1e-4 px on the GPU (R14) -> depth differences up to ~1e-8 relative.
ORDER_BAND_GLOBAL = 1e-12
ORDER_BAND_RS = 2e-8


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


def order_band(cam):
    return ORDER_BAND_GLOBAL if cam is None or cam.shutter == "global" else ORDER_BAND_RS


def pixel_mask(diag, cam=None):
    """True where the strict comparison applies (cam: selects the order band)."""
    m = (diag["min_alpha_gap"] > ALPHA_BAND) & (diag["min_term_gap"] > TERM_BAND)
    m &= diag["min_order_gap"] > order_band(cam)
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
