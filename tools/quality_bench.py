"""Projection quality on synthetic scenes (PAPER Supp. C analogues; the
paper's own numbers need the trained MipNeRF360 *bicycle* scene): median and
90th-percentile KL(MC || UT) vs KL(MC || EWA) per Gaussian whose UT mean
lands in the image, for
  (1) static / rolling-shutter pinhole and fisheye (Fig. 12 analogue),
  (2) equidistant fisheye over the field of view (Fig. 9 analogue),
  (3) OpenCV radial distortion k2 in {0, 0.25, 0.5}, static and RS (Fig. 10).
500 Monte-Carlo samples per Gaussian, gut_projection_quality on the GPU (fp64),
plus its kernel time.  GPU box only.  Output: JSON lines."""
import dataclasses
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402

N = int(os.environ.get("QN", "200000"))
SCALE = float(os.environ.get("QSCALE", "1"))  # Gaussian size multiplier (the recipe's s_med 0.007 is nearly linear)


def rs(cam):
    """Rolling shutter over the readout (top to bottom): 0.35 m sideways, 2 deg yaw (Supp. C / PAPER L588)."""
    q0 = np.array(cam.q_c2w[0])
    w, x, y, z = q0
    R0 = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                   [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                   [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    a = math.radians(2.0)
    Ry = np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]])
    q1 = S._mat_to_quat(R0 @ Ry)
    c0 = np.array(cam.c_w[0])
    c1 = c0 + R0 @ np.array([0.35, 0.0, 0.0])
    return dataclasses.replace(cam, shutter="top_to_bottom", q_c2w=(tuple(q0), tuple(q1)), c_w=(tuple(c0), tuple(c1)))


def run(r, cam, label, **extra):
    t0 = time.perf_counter()
    q = r.projection_quality(cam, None, n_samples=500, seed=1)
    dt = time.perf_counter() - t0
    v = q["valid"] == 1
    inside = (q["ut"][:, 0] >= 0) & (q["ut"][:, 0] < cam.width) & (q["ut"][:, 1] >= 0) & (q["ut"][:, 1] < cam.height)
    m = v & inside
    row = {"case": label, "scale_x": SCALE, "gaussians": int(m.sum()),
           "kl_ut_median": float(np.median(q["kl_ut"][m])), "kl_ewa_median": float(np.median(q["kl_ewa"][m])),
           "kl_ut_p90": float(np.percentile(q["kl_ut"][m], 90)), "kl_ewa_p90": float(np.percentile(q["kl_ewa"][m], 90)),
           "ut_better_frac": float((q["kl_ut"][m] < q["kl_ewa"][m]).mean()), "seconds_incl_copy": dt, **extra}
    print(json.dumps(row), flush=True)


def main():
    scene = S.make_scene("multiview", n=N)
    scene.scales[:] *= SCALE
    base = S.make_views("multiview")[0]          # fisheye 1920x1080, f = 620, theta_max 105 deg
    W, H = 1280, 720
    r = gut.Renderer(scene)
    pin = dataclasses.replace(base, model="pinhole", width=W, height=H, fx=640.0, fy=640.0, cx=W / 2, cy=H / 2,
                              k=(0,) * 6, fov_limit=0.0)
    fe = dataclasses.replace(base, width=W, height=H, cx=W / 2, cy=H / 2, fx=420.0, fy=420.0,
                             fov_limit=math.radians(100.0))
    # kernel time alone (device events)
    buf = torch.empty((scene.count, 18), dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gut.gut_projection_quality(r.ctx, r.scene, gut.make_camera(fe), gut.make_options(), 500, 1, buf.data_ptr())
    e0.record()
    gut.gut_projection_quality(r.ctx, r.scene, gut.make_camera(fe), gut.make_options(), 500, 1, buf.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"kernel_ms": e0.elapsed_time(e1), "gaussians": scene.count, "samples": 500,
                      "projections_per_s": scene.count * 507 / (e0.elapsed_time(e1) * 1e-3)}), flush=True)
    # (1) Fig. 12 analogue
    for lab, cam in (("pinhole static", pin), ("pinhole RS", rs(pin)), ("fisheye static", fe), ("fisheye RS", rs(fe))):
        run(r, cam, lab)
    # (2) Fig. 9 analogue: equidistant fisheye, FoV across the image width
    for fov in (60, 90, 120, 150, 180):
        f = (W / 2) / math.radians(fov / 2)
        cam = dataclasses.replace(fe, fx=f, fy=f, fov_limit=math.radians(max(fov / 2 * 1.2, 60)))
        run(r, cam, f"fisheye FoV {fov}", fov_deg=fov)
    # (3) Fig. 10 analogue: OpenCV radial k2, static and RS
    for k2 in (0.0, 0.25, 0.5):
        cam = dataclasses.replace(pin, model="opencv", k=(0.0, k2, 0, 0, 0, 0), fov_limit=1.2)
        run(r, cam, f"opencv k2={k2}", k2=k2)
        run(r, rs(cam), f"opencv k2={k2} RS", k2=k2)
    r.close()


if __name__ == "__main__":
    main()
