"""Diagnostics: the Gaussians with the largest K1 (GPU) vs oracle differences."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def main(config="mipnerf360", n=60000, factor=0.25, view=0):
    scene = S.make_scene(config, n=n)
    cam = S.scaled_camera(S.make_views(config)[view], factor)
    opt = S.RenderOptions()
    r = gut.Renderer(scene)
    r.render(cam, opt)
    g = r.stage(gut.STAGE_PROJECT)
    o = O.preprocess(scene, cam, opt)
    both = (g["tiles"] > 0) & (o["reason"] == 0)
    idx = np.nonzero(both)[0]
    err = np.maximum(np.abs(g["vx"][idx] - o["vx"][idx]), np.abs(g["vy"][idx] - o["vy"][idx]))
    for j in np.argsort(-err)[:5]:
        i = idx[j]
        R = O.quat_to_rot(scene.rotations[i].astype(float))
        Rc, cc = O.pose_at(cam, 0.0)
        X = O.sigma_points(scene.means[i].astype(float), R, scene.scales[i].astype(float), 0.0)
        uv = [O.project_point(cam, opt, x)[1] for x in X]
        print(f"gid {i} err {err[j]:.3e} v_gpu ({g['vx'][i]:.5f},{g['vy'][i]:.5f}) v_orc ({o['vx'][i]:.5f},"
              f"{o['vy'][i]:.5f}) h ({o['hx'][i]:.2f},{o['hy'][i]:.2f}) depth {o['depth'][i]:.3f} "
              f"cov_rel {abs(g['cxx'][i]-o['cxx'][i])/o['cxx'][i]:.2e} sigma pts max|uv-c| "
              f"{max(abs(u[0]-cam.cx) for u in uv):.1f},{max(abs(u[1]-cam.cy) for u in uv):.1f} "
              f"s {scene.scales[i]} ambig {o['bin_ambig'][i]} tiles {g['tiles'][i]}/{o['tiles'][i]}")
    hg = np.sqrt(g["k2"][idx].astype(np.float64) * g["cxx"][idx])
    herr = np.abs(hg - o["hx"][idx])
    for j in np.argsort(-herr)[:5]:
        i = idx[j]
        print(f"h: gid {i} |dh| {herr[j]:.3e} h {o['hx'][i]:.4f} k2 gpu {g['k2'][i]:.7f} orc {o['k2'][i]:.7f} "
              f"cxx gpu {g['cxx'][i]:.7f} orc {o['cxx'][i]:.7f} sigma {scene.opacities[i]!r} "
              f"tiles {g['tiles'][i]}/{o['tiles'][i]} ambig {o['bin_ambig'][i]}")
    r.close()


if __name__ == "__main__":
    main()
