"""Debug: worst K1 extent deviations vs the oracle for one full-size view."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import scenegen as S
from oracle import oracle as O
from gpu_common import gpu_render

config, view = sys.argv[1], int(sys.argv[2])
scene = S.make_scene(config)
cam = S.make_views(config)[view]
g = gpu_render(scene, cam, reserve=int(scene.count * 12))
o = O.preprocess(scene, cam, S.RenderOptions())
gp = g["proj"]
both = (gp["tiles"] > 0) & (o["reason"] == 0) & (o["cull_ambig"] == 0) & (o["bin_ambig"] == 0)
for f, h in (("cxx", "hx"), ("cyy", "hy")):
    hg = np.sqrt(gp["k2"].astype(np.float64) * gp[f])
    err = np.abs(hg - o[h]) - (5e-4 + 1e-6 * o[h])
    idx = np.nonzero(both & (err > 0))[0]
    print(f, "violations", len(idx))
    for i in idx[:8]:
        print(f"  i={i} gpu {hg[i]:.6f} orc {o[h][i]:.6f} d={hg[i]-o[h][i]:.3e} vx {o['vx'][i]:.1f} vy {o['vy'][i]:.1f} "
              f"cov {o[f][i]:.4e} gpu_cov {gp[f][i]:.4e} k2 {o['k2'][i]:.5f} gk2 {gp['k2'][i]:.5f} depth {o['depth'][i]:.3f} "
              f"tiles {gp['tiles'][i]} scale {scene.scales[i]}")
