"""Key-count distribution of the K2 'big' Gaussians (tile rectangle > 3x3) of one view."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import scenegen as S
from gpu_common import gpu_render

config, view = sys.argv[1], int(sys.argv[2])
scene = S.make_scene(config)
cam = S.make_views(config)[view]
g = gpu_render(scene, cam, reserve=int(scene.count * 12))
t = g["proj"]["tiles"].astype(np.int64)
r = g["proj"]["rect"].astype(np.int64)
area = (r[:, 2] - r[:, 0] + 1) * (r[:, 3] - r[:, 1] + 1)
big = (t > 0) & (area > 9)
print(config, "keys", t.sum(), "visible", (t > 0).sum(), "big", big.sum(), "big keys", t[big].sum())
for q in (50, 90, 99, 99.9, 100):
    print(f"  big keys per Gaussian p{q}: {np.percentile(t[big], q):.0f}")
print("  Gaussians with > 1000 keys:", (t > 1000).sum(), "keys", t[t > 1000].sum())
