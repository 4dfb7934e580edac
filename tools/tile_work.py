"""Diagnostics: per-tile list length vs entries the blend actually visited, for
the bench workload (multiview config).  Run on the GPU box."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def main():
    views = [int(v) for v in (sys.argv[1:] or ["0", "1", "2", "3"])]
    scene = S.make_scene("multiview")
    cams = S.make_views("multiview")
    r = gut.Renderer(scene)
    for v in views:
        cam = cams[v]
        for _ in range(2):  # the first render of a process pays module-load / LUT costs
            _, _, _, st = r.render(cam, timing=True)
        tw = r.stage(gut.STAGE_TILE_WORK)
        L, P = tw[:, 0].astype(np.int64), tw[:, 1].astype(np.int64)
        tx = cam.tiles[0]
        ms = list(st.ms_stage)
        order = np.argsort(-P)
        print(f"view {v}: K={st.n_keys} vis={st.n_visible} blend {ms[5]:.3f} ms total {ms[6]:.3f} ms; "
              f"sum len={L.sum()} sum processed={P.sum()} max len={L.max()} max processed={P.max()}")
        print("  len pct 50/90/99/99.9/max:", np.percentile(L, [50, 90, 99, 99.9]).astype(int), L.max())
        print("  proc pct 50/90/99/99.9/max:", np.percentile(P, [50, 90, 99, 99.9]).astype(int), P.max())
        for t in order[:8]:
            print(f"    tile ({t % tx},{t // tx}) len {L[t]} processed {P[t]}")
    r.close()


if __name__ == "__main__":
    main()
