"""The paper's variants on one B200: "Ours" vs "Ours (sorted)"
(per-ray k-buffer, Tab. 2 / P:L271-275) and the generalized kernel degrees of
Tab. 4, per config at full size: the first V views one at a time
on one stream (library stage events, capacity mode).  GPU box only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402

VARIANTS = [(0, 2), (16, 2), (16, 3), (16, 4), (16, 5), (16, 8), (0, 4), (8, 2), (4, 2), (1, 2)]


def run(config, nviews):
    scene = S.make_scene(config)
    cams = S.make_views(config)[:nviews]
    W, H = max(c.width for c in cams), max(c.height for c in cams)
    r = gut.Renderer(scene)
    rows = []
    for kbuf, deg in VARIANTS:
        opt = S.RenderOptions(kbuffer=kbuf, kernel_degree=deg)
        st = [r.render(c, opt, timing=True)[3] for c in cams]
        kmax = max(s.n_keys for s in st)
        gut.gut_workspace_reserve(r.ctx, int(kmax * 1.05) + 65536, scene.count, W, H)
        for c in cams:
            r.render(c, opt, timing=True, stats=False)
        torch.cuda.synchronize()
        gut.gut_timing_read(r.ctx, reset=True)
        for c in cams:
            r.render(c, opt, timing=True, stats=False)
        torch.cuda.synchronize()
        ms, n = gut.gut_timing_read(r.ctx, reset=True)
        ms = {k: v / n for k, v in ms.items()}
        row = {"config": config, "variant": "Ours" if kbuf == 0 else f"Ours (sorted) k={kbuf}", "degree": deg,
               "views": len(cams), "ms_stage": ms, "fps": 1e3 / ms["total"],
               "keys": sum(s.n_keys for s in st) / len(st),
               "pairs_contrib_per_px": sum(s.pairs_contributing for s in st) / len(st) / (cams[0].width * cams[0].height)}
        print(json.dumps(row), flush=True)
        rows.append(row)
    r.close()
    return rows


def main():
    for cfg in sys.argv[1:] or ["mipnerf360", "multiview"]:
        run(cfg, int(os.environ.get("VIEWS", "8")))


if __name__ == "__main__":
    main()
