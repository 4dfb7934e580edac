"""Per-config stage timings: every BASELINE.json config
at full size, the first V views one at a time on one stream (library stage
events), plus the 3-in-flight throughput.  GPU box only; no oracle here (the
parity numbers come from tests/test_gpu_parity.py)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def run(config, nviews):
    scene = S.make_scene(config)
    cams = S.make_views(config)[:nviews]
    W, H = max(c.width for c in cams), max(c.height for c in cams)
    r = gut.Renderer(scene)
    st = [r.render(c, timing=True)[3] for c in cams]  # sizing + warm-up (sync mode)
    kmax = max(s.n_keys for s in st)
    gut.gut_workspace_reserve(r.ctx, int(kmax * 1.05) + 65536, scene.count, W, H)
    for c in cams:
        r.render(c, timing=True, stats=False)
    torch.cuda.synchronize()
    gut.gut_timing_read(r.ctx, reset=True)
    for c in cams:
        r.render(c, timing=True, stats=False)
    torch.cuda.synchronize()
    ms, n = gut.gut_timing_read(r.ctx, reset=True)
    ms = {k: v / n for k, v in ms.items()}
    cnt = r.stage(gut.STAGE_COUNTERS)  # last render's device counters (csrc/launch.h)
    px = cams[0].width * cams[0].height
    out = {"config": config, "views": len(cams), "N": scene.count, "res": [cams[0].width, cams[0].height],
           "camera": cams[0].model, "shutter": cams[0].shutter, "ms_stage": ms, "fps": 1e3 / ms["total"],
           "mpix_s": px * 1e-3 / ms["total"], "n_visible": float(np.mean([s.n_visible for s in st])),
           "keys": float(np.mean([s.n_keys for s in st])), "deferred_fp64": int(cnt[28]), "big_k2": int(cnt[37])}
    r.close()
    return out


def main():
    configs = sys.argv[1:] or ["mipnerf360", "scannetpp", "waymo", "multiview"]
    for cfg in configs:
        print(json.dumps(run(cfg, int(os.environ.get("VIEWS", "8")))), flush=True)


if __name__ == "__main__":
    main()
