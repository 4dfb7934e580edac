"""Per-stage device times of the bench workload with the library named by GUT_LIB
(tuning variants built with GUT_LIB_OUT / GUT_EXTRA_FLAGS).  GPU box only.
usage: GUT_LIB=... python tools/stage_bench.py [views] [label]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    label = sys.argv[2] if len(sys.argv) > 2 else os.environ.get("GUT_LIB", "default")
    config = os.environ.get("TRACE_CONFIG", "multiview")
    scene = S.make_scene(config)
    cams = S.make_views(config)[:nv]
    r = gut.Renderer(scene)
    st = [r.render(c, timing=True)[3] for c in cams]
    kmax = max(s.n_keys for s in st)
    gut.gut_workspace_reserve(r.ctx, int(kmax * 1.05) + 65536, scene.count, cams[0].width, cams[0].height)
    for rep in range(2):
        for c in cams:
            r.render(c, timing=True, stats=False)
        torch.cuda.synchronize()
        ms, n = gut.gut_timing_read(r.ctx, reset=True)
    print(label, {k: round(v / n, 4) for k, v in ms.items()}, flush=True)
    r.close()


if __name__ == "__main__":
    main()
