"""Forward + backward of one multiview view (profiling driver for K6:
ncu -k regex:backward ...).  GPU box only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def main():
    view = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    scene = S.make_scene(os.environ.get("TRACE_CONFIG", "multiview"))
    cam = S.make_views(os.environ.get("TRACE_CONFIG", "multiview"))[view]
    r = gut.Renderer(scene)
    g = torch.Generator(device="cuda").manual_seed(0)
    for _ in range(reps):
        out = r.render(cam)[:3]
        gr = torch.randn(out[0].shape, device="cuda", generator=g)
        ga = torch.randn(out[1].shape, device="cuda", generator=g)
        r.backward(cam, None, out, gr, ga)
    torch.cuda.synchronize()
    r.close()


if __name__ == "__main__":
    main()
