"""Driver for compute-sanitizer (racecheck / synccheck / memcheck): renders
through every kernel family on small inputs -- tiny scenes of all five camera
variants, a reduced multiview frame with short blend segments (look-back,
speculation, re-runs, work queues), the k-buffer variant, the backward pass,
a capacity-mode render and the projection-quality tool.  GPU box only:
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

os.environ.setdefault("GUT_BLEND_SEG", "256")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def main():
    for variant in S.TINY_VARIANTS:
        scene, cam = S.tiny(1, variant, n=96)
        r = gut.Renderer(scene)
        out = r.render(cam)[:3]
        if variant != "ortho":
            r.backward(cam, S.RenderOptions(), out, torch.randn_like(out[0]), torch.randn_like(out[1]))
        r.render(cam, S.RenderOptions(kbuffer=4))
        r.projection_quality(cam, n_samples=64)
        r.close()
    for config, n, f in (("multiview", 20000, 0.12), ("waymo", 20000, 0.1)):
        scene = S.make_scene(config, n=n)
        cam = S.scaled_camera(S.make_views(config)[1], f)
        r = gut.Renderer(scene, reserve_keys=n * 16, max_wh=(cam.width, cam.height))
        out = r.render(cam)[:3]
        r.render(cam, stats=False)
        r.backward(cam, S.RenderOptions(), out, torch.randn_like(out[0]), torch.randn_like(out[1]))
        r.render(cam, S.RenderOptions(kbuffer=16))
        torch.cuda.synchronize()
        print(config, cam.width, cam.height, "ok", flush=True)
        r.close()
    torch.cuda.synchronize()
    print("sanitize_run done")


if __name__ == "__main__":
    main()
