"""Renders one multiview view `reps` times (profiling driver: ncu -k ... -s N -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def main():
    view = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    config = os.environ.get("TRACE_CONFIG", "multiview")
    scene = S.make_scene(config)
    cam = S.make_views(config)[view]
    r = gut.Renderer(scene)
    opt = S.RenderOptions(kbuffer=int(os.environ.get("KBUF", "0")))
    for _ in range(reps):
        _, _, _, st = r.render(cam, opt, timing=True)
    print("ms_stage", [round(x, 3) for x in st.ms_stage])
    r.close()


if __name__ == "__main__":
    main()
