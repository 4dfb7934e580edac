"""A/B bitwise check of two builds of libgut (tuning experiments): renders a
fixed set of views (every camera model, the four large configs, the k-buffer,
degree-n kernels) and prints one BLAKE2b digest per output image.
    GUT_LIB=<lib.so> python tools/ab_compare.py > digests_X.txt   (on the GPU box)
then diff the two files.  A change that must not alter results (e.g. a
conservative cull) shows no difference."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def dig(*ts):
    h = hashlib.blake2b(digest_size=12)
    for t in ts:
        h.update(np.ascontiguousarray(t.detach().cpu().numpy()).tobytes())
    return h.hexdigest()


def main():
    full = "--quick" not in sys.argv
    for v in S.TINY_VARIANTS:
        for seed in range(6):
            for deg in (0, 3):
                scene, cam = S.tiny(seed, v, n=256, size=96, sh_degree=deg)
                r = gut.Renderer(scene)
                for kb in (0, 4):
                    for kd in (2, 4):
                        if kb and kd != 2:
                            continue
                        o = S.RenderOptions(kbuffer=kb, kernel_degree=kd)
                        rgb, a, d, _ = r.render(cam, o)
                        print(f"tiny {v} s{seed} d{deg} kb{kb} kd{kd}", dig(rgb, a, d), flush=True)
                r.close()
    # stress scenes: the tiny cameras with Gaussians rescaled to extremes --
    # sub-pixel dust, needles (one long axis), large flat splats near the
    # camera, opacities at alpha_min -- where conservative culls are tightest
    for v in S.TINY_VARIANTS:
        for seed in range(4):
            scene, cam = S.tiny(100 + seed, v, n=512, size=96, sh_degree=1)
            rng = np.random.default_rng(seed)
            sc = scene.scales.copy()
            kind = rng.integers(0, 4, size=len(sc))
            sc[kind == 0] *= 0.05                                        # dust
            sc[kind == 1] *= np.array([8.0, 0.05, 0.05], np.float32)     # needles
            sc[kind == 2] *= np.array([6.0, 6.0, 0.02], np.float32)      # flat splats
            op = scene.opacities.copy()
            op[kind == 3] = np.float32(1.0 / 255.0) * np.float32(1.0001)  # at alpha_min
            scene.scales = sc.astype(np.float32)
            scene.opacities = op.astype(np.float32)
            r = gut.Renderer(scene)
            for kb in (0, 4):
                rgb, a, d, _ = r.render(cam, S.RenderOptions(kbuffer=kb))
                print(f"stress {v} s{seed} kb{kb}", dig(rgb, a, d), flush=True)
            r.close()
    cfgs = [("multiview", 4 if full else 1), ("mipnerf360", 2), ("scannetpp", 2), ("waymo", 2)]
    for cfg, nv in cfgs:
        scene = S.make_scene(cfg, None if full else 200_000)
        r = gut.Renderer(scene)
        for i, cam in enumerate(S.make_views(cfg)[:nv]):
            rgb, a, d, st = r.render(cam, S.RenderOptions())
            print(f"{cfg} v{i}", dig(rgb, a, d), flush=True)
            if i == 0:
                rgb, a, d, st = r.render(cam, S.RenderOptions(kbuffer=16))
                print(f"{cfg} v{i} kb16", dig(rgb, a, d), flush=True)
        r.close()


if __name__ == "__main__":
    main()
