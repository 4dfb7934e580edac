"""CPU oracle timing: full frames of every config, fp64, on the
host cores (OMP threads = the affinity set) and with 1 thread (a child process
with OMP_NUM_THREADS=1).  Prints one JSON line per (config, threads).
usage: python tools/oracle_timing.py [config ...]   (default: all five)
The oracle is test infrastructure; this tool only times it."""
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {"tiny": None, "mipnerf360": 0, "scannetpp": 0, "waymo": [0, 1, 2], "multiview": [0, 1]}


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def time_config(config):
    import scenegen as S
    from oracle import oracle as O
    opt = S.RenderOptions()
    if config == "tiny":
        t = 0.0
        n = 0
        for variant in S.TINY_VARIANTS:
            for seed in range(32):
                scene, cam = S.tiny(seed, variant)
                t0 = time.perf_counter()
                O.render(scene, cam, opt, ambiguity=False)
                t += time.perf_counter() - t0
                n += 1
        return {"frames": n, "s_per_frame": t / n, "what": f"32 seeds x {len(S.TINY_VARIANTS)} variants"}
    scene = S.make_scene(config)
    views = S.make_views(config)
    idx = CONFIGS[config]
    idx = idx if isinstance(idx, list) else [idx]
    tt = []
    for v in idx:
        t0 = time.perf_counter()
        O.render(scene, views[v], opt, ambiguity=False)
        tt.append(time.perf_counter() - t0)
    return {"frames": len(tt), "s_per_frame": sum(tt) / len(tt), "views": idx,
            "what": "full frames (O1-O6, every tile), no extrapolation"}


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        from oracle import oracle as O
        r = time_config(sys.argv[2])
        r.update(config=sys.argv[2], threads=O.threads())
        print(json.dumps(r), flush=True)
        return
    configs = sys.argv[1:] or list(CONFIGS)
    ncores = len(os.sched_getaffinity(0))
    for c in configs:
        for th in ([ncores, 1] if c in ("tiny", "mipnerf360") else [ncores]):
            env = dict(os.environ, OMP_NUM_THREADS=str(th))
            out = subprocess.run([sys.executable, __file__, "--child", c], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else json.dumps({"error": out.stderr[-300:]})
            d = json.loads(line)
            d["cpu"] = cpu_model()
            print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
