"""Diagnostics: K5 work-item timeline (needs GUT_BLEND_TRACE=1; run on the GPU box).

For each view: kernel span, concurrency over time, the sum of item durations
(the ideal span if the items were perfectly packed at the observed
concurrency) and the items that form the tail."""
import os
import sys

os.environ.setdefault("GUT_BLEND_TRACE", "1")
import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2412_12507_b200 import gut  # noqa: E402


def analyse(tr, ranges, tx, seg, label):
    used = tr[:, 3] != 0
    tr = tr[used].astype(np.int64)
    proc, nev, ncon, nredo = tr[:, 4], tr[:, 5], tr[:, 6], tr[:, 7] & 1
    nalive = tr[:, 7] >> 1
    tile, s = tr[:, 0] & 0xFFFF, (tr[:, 0] >> 16) & 0x1FFF
    t0 = tr[:, 2].min()
    b, e = tr[:, 2] - t0, tr[:, 3] - t0
    span = e.max()
    dur = e - b
    ev = np.concatenate([np.stack([b, np.ones_like(b)], 1), np.stack([e, -np.ones_like(e)], 1)])
    ev = ev[np.lexsort((ev[:, 1], ev[:, 0]))]
    conc = np.cumsum(ev[:, 1])
    peak = conc.max()
    # concurrency profile in 10 slices of the span
    prof = []
    for q in range(10):
        lo, hi = span * q / 10, span * (q + 1) / 10
        ov = np.clip(np.minimum(e, hi) - np.maximum(b, lo), 0, None).sum()
        prof.append(ov / (hi - lo))
    print(f"{label}: units {len(tr)} span {span / 1e3:.1f} us, peak concurrency {peak} warps, "
          f"sum dur {dur.sum() / 1e3:.0f} us -> packed span {dur.sum() / peak / 1e3:.1f} us")
    print("  mean concurrency per 10% slice:", " ".join(f"{p:.0f}" for p in prof))
    print("  item dur pct 50/90/99/max [us]:", (np.percentile(dur, [50, 90, 99]) / 1e3).round(1), dur.max() / 1e3)
    tsp = (tr[:, 1] & 0xFFFF) * 16
    tlb = (tr[:, 1] >> 16) * 16
    for lab, sel in (("s=0", s == 0), ("s>0", s > 0)):
        if sel.any():
            print(f"  {lab}: spec pass {tsp[sel].sum() / 1e3:.0f} us, look-back wait {(tlb - tsp)[sel].sum() / 1e3:.0f} us, "
                  f"redo+outputs {(dur - tlb)[sel].sum() / 1e3:.0f} us (warp-time)")
    sp = s > 0
    if sp.any():
        dead = sp & (nalive == 0)
        print(f"  s>0 items with no pixel alive at their start (pure speculation waste): {dead.sum()} of {sp.sum()}, "
              f"warp-time {dur[dead].sum() / 1e3:.0f} of {dur[sp].sum() / 1e3:.0f} us, visited {proc[dead].sum()}")
        L0 = (ranges[:, 1] - ranges[:, 0]).astype(np.int64)
        for lab, sel in (("wasted", dead), ("useful", sp & ~dead)):
            if sel.any():
                ll = L0[tile[sel]]
                print(f"    {lab} s>0: tile len pct 10/50/90 {np.percentile(ll, [10, 50, 90]).astype(int)}, "
                      f"s values {np.bincount(s[sel])[:8]}")
    print(f"  totals: warp-entries visited {proc.sum()} pairs eval {nev.sum()} contrib {ncon.sum()} "
          f"redo warps {nredo.sum()};  ns per warp-entry {dur.sum() / max(proc.sum(), 1):.1f} (warp-time)")
    s0 = s == 0
    print(f"  s=0 items: {s0.sum()} dur {dur[s0].sum() / 1e3:.0f} us visited {proc[s0].sum()} eval {nev[s0].sum()}; "
          f"s>0 items: {(~s0).sum()} dur {dur[~s0].sum() / 1e3:.0f} us visited {proc[~s0].sum()} eval {nev[~s0].sum()} "
          f"contrib {ncon[~s0].sum()}")
    L = (ranges[:, 1] - ranges[:, 0]).astype(np.int64)
    last = np.argsort(-e)[:10]
    for i in last:
        t = tile[i]
        print(f"    tile ({t % tx},{t // tx}) s {s[i]} len {L[t]} start {b[i] / 1e3:.1f} end {e[i] / 1e3:.1f} "
              f"dur {dur[i] / 1e3:.1f} spec {tsp[i] / 1e3:.1f} lb {tlb[i] / 1e3:.1f} visited {proc[i]} eval {nev[i]} contrib {ncon[i]} redo {nredo[i]}")
    longest = np.argsort(-dur)[:5]
    for i in longest:
        t = tile[i]
        print(f"    longest: tile ({t % tx},{t // tx}) s {s[i]} len {L[t]} start {b[i] / 1e3:.1f} dur {dur[i] / 1e3:.1f} spec {tsp[i] / 1e3:.1f} lb {tlb[i] / 1e3:.1f} "
              f"visited {proc[i]} eval {nev[i]} contrib {ncon[i]} redo {nredo[i]}")
    # late starters: items whose ticket started after 80% of the span
    late = b > 0.8 * span
    print(f"  items starting after 80% of span: {late.sum()} (their mean dur {dur[late].mean() / 1e3 if late.any() else 0:.1f} us)")


def main():
    config = os.environ.get("TRACE_CONFIG", "multiview")
    views = [int(v) for v in (sys.argv[1:] or ["0", "1", "2", "3"])]
    scene = S.make_scene(config)
    cams = S.make_views(config)
    r = gut.Renderer(scene)
    for v in views:
        cam = cams[v]
        for _ in range(2):
            _, _, _, st = r.render(cam, timing=True)
        tr = r.stage(gut.STAGE_BLEND_TRACE)
        ranges = r.stage(gut.STAGE_RANGES)
        ms = list(st.ms_stage)
        analyse(tr, ranges, cam.tiles[0], int(os.environ.get("GUT_BLEND_SEG", "2560")),  # (library default)
                f"view {v} (blend {ms[5]:.3f} ms, K={st.n_keys})")
    r.close()


if __name__ == "__main__":
    main()
