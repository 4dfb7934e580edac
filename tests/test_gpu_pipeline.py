"""GPU: the throughput machinery around the render is result-neutral.
- gut_render_batch with frames in flight (lane contexts on their own streams)
  returns exactly what views rendered one by one return;
- a render captured as a CUDA graph (device-side look-back epochs) replays to
  the same image, also interleaved with ordinary renders;
- views sharded round-robin over ranks (parallel.views_of_rank, two contexts
  on one GPU standing in for two ranks) give the images of world size 1."""
import numpy as np
import pytest

import scenegen as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import build
    build.build()
    scene = S.make_scene("multiview", n=60_000)
    cams = [S.scaled_camera(c, 0.25) for c in S.make_views("multiview")[:6]]
    return scene, cams


def _outs(torch, cams, n=None):
    from paper_2412_12507_b200 import gut
    bufs, outs = [], []
    for c in cams[:n]:
        b = (torch.empty((c.height, c.width, 3), device="cuda"), torch.empty((c.height, c.width), device="cuda"),
             torch.empty((c.height, c.width), device="cuda"))
        bufs.append(b)
        outs.append(gut.gut_outputs(b[0].data_ptr(), b[1].data_ptr(), b[2].data_ptr(), 1, 0))
    return bufs, outs


def _one_by_one(scene, cams):
    import torch
    from paper_2412_12507_b200 import gut
    r = gut.Renderer(scene, max_wh=(cams[0].width, cams[0].height))
    ref = []
    for c in cams:
        rgb, a, d, _ = r.render(c)
        ref.append((rgb.clone(), a.clone(), d.clone()))
    torch.cuda.synchronize()
    r.close()
    return ref


@pytest.mark.parametrize("reserve,fif", [(True, 3), (False, 3), (True, 1), (True, 4)])
def test_render_batch_matches_one_by_one(setup, reserve, fif):
    import torch
    from paper_2412_12507_b200 import gut
    scene, cams = setup
    ref = _one_by_one(scene, cams)
    r = gut.Renderer(scene, reserve_keys=2_000_000 if reserve else None, max_wh=(cams[0].width, cams[0].height))
    gut.gut_context_set_frames_in_flight(r.ctx, fif)
    bufs, outs = _outs(torch, cams)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):  # twice: the second call reuses the lanes
            for b in bufs:
                for t in b:
                    t.fill_(-1.0)
            gut.gut_render_batch(r.ctx, r.scene, [gut.make_camera(c) for c in cams], gut.make_options(), outs,
                                 stream=s)
    s.synchronize()
    for (a, b) in zip(ref, bufs):
        for x, y in zip(a, b):
            assert torch.equal(x, y)
    gut.gut_check(r.ctx)
    r.close()


def test_cuda_graph_replay(setup):
    import torch
    from paper_2412_12507_b200 import gut
    scene, cams = setup
    ref = _one_by_one(scene, cams)
    r = gut.Renderer(scene, reserve_keys=2_000_000, max_wh=(cams[0].width, cams[0].height))
    cam, opt = gut.make_camera(cams[1]), gut.make_options()
    (buf,), (out,) = _outs(torch, cams[1:2])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm-up (ray table of the intrinsics, workspace)
        gut.gut_render(r.ctx, r.scene, cam, opt, out, stream=s, stats=False)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        gut.gut_render(r.ctx, r.scene, cam, opt, out, stream=s, stats=False)
    for k in range(3):
        for t in buf:
            t.fill_(-1.0)
        g.replay()
        torch.cuda.synchronize()
        for x, y in zip(ref[1], buf):
            assert torch.equal(x, y), k
        # an ordinary render of another view in between (it advances the epochs too)
        rgb, _, _, _ = r.render(cams[k + 2])
        torch.cuda.synchronize()
        assert torch.equal(rgb, ref[k + 2][0])
    gut.gut_check(r.ctx)
    r.close()


def test_view_sharding_is_bitwise_equal_across_world_sizes(setup):
    import torch
    from paper_2412_12507_b200 import gut
    from paper_2412_12507_b200 import parallel as P
    scene, cams = setup
    steps = 3
    world1 = {}
    r = gut.Renderer(scene, max_wh=(cams[0].width, cams[0].height))
    for v in P.views_of_rank(steps * 2, 0, 1, len(cams)):
        world1[v] = r.render(cams[v])[0].clone()
    r.close()
    world2 = {}
    for rank in range(2):  # two contexts standing in for two ranks
        rr = gut.Renderer(scene, max_wh=(cams[0].width, cams[0].height))
        for v in P.views_of_rank(steps, rank, 2, len(cams)):
            world2[v] = rr.render(cams[v])[0].clone()
        rr.close()
    torch.cuda.synchronize()
    assert set(world2) <= set(world1) and len(world2) == min(2 * steps, len(cams))
    for v, img in world2.items():
        assert torch.equal(img, world1[v]), v
    # per-view 8-byte checksums (what bench.py gathers across ranks) agree too
    ck = {v: P.image_checksum(img) for v, img in world2.items()}
    assert all(ck[v] == P.image_checksum(world1[v]) for v in ck)


@pytest.mark.parametrize("fif", [1, 4])
def test_render_batch_host_outputs(setup, fif):
    """Host (pinned) outputs through the batch: the copies run on each lane's
    copy stream from two alternating staging slots; every view's host image
    equals the device render, also when more views than slots are in flight."""
    import torch
    from paper_2412_12507_b200 import gut
    scene, cams = setup
    ref = _one_by_one(scene, cams)
    r = gut.Renderer(scene, reserve_keys=2_000_000, max_wh=(cams[0].width, cams[0].height))
    gut.gut_context_set_frames_in_flight(r.ctx, fif)
    hb, outs = [], []
    for c in cams:
        b = (torch.full((c.height, c.width, 3), -1.0, pin_memory=True), torch.full((c.height, c.width), -1.0, pin_memory=True),
             torch.full((c.height, c.width), -1.0, pin_memory=True))
        hb.append(b)
        outs.append(gut.gut_outputs(b[0].data_ptr(), b[1].data_ptr(), b[2].data_ptr(), 0, 0))
    s = torch.cuda.Stream()
    for _ in range(2):
        gut.gut_render_batch(r.ctx, r.scene, [gut.make_camera(c) for c in cams], gut.make_options(), outs, stream=s)
    s.synchronize()  # the call's copies are complete once the stream reaches this point
    for a, b in zip(ref, hb):
        for x, y in zip(a, b):
            assert torch.equal(x.cpu(), y)
    # an ordinary host-output render after the batch on another stream
    b0 = hb[0]
    for t in b0:
        t.fill_(-1.0)
    gut.gut_render(r.ctx, r.scene, gut.make_camera(cams[0]), gut.make_options(), outs[0])
    torch.cuda.synchronize()
    assert torch.equal(ref[0][0].cpu(), b0[0])
    r.close()


def test_render_batch_stats_timing_overflow_and_errors(setup):
    """Batch edge cases: stats (one view at a time, filled per view), timing of
    the lanes' renders, a reservation too small for the views (the overflow of
    a lane context is latched and reported by gut_check on the parent), and
    invalid frames-in-flight values."""
    import torch
    from paper_2412_12507_b200 import gut
    scene, cams = setup
    r = gut.Renderer(scene, max_wh=(cams[0].width, cams[0].height))
    bufs, outs = _outs(torch, cams)
    gc = [gut.make_camera(c) for c in cams]
    st = gut.gut_render_batch(r.ctx, r.scene, gc, gut.make_options(), outs, stats=True)
    keys = [s.n_keys for s in st]
    assert len(keys) == len(cams) and all(k > 0 for k in keys)
    gut.gut_render_batch(r.ctx, r.scene, gc, gut.make_options(timing=True), outs)
    ms, n = gut.gut_timing_read(r.ctx, reset=True)
    assert n == len(cams) and ms["total"] > 0
    with pytest.raises(gut.GutError):
        gut.gut_context_set_frames_in_flight(r.ctx, 0)
    with pytest.raises(gut.GutError):
        gut.gut_context_set_frames_in_flight(r.ctx, 9)
    r.close()
    small = gut.Renderer(scene, reserve_keys=max(keys) // 3, max_wh=(cams[0].width, cams[0].height))
    gut.gut_context_set_frames_in_flight(small.ctx, 3)
    gut.gut_render_batch(small.ctx, small.scene, gc, gut.make_options(), outs)
    with pytest.raises(gut.GutError) as e:
        gut.gut_check(small.ctx)
    assert e.value.status == 4
    gut.gut_check(small.ctx)  # (cleared on every lane)
    torch.cuda.synchronize()
    small.close()


@pytest.mark.parametrize("window,cap,x4", [(1, 1, 4), (2, 0, 8), (3, 2, 5), (1, 4, 5)])
def test_batch_scheduling_is_result_neutral(setup, window, cap, x4, monkeypatch):
    """The frames-in-flight blend schedule (speculation window, successor
    grant cap, persistent grid) changes only who computes what when: with
    short segments (most tiles split, so speculation, look-back, re-runs and
    grants all happen) a batch returns exactly the single renders' images."""
    import torch
    from paper_2412_12507_b200 import gut
    monkeypatch.setenv("GUT_BLEND_SEG", "256")
    monkeypatch.setenv("GUT_BLEND_WINDOW_BATCH", str(window))
    monkeypatch.setenv("GUT_BATCH_GRANT_CAP", str(cap))
    monkeypatch.setenv("GUT_BATCH_BLEND_X4", str(x4))
    scene, cams = setup
    ref = _one_by_one(scene, cams)
    r = gut.Renderer(scene, max_wh=(cams[0].width, cams[0].height))
    gut.gut_context_set_frames_in_flight(r.ctx, 3)
    bufs, outs = _outs(torch, cams)
    gut.gut_render_batch(r.ctx, r.scene, [gut.make_camera(c) for c in cams], gut.make_options(), outs)
    torch.cuda.synchronize()
    for (a, b) in zip(ref, bufs):
        for x, y in zip(a, b):
            assert torch.equal(x, y)
    r.close()


def test_bench_launch_configuration_full_size():
    """bench.py times gut_render_batch (4 frames in flight: window-1 blend on the
    1.25-CTA/SM grid, capacity mode) on the full 3M-Gaussian fisheye frames;
    the parity tests check single renders of those frames against the oracle.
    This ties the two: at full size the batch returns exactly the single
    renders' images (RGB, alpha, depth)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import gut
    scene = S.make_scene("multiview")
    cams = S.make_views("multiview")[:4]
    r = gut.Renderer(scene, reserve_keys=8_000_000, max_wh=(cams[0].width, cams[0].height))
    ref = []
    for c in cams:
        rgb, a, d, _ = r.render(c)
        ref.append((rgb.clone(), a.clone(), d.clone()))
    gut.gut_context_set_frames_in_flight(r.ctx, 4)
    bufs, outs = _outs(torch, cams)
    gut.gut_render_batch(r.ctx, r.scene, [gut.make_camera(c) for c in cams], gut.make_options(), outs)
    torch.cuda.synchronize()
    for (a, b) in zip(ref, bufs):
        for x, y in zip(a, b):
            assert torch.equal(x, y)
    gut.gut_check(r.ctx)
    r.close()
