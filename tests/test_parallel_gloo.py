"""Host logic of the N>1 path on CPU: world_size 2 over gloo — view sharding,
scene broadcast, max-over-ranks timing reduction and the stats gather."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_12507_b200 import parallel as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), LOCAL_RANK=str(rank),
                      WORLD_SIZE=str(world))
    P.init(backend="gloo")
    # scene broadcast: rank 0 holds the data, the others receive into empty tensors
    shapes = {"means": (37, 3), "rotations": (37, 4), "scales": (37, 3), "opacities": (37,), "sh": (37, 16, 3)}
    g = torch.Generator().manual_seed(123)
    ref = {k: torch.rand(s, generator=g) for k, s in shapes.items()}
    t = {k: (v.clone() if rank == 0 else torch.zeros_like(v)) for k, v in ref.items()}
    P.broadcast_scene(t)
    ok_bcast = all(torch.equal(t[k], ref[k]) for k in ref)
    # timing reduction = max over ranks
    mx = P.max_over_ranks(10.0 + rank)
    # stats gather with uneven row counts
    rows = [[rank, i, 3.5] for i in range(rank + 1)]
    allrows = P.gather_stats(rows)
    P.barrier()
    q.put((rank, ok_bcast, mx, allrows))
    dist.destroy_process_group()


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, mx, rows in res:
        assert ok
        assert mx == 11.0
        assert rows == [[0.0, 0.0, 3.5], [1.0, 0.0, 3.5], [1.0, 1.0, 3.5]]


def test_view_sharding_partitions_steps():
    world, n_views, steps = 4, 256, 64
    seen = []
    for s in range(steps):
        vs = [P.view_of(s, r, world, n_views) for r in range(world)]
        assert len(set(vs)) == world  # distinct views per step
        seen.extend(vs)
    assert sorted(seen) == list(range(256))  # every view exactly once over 64 steps x 4 ranks
    for world in (1, 2, 4, 8):
        allv = sorted(v for r in range(world) for v in P.views_of_rank(256 // world, r, world, 256))
        assert allv == list(range(256))
