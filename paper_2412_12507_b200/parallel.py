"""View data-parallelism: the scene is replicated on every GPU,
views are sharded round-robin over ranks, and NCCL (through torch.distributed)
is used only to broadcast the scene once and to gather per-view statistics
after the timed window.  There is no collective in the data path: views are
independent (PAPER L290 defines FPS per single image) and compositing is
order dependent, so sharding the Gaussians would need a per-pixel ordered
merge across GPUs — not done.

Every function here also works with the gloo backend on CPU tensors (tests).
"""
from __future__ import annotations

import os
from typing import Dict, List, Sequence

import torch
import torch.distributed as dist


def env_rank_world():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def init(backend: str = "nccl"):
    """Initialises the default process group from the torchrun environment."""
    rank, local, world = env_rank_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {}
        if backend == "nccl":
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend=backend, rank=rank, world_size=world, **kw)
    return rank, local, world


def view_of(step: int, rank: int, world: int, n_views: int) -> int:
    """Round-robin assignment: step s on rank r renders view (s * world + r) mod n_views,
    so each step every rank renders a distinct view (weak scaling in views)."""
    return (step * world + rank) % n_views


def views_of_rank(steps: int, rank: int, world: int, n_views: int, first_step: int = 0) -> List[int]:
    return [view_of(s, rank, world, n_views) for s in range(first_step, first_step + steps)]


def broadcast_scene(tensors: Dict[str, torch.Tensor], src: int = 0) -> Dict[str, torch.Tensor]:
    """In-place broadcast of the packed scene arrays from `src` (NCCL over
    NVLink on GPUs, gloo on CPU).  Non-source ranks pass empty tensors of the
    right shape/dtype."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        gloo = dist.get_backend() == "gloo"
        for k in sorted(tensors):
            t = tensors[k]
            if gloo and t.is_cuda:  # (gloo: through host memory)
                h = t.cpu()
                dist.broadcast(h, src=src)
                t.copy_(h)
            else:
                dist.broadcast(t, src=src)
    return tensors


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over ranks (device-timed step times are reduced this way)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_stats(rows: Sequence[Sequence[float]], device=None) -> List[List[float]]:
    """All-gather fixed-width per-view statistic rows (after the timed window)."""
    t = torch.tensor([list(map(float, r)) for r in rows], dtype=torch.float64, device=device)
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return t.tolist()
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    width = t.shape[1] if t.ndim == 2 and t.shape[0] else 0
    m = int(max(s.item() for s in sizes))
    wt = torch.tensor([width], dtype=torch.int64, device=device)
    dist.all_reduce(wt, op=dist.ReduceOp.MAX)
    width = int(wt.item())
    pad = torch.zeros((m, width), dtype=torch.float64, device=device)
    if t.numel():
        pad[: t.shape[0]] = t
    out = [torch.zeros_like(pad) for _ in range(dist.get_world_size())]
    dist.all_gather(out, pad)
    rows_all: List[List[float]] = []
    for s, o in zip(sizes, out):
        rows_all.extend(o[: int(s.item())].tolist())
    return rows_all


def image_checksum(t: torch.Tensor) -> int:
    """48-bit digest (BLAKE2b) of the tensor's bytes, hashed on the host (no
    device kernels): exact in the float64 stats rows that gather_stats carries.
    Equal images <=> equal checksums (up to collisions)."""
    import hashlib
    b = t.detach().contiguous().cpu().numpy().tobytes()
    return int.from_bytes(hashlib.blake2b(b, digest_size=6).digest(), "little")


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
