"""Multi-GPU host logic: pose sharding and the RGB+depth+opacity gather.

The hot path is embarrassingly parallel over views ("for each
viewpoint", P:280 n refinement renders): every rank holds a replica of the
(block-partitioned) scene and renders its own shard of the pose batch.  The
only exchange is the optional gather of the rendered RGB + depth + opacity
planes (BASELINE north_star: "using NCCL over NVLink only to gather rendered
depth and colour tiles"), issued with torch.distributed (NCCL on GPUs, gloo
in the CPU tests).  No arithmetic of the method happens here.
"""
from __future__ import annotations

import heapq
import os
from typing import List, Optional, Sequence

import torch
import torch.distributed as dist


def env_rank_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def shard_views(n_views: int, world: int, rank: int, costs: Optional[Sequence[float]] = None) -> List[int]:
    """Indices of the views rank `rank` renders.

    Without costs: contiguous blocks of near-equal size (views are spatially
    ordered, so neighbours share scene blocks in L2).  With costs (e.g. the
    per-view pair counts of a projection pre-pass): greedy
    longest-processing-time assignment, ties broken by view index, returned in
    ascending view order.  Every view is assigned to exactly one rank and the
    result is a pure function of (n_views, world, costs)."""
    assert world >= 1 and 0 <= rank < world
    if costs is None:
        base, rem = divmod(n_views, world)
        start = rank * base + min(rank, rem)
        return list(range(start, start + base + (1 if rank < rem else 0)))
    assert len(costs) == n_views
    order = sorted(range(n_views), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    owner = [0] * n_views
    for i in order:
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [i for i in range(n_views) if owner[i] == rank]


def shard_sizes(n_views: int, world: int, costs: Optional[Sequence[float]] = None) -> List[int]:
    return [len(shard_views(n_views, world, r, costs)) for r in range(world)]


def pack_planes(rgb: torch.Tensor, depth: torch.Tensor, alpha: torch.Tensor, n_views: int, hw: int,
                pad_views: int) -> torch.Tensor:
    """[pad_views, 5, hw] float32 payload (RGB, Dz, A per view; zero padded)."""
    out = torch.zeros((pad_views, 5, hw), dtype=torch.float32, device=rgb.device)
    if n_views:
        out[:n_views, 0:3] = rgb.view(n_views, 3, hw)
        out[:n_views, 3] = depth.view(n_views, hw)
        out[:n_views, 4] = alpha.view(n_views, hw)
    return out


def gather_planes(payload: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """all_gather_into_tensor of equally padded per-rank payloads
    -> [world * pad_views, 5, hw]."""
    if world == 1:
        return payload
    out = torch.empty((world * payload.shape[0],) + tuple(payload.shape[1:]), dtype=payload.dtype,
                      device=payload.device)
    dist.all_gather_into_tensor(out, payload.contiguous(), group=group)
    return out


def unshard(gathered: torch.Tensor, n_views: int, world: int, costs: Optional[Sequence[float]] = None) -> torch.Tensor:
    """Reorder a gathered [world * pad, 5, hw] tensor into global view order."""
    pad = gathered.shape[0] // world
    out = torch.empty((n_views,) + tuple(gathered.shape[1:]), dtype=gathered.dtype, device=gathered.device)
    for r in range(world):
        idx = shard_views(n_views, world, r, costs)
        if idx:
            out[torch.tensor(idx, device=gathered.device)] = gathered[r * pad:r * pad + len(idx)]
    return out
