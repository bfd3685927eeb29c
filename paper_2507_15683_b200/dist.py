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
import math
import os
from typing import Callable, List, Optional, Sequence

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


def all_gather_flat(out: torch.Tensor, x: torch.Tensor, group=None):
    """out[r * n:(r + 1) * n] = rank r's x.  NCCL: all_gather_into_tensor (one
    contiguous receive buffer); gloo (CPU tests): all_gather into views of out."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, x, group=group)
    else:
        dist.all_gather(list(out.view(world, -1).unbind(0)), x, group=group)


class ChunkedGather:
    """The multi-GPU step of SURVEY.md §8(e): every rank renders its shard of the
    pose batch in chunks of `chunk` views; each chunk is rendered straight into
    its send buffer and gathered with one collective on a dedicated comm stream
    that waits only for that chunk's render, so the gather of chunk k overlaps
    the render of chunk k + 1.

    Send buffer of chunk k (one flat tensor, the render's output planes):
        [ RGB  3 x c x hw | Dz  c x hw | A  c x hw ]   (c = `chunk` views)
    i.e. the planar layout of gs_images for the chunk's views (RGB at
    3 * pix_offset, Dz / A at pix_offset) -- no packing copy, no zero fill.  A
    rank whose shard is shorter renders fewer views into its last chunk(s); the
    unused tail is never read.  Views are assigned by shard_views (LPT over
    per-view costs when given, e.g. pair counts of a projection pre-pass).
    Every rank issues the same number of equally sized collectives."""

    def __init__(self, n_views: int, hw: int, world: int, rank: int, chunk: int,
                 costs: Optional[Sequence[float]] = None, device="cpu", group=None, comm_stream=None,
                 always_gather: bool = False, payload: str = "f32"):
        self.n_views, self.hw, self.world, self.rank, self.chunk = n_views, hw, world, rank, max(1, chunk)
        # payload "f32": the fp32 RGB + Dz + A planes, rendered straight into the send buffer;
        # "dense11": the GS_PACK_DENSE11 bytes of the chunk (11 B/px, gs_pack_images, reading
        # Q39), packed into the send buffer after the render
        assert payload in ("f32", "dense11")
        self.payload = payload
        # always_gather: issue the collectives even for a one-rank group (exercises the N > 1
        # path -- collective, comm stream, events -- on one GPU)
        self.always = always_gather
        self.costs = costs
        self.group = group
        self.shards = [shard_views(n_views, world, r, costs) for r in range(world)]
        self.mine = self.shards[rank]
        self.n_chunks = max(1, math.ceil(max(len(sh) for sh in self.shards) / self.chunk))
        if payload == "f32":
            n, dt = 5 * self.chunk * hw, torch.float32
        else:
            n, dt = (11 * self.chunk * hw + 15) // 16 * 16, torch.uint8
        self.send = [torch.empty(n, dtype=dt, device=device) for _ in range(self.n_chunks)]
        self.recv = [torch.empty(world * n, dtype=dt, device=device) for _ in range(self.n_chunks)]
        self.cuda = torch.device(device).type == "cuda"
        self.comm = comm_stream if comm_stream is not None else (torch.cuda.Stream(device) if self.cuda else None)
        self.rendered = [torch.cuda.Event() for _ in range(self.n_chunks)] if self.cuda else None
        self.sent = [torch.cuda.Event() for _ in range(self.n_chunks)] if self.cuda else None
        self.steps = 0

    def chunk_views(self, k: int) -> List[int]:
        """Global indices of the views this rank renders in chunk k (may be empty)."""
        return self.mine[k * self.chunk:(k + 1) * self.chunk]

    def planes(self, k: int):
        """(rgb, depth, alpha) output planes of chunk k inside its send buffer (f32 payload)."""
        assert self.payload == "f32"
        c, hw, b = self.chunk, self.hw, self.send[k]
        return b[:3 * c * hw], b[3 * c * hw:4 * c * hw], b[4 * c * hw:5 * c * hw]

    @property
    def bytes_per_step(self) -> int:
        """Bytes each rank receives per step (all chunks, all ranks' payloads)."""
        return sum(t.numel() * t.element_size() for t in self.recv)

    def step(self, render_chunk: Callable[[int], None], stream=None, gather: bool = True):
        """render_chunk(k) enqueues chunk k's render (into planes(k)) on `stream`."""
        for k in range(self.n_chunks):
            if self.cuda and self.steps > 0 and gather:
                stream.wait_event(self.sent[k])          # the send buffer is free again
            render_chunk(k)
            if not gather or (self.world == 1 and not self.always):
                continue
            if self.cuda:
                self.rendered[k].record(stream)
                self.comm.wait_event(self.rendered[k])
                with torch.cuda.stream(self.comm):
                    all_gather_flat(self.recv[k], self.send[k], self.group)
                self.sent[k].record(self.comm)
            else:
                all_gather_flat(self.recv[k], self.send[k], self.group)
        self.steps += 1

    def wait(self, stream=None):
        """Make `stream` wait for every gather of the last step."""
        if self.cuda and (self.world > 1 or self.always):
            for e in self.sent:
                stream.wait_event(e)

    def check_own_slot(self) -> bool:
        """After a gathered step: this rank's slot of every receive buffer equals its send
        buffer bit for bit (the collective moved the rendered planes unchanged)."""
        if self.world == 1 and not self.always:
            return True
        if self.cuda:
            torch.cuda.synchronize()
        n = self.send[0].numel()
        # bit patterns (an unused tail of a short shard's buffer may hold NaN patterns)
        return all(torch.equal(self.recv[k][self.rank * n:(self.rank + 1) * n].view(torch.int32),
                               self.send[k].view(torch.int32))
                   for k in range(self.n_chunks))

    def received(self, k: int, r: int) -> torch.Tensor:
        """Rank r's payload of chunk k in this rank's receive buffer."""
        n = self.send[0].numel()
        if self.world == 1 and not self.always:
            return self.send[k]
        return self.recv[k][r * n:(r + 1) * n]

    def assemble(self) -> torch.Tensor:
        """[n_views, 5, hw] in global view order from the receive buffers (planes
        RGB, Dz, A) -- what a consumer of the gathered batch reads (f32 payload)."""
        assert self.payload == "f32"
        c, hw = self.chunk, self.hw
        out = torch.empty((self.n_views, 5, hw), dtype=torch.float32, device=self.recv[0].device)
        for k in range(self.n_chunks):
            rv = self.recv[k].view(self.world, 5 * c * hw) if self.world > 1 else self.send[k].view(1, -1)
            for r in range(self.world):
                idx = self.shards[r][k * c:(k + 1) * c]
                for j, g in enumerate(idx):
                    buf = rv[r]
                    out[g, 0:3] = buf[3 * j * hw:3 * (j + 1) * hw].view(3, hw)
                    out[g, 3] = buf[3 * c * hw + j * hw:3 * c * hw + (j + 1) * hw]
                    out[g, 4] = buf[4 * c * hw + j * hw:4 * c * hw + (j + 1) * hw]
        return out


def view_costs_from_ranges(ranges: torch.Tensor, tile_offsets: Sequence[int], tiles_per_view: Sequence[int]):
    """Per-view pair counts from a binned batch's tile ranges (lower-bound
    convention: a view's pairs are [start of its first tile, end of its last))."""
    r = ranges.view(-1, 2).to("cpu").numpy().view("uint32").astype("int64")
    out = []
    for t0, nt in zip(tile_offsets, tiles_per_view):
        out.append(float(r[t0 + nt - 1, 1] - r[t0, 0]))
    return out
