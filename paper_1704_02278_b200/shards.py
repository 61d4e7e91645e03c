"""Multi-GPU sharding of the PFAC path.

One process per GPU.  GPU g owns start positions [g*S, min((g+1)*S, N)) and
reads an (lmax-1)-byte halo past its end; offsets are global.  The scans are
independent (no data-path collective).  The only exchange is the final one:
per-pattern alert counts are all-reduced and the alert lists gathered to
rank 0 -- rank order concatenation is already globally sorted because owned
ranges are ascending and disjoint (the ownership rule of scan.hpp:230-232).
torch.distributed is plumbing only (NCCL on the B200 box, gloo in CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    lo: int       # first owned start (global offset)
    own: int      # owned start positions
    read: int     # bytes read: own + halo, clipped to the text end

    @property
    def hi(self) -> int:
        return self.lo + self.own


def plan_shards(total: int, world: int, halo: int) -> list[Shard]:
    """Contiguous equal shards (the first total % world get one extra byte),
    mirroring detail::parallel_ranges (scan.hpp:59-79)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    per, extra = divmod(total, world)
    out, lo = [], 0
    for r in range(world):
        own = per + (1 if r < extra else 0)
        read = min(own + halo, total - lo)
        out.append(Shard(r, lo, own, read))
        lo += own
    return out


def reduce_counts(counts, group=None):
    """All-reduce per-pattern alert counts (sum) in place; torch tensor."""
    import torch.distributed as dist

    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def gather_alerts(alerts, n: int, group=None):
    """Gather each rank's first n alert records (a 2-D uint8/int64 torch
    tensor, one row per alert) to every rank, concatenated in rank order.
    Returns the concatenation (rows) on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cnt = torch.tensor([n], dtype=torch.int64, device=alerts.device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    m = max(sizes) if sizes else 0
    pad = torch.zeros((max(m, 1),) + tuple(alerts.shape[1:]), dtype=alerts.dtype, device=alerts.device)
    if n:
        pad[:n] = alerts[:n]
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)


def gather_alerts_to_root(alerts, n: int, root: int = 0, group=None):
    """Gather each rank's first n alert rows (a 2-D torch tensor, one row per
    alert) to `root` only, concatenated in rank order (already globally
    sorted: owned ranges are ascending and disjoint).  One all_gather of the
    row counts, then point-to-point sends to the root (NCCL send/recv over
    NVLink on the B200 box; gloo in the CPU tests).  Returns the
    concatenation on the root and None elsewhere.  `root` is a rank of `group`
    (the default group: a global rank)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if alerts.is_cuda and dist.get_backend(group) == "gloo":  # gloo p2p moves host memory only
        out = gather_alerts_to_root(alerts[:n].cpu(), n, root, group)
        return None if out is None else out.to(alerts.device)
    cnt = torch.tensor([n], dtype=torch.int64, device=alerts.device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]

    def glob(r):  # send/recv address GLOBAL ranks; `root` and the loop index are group ranks
        return r if group is None else dist.get_global_rank(group, r)

    if rank != root:
        if n:
            dist.send(alerts[:n].contiguous(), dst=glob(root), group=group)
        return None
    parts = []
    for r, sz in enumerate(sizes):
        if r == root:
            parts.append(alerts[:n])
        elif sz:
            buf = torch.empty((sz,) + tuple(alerts.shape[1:]), dtype=alerts.dtype, device=alerts.device)
            dist.recv(buf, src=glob(r), group=group)
            parts.append(buf)
    return torch.cat(parts, dim=0) if parts else alerts[:0]


def merge_host(parts: list[np.ndarray]) -> np.ndarray:
    """Rank-order concatenation (globally sorted by construction)."""
    return np.concatenate(parts) if parts else np.zeros(0)
