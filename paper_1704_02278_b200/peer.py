"""The exchange step of the sharded path over CUDA IPC and
copy engines, one process per GPU (torchrun).

Each rank's pipeline writes its alerts and per-pattern counts into buffers
allocated by libglop (glop_peer_alloc) whose IPC handles are shared once at
start; per step the root pulls every peer's alert list (in rank order, the
concatenation already globally sorted: owned ranges are ascending and
disjoint, scan.hpp:230-232) and count vector with device-to-device copies on
its own copy stream.  Copy engines move the bytes over NVLink while the next
step's scan -- a persistent kernel on every SM -- runs; an NCCL collective
would need SMs and could only start after that kernel.  torch.distributed
(a gloo group) carries only the handles and the per-step alert counts.

Ordering: a peer reuses buffer b (double-buffered) only after the root's
copies out of it: the root records an interprocess event after them, and a
host barrier per step guarantees the peer enqueues its wait after that
record.  The counts are summed lazily (`counts()`); the data movement is what
the step times.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import glop
from .glop import _check, _lib, vp

ALERT_BYTES = 16


class PeerExchange:
    def __init__(self, ctx: "glop.Context", rank: int, world: int, k: int, cap: int, group=None, root: int = 0):
        import torch.distributed as dist

        self.ctx, self.rank, self.world, self.k, self.cap, self.root = ctx, rank, world, k, cap, root
        self.group = group
        self._dist = dist
        self.alerts, self.counts_buf, handles = [], [], []
        for _ in range(2):  # double-buffered: step i writes buffer i & 1
            for lst, nbytes in ((self.alerts, cap * ALERT_BYTES), (self.counts_buf, k * 8)):
                p, h = vp(), (C.c_ubyte * 64)()
                _check(_lib.glop_peer_alloc(ctx.h, nbytes, C.byref(p), h), "glop_peer_alloc")
                lst.append(p.value)
                handles.append(bytes(h))
        self.ev_copied, ev_handles = [], []
        if rank == root:
            for _ in range(2):
                e, h = vp(), (C.c_ubyte * 64)()
                _check(_lib.glop_peer_event(ctx.h, C.byref(e), h), "glop_peer_event")
                self.ev_copied.append(e.value)
                ev_handles.append(bytes(h))
        allh = [None] * world
        dist.all_gather_object(allh, (handles, ev_handles), group=group)
        self.peer_alerts = [[None, None] for _ in range(world)]
        self.peer_counts = [[None, None] for _ in range(world)]
        self.opened = []
        if rank == root:
            import torch

            for r in range(world):
                if r == root:
                    continue
                for b in range(2):
                    for j, dst in ((0, self.peer_alerts), (1, self.peer_counts)):
                        p = vp()
                        _check(_lib.glop_peer_open(ctx.h, allh[r][0][2 * b + j], C.byref(p)), "glop_peer_open")
                        dst[r][b] = p.value
                        self.opened.append(p.value)
            # the gathered alerts (rank order) and counts of the last exchange, per buffer
            self.gather = [torch.empty(world * cap * ALERT_BYTES, dtype=torch.uint8, device=f"cuda:{ctx.device}")
                           for _ in range(2)]
            self.gcounts = [torch.zeros(world * k, dtype=torch.int64, device=f"cuda:{ctx.device}") for _ in range(2)]
            self.comm = torch.cuda.Stream(device=ctx.device)
        else:  # the root's "copied out of your buffer b" events
            self.root_copied = []
            for b in range(2):
                e = vp()
                _check(_lib.glop_peer_event_open(ctx.h, allh[root][1][b], C.byref(e)), "glop_peer_event_open")
                self.root_copied.append(e.value)
        self.sizes = [[0] * world, [0] * world]

    def exchange(self, b: int, n_alerts: int, lib_stream: int, done_event):
        """Step whose results are in buffer b; its scan has finished on this
        rank (the caller synchronized `done_event`, a torch.cuda.Event
        recorded on the library stream after it).  The root enqueues the
        pulls on its copy stream; every rank returns once the root has
        enqueued them, and each library stream then waits (device side) for
        the root's copies before its next use of buffer b."""
        import torch

        dist = self._dist
        n = torch.tensor([n_alerts], dtype=torch.int64)
        ns = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        self.sizes[b] = [int(x.item()) for x in ns]
        if self.rank == self.root:
            comm = self.comm.cuda_stream
            self.comm.wait_event(done_event)
            off = 0
            base = self.gather[b].data_ptr()
            cbase = self.gcounts[b].data_ptr()
            for r in range(self.world):
                src = self.alerts[b] if r == self.root else self.peer_alerts[r][b]
                csrc = self.counts_buf[b] if r == self.root else self.peer_counts[r][b]
                _check(_lib.glop_peer_copy(self.ctx.h, base + off, src, self.sizes[b][r] * ALERT_BYTES, comm),
                       "glop_peer_copy")
                _check(_lib.glop_peer_copy(self.ctx.h, cbase + r * self.k * 8, csrc, self.k * 8, comm),
                       "glop_peer_copy")
                off += self.sizes[b][r] * ALERT_BYTES
            _check(_lib.glop_peer_record(self.ctx.h, self.ev_copied[b], comm), "glop_peer_record")
            # the root's own buffer b is reused by its library stream after the copies too
            _check(_lib.glop_peer_wait(self.ctx.h, lib_stream, self.ev_copied[b]), "glop_peer_wait")
        dist.barrier(group=self.group)  # the root has recorded ev_copied[b] before any peer waits on it
        if self.rank != self.root:
            _check(_lib.glop_peer_wait(self.ctx.h, lib_stream, self.root_copied[b]), "glop_peer_wait")

    def gathered(self, b: int):
        """(alerts ALERT_DTYPE in rank order, summed counts) of buffer b's last
        exchange, on the root (None elsewhere); synchronizes the copy stream."""
        if self.rank != self.root:
            return None
        self.comm.synchronize()
        tot = sum(self.sizes[b])
        a = self.gather[b][: tot * ALERT_BYTES].cpu().numpy().view(glop.ALERT_DTYPE)
        c = self.gcounts[b].view(self.world, self.k).sum(0).cpu().numpy().astype(np.uint64)
        return a, c

    def close(self):
        ctx = self.ctx
        for p in self.opened:
            _lib.glop_peer_close(ctx.h, p)
        for p in self.alerts + self.counts_buf:
            _lib.glop_peer_free(ctx.h, p)
        for e in getattr(self, "ev_copied", []) + getattr(self, "root_copied", []):
            _lib.glop_peer_event_destroy(ctx.h, e)
        self.opened, self.alerts, self.counts_buf = [], [], []
