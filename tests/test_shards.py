"""Multi-GPU sharding host logic on CPU: contiguous shards with
an (lmax-1)-byte halo, start ownership (scan.hpp:230-232), global offsets,
then the final exchange -- per-pattern count all-reduce and rank-order alert
gather -- over a world-size-2 gloo group.  The per-shard matcher here is the
oracle (the checker); the GPU version of the same sharded scan is
test_gpu_parity.py::test_shards_with_halo_equal_whole."""
import os
import socket

import numpy as np
import pytest

import oracle_ffi as O
from paper_1704_02278_b200 import glop
from paper_1704_02278_b200.shards import merge_host, plan_shards


def _text_and_rules(n=200_000, k=40, seed=5):
    text = glop.gen_syslog_host(n, seed=seed)
    pats, _ = glop.gen_rules(k, seed=seed + 1)
    return text, pats


def shard_scan(text, pats, L, sh):
    """Oracle PFAC over text[lo, lo+read), keeping starts < own, global offsets."""
    part = text[sh.lo: sh.lo + sh.read]
    hits = O.pfac_scan(part, O.Trie(pats, L)) if part.size else np.zeros(0, dtype=glop.HIT_DTYPE)
    hits = hits[hits["offset"] < sh.own].copy()
    hits["offset"] += sh.lo
    return hits


@pytest.mark.parametrize("total,world,halo", [(0, 2, 7), (1, 4, 7), (10, 3, 7), (1001, 8, 7), (17, 2, 30)])
def test_plan_shards_cover_and_clip(total, world, halo):
    sh = plan_shards(total, world, halo)
    assert len(sh) == world
    assert sum(s.own for s in sh) == total
    lo = 0
    for s in sh:  # contiguous, ascending, first total % world get one extra
        assert s.lo == lo and s.own in (total // world, total // world + 1)
        assert s.read == min(s.own + halo, total - s.lo)
        lo += s.own
    with pytest.raises(ValueError):
        plan_shards(10, 0, 7)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_oracle_equals_whole(world):
    text, pats = _text_and_rules()
    L = 8
    whole = O.pfac_scan(text, O.Trie(pats, L))
    halo = max(len(p) for p in pats) - 1
    parts = [shard_scan(text, pats, L, s) for s in plan_shards(text.size, world, halo)]
    got = merge_host(parts) if parts else whole[:0]
    assert got.tobytes() == whole.tobytes()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1704_02278_b200.shards import gather_alerts, gather_alerts_to_root, reduce_counts

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        text, pats = _text_and_rules()
        L = 8
        halo = max(len(p) for p in pats) - 1
        sh = plan_shards(text.size, world, halo)[rank]
        hits = shard_scan(text, pats, L, sh)
        counts = torch.from_numpy(np.bincount(hits["pattern_id"], minlength=len(pats)).astype(np.int64))
        reduce_counts(counts)
        rows = torch.from_numpy(hits.view(np.uint8).reshape(-1, 16).copy())
        allrows = gather_alerts(rows, len(hits))
        root = gather_alerts_to_root(rows, len(hits), root=0)
        assert (root is None) == (rank != 0)
        if root is not None:
            assert root.numpy().tobytes() == allrows.numpy().tobytes()
        q.put((rank, counts.numpy().tobytes(), allrows.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reduce_and_gather():
    import torch.multiprocessing as mp

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    text, pats = _text_and_rules()
    whole = O.pfac_scan(text, O.Trie(pats, 8))
    want_counts = np.bincount(whole["pattern_id"], minlength=len(pats)).astype(np.int64)
    assert whole.size > 0
    for _, counts, rows in res:
        assert np.frombuffer(counts, np.int64).tolist() == want_counts.tolist()
        assert rows == whole.tobytes()  # rank-order concatenation is globally sorted


def test_plan_shards_c_abi_matches_python():
    """glop_plan_shards (the C ABI's shard plan, host only) == shards.plan_shards."""
    from paper_1704_02278_b200 import glop

    for n, world, halo in [(10, 3, 7), (8_000_000_000, 8, 7), (0, 2, 7), (5, 8, 23), (1 << 40, 7, 14)]:
        c = glop.plan_shards_c(n, world, halo)
        py = [(s.lo, s.own, s.read) for s in plan_shards(n, world, halo)]
        assert c == py, (n, world, halo)


def _subgroup_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1704_02278_b200.shards import gather_alerts_to_root

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sub = dist.new_group([1, 2])  # group ranks 0, 1 = global ranks 1, 2
        if rank in (1, 2):
            rows = torch.full((rank, 16), rank, dtype=torch.uint8)
            out = gather_alerts_to_root(rows, rank, root=0, group=sub)  # root: group rank 0 = global rank 1
            q.put((rank, None if out is None else out.numpy().tobytes()))
        else:
            q.put((rank, None))
    finally:
        dist.destroy_process_group()


def test_gloo_gather_to_root_in_a_subgroup():
    """with a non-default group, send/recv must address global
    ranks: root = group rank 0 (global 1) receives group rank 1's rows."""
    import torch.multiprocessing as mp

    world, port = 3, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_subgroup_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] is None and res[2] is None
    assert res[1] == bytes([1] * 16 + [2] * 32)
