"""Multi-process (one process per GPU) merge logic, on CPU with gloo, world_size 2.

Each rank holds the aggregate of its contiguous shard; allreduce_aggregate
must reproduce the single-process report on every rank."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shards, q):
    import torch.distributed as dist

    from paper_2604_09221_b200.distributed import allreduce_aggregate

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    h, tot, k, c, w = shards[rank]
    out = allreduce_aggregate(h, tot, np.array(k, np.uint64), np.array(c, np.int64),
                              np.array(w, np.int64))
    q.put((rank, out[0], out[1], [int(x) for x in out[2]], [int(x) for x in out[3]],
           [int(x) for x in out[4]]))
    dist.destroy_process_group()


def test_gloo_world2_merge_equals_single_process():
    from paper_2604_09221_b200.distributed import merge_tables, shard

    assert shard(0, 10, 0, 3) == (0, 3) and shard(0, 10, 2, 3) == (6, 10)
    g = golden("reports.json")
    parts = [g["sweep-delaunay-3-0-40"], g["sweep-delaunay-3-40-100"]]
    extra = g["sweep-delaunay-3-100-128"]
    keymap = {}

    def table(rep):
        ks, cs, ws = [], [], []
        for s, (c, w) in rep["schemes"].items():
            keymap.setdefault(s, 1000 + len(keymap))
            ks.append(keymap[s]); cs.append(c); ws.append(w)
        return ks, cs, ws

    shards = []
    for i, rep in enumerate(parts):
        k, c, w = table(rep)
        if i == 1:  # rank 1 also carries the third range
            k2, c2, w2 = table(extra)
            k, c, w = [list(x) for x in merge_tables([(k, c, w), (k2, c2, w2)])]
            h = [a + b for a, b in zip(rep["hist"], extra["hist"])]
            tot = rep["total"] + extra["total"]
        else:
            h, tot = rep["hist"], rep["total"]
        shards.append((h, tot, k, c, w))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shards, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = g["sweep-delaunay-3-rep"]
    inv = {v: s for s, v in keymap.items()}
    for rank, hist, total, keys, counts, wits in res:
        assert hist[: len(full["hist"])] == full["hist"]
        assert total == full["total"]
        got = {inv[k]: [c, w] for k, c, w in zip(keys, counts, wits)}
        assert got == full["schemes"]


def _worker_uneven(rank, world, port, q):
    import torch.distributed as dist

    from paper_2604_09221_b200.distributed import allreduce_aggregate

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    # rank 0: 20,000 distinct keys (more than any fixed gather table used to
    # hold); rank 1: none.  Every rank must reach every collective.
    n = 20_000 if rank == 0 else 0
    keys = np.arange(n, dtype=np.uint64) * np.uint64(7) + np.uint64(5)
    out = allreduce_aggregate([n, 0], n, keys, np.ones(n, np.int64),
                              np.arange(n, dtype=np.int64) + 100)
    q.put((rank, out[0], out[1], len(out[2]), int(out[3].sum()), int(out[4].min())))
    dist.destroy_process_group()


def test_gloo_world2_uneven_tables_no_deadlock():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_uneven, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, hist, total, nkeys, csum, wmin in res:
        assert hist == [20_000, 0] and total == 20_000
        assert nkeys == 20_000 and csum == 20_000 and wmin == 100
