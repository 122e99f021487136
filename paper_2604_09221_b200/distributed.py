"""One process per GPU: shard an enumeration, merge aggregates with collectives.

The sign-index space shards with no data-path exchange (every patchwork is
independent); the only collective is the final merge of
per-rank aggregates, the multi-process form of the reference's
``_run_chunks`` merge (sweep.py:168-180):

* ``all_reduce(SUM)`` of the int64 oval histogram plus the total;
* ``all_gather`` of fixed-capacity (key, count, witness) tables, then a
  local merge (count sum, witness min) -- identical on every rank.

With the NCCL backend the tensors live on the rank's GPU and the exchange
rides NVLink/NVSwitch (a few KB per sweep); with gloo (tests on CPU) they
stay on the host.  Shards are contiguous, so the merged report is
byte-identical for any world size.
"""

from __future__ import annotations

import numpy as np

def shard(start: int, end: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of [start, end) for ``rank`` of ``world``."""
    n = end - start
    return start + n * rank // world, start + n * (rank + 1) // world


def merge_tables(parts):
    """Merge [(keys, counts, witnesses)] by key: count sum, witness min."""
    acc: dict[int, list[int]] = {}
    for keys, counts, wits in parts:
        for k, c, w in zip(keys, counts, wits):
            k, c, w = int(k), int(c), int(w)
            if k in acc:
                acc[k][0] += c
                acc[k][1] = min(acc[k][1], w)
            else:
                acc[k] = [c, w]
    ks = sorted(acc)
    return (np.array(ks, np.uint64), np.array([acc[k][0] for k in ks], np.int64),
            np.array([acc[k][1] for k in ks], np.int64))


def allreduce_aggregate(hist, total, keys, counts, wits, group=None, device=None):
    """Merge one rank's aggregate with every other rank's; returns the global
    (hist, total, keys, counts, witnesses) on all ranks.

    Three collectives, every rank always takes part in all of them (a rank
    can never raise before the others reach a collective): all_reduce(SUM)
    of [hist..., total], all_reduce(MAX) of the table size, all_gather of
    the (key, count, witness) tables padded to that size."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return list(hist), int(total), keys, counts, wits
    dev = device if device is not None else torch.device("cpu")
    n = len(keys)
    h = torch.tensor(list(hist) + [int(total)], dtype=torch.int64, device=dev)
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    width = torch.tensor([n], dtype=torch.int64, device=dev)
    dist.all_reduce(width, op=dist.ReduceOp.MAX, group=group)
    cap = max(1, int(width.item()))
    tab = torch.zeros((3, cap + 1), dtype=torch.int64, device=dev)
    tab[0, 0] = n
    if n:
        tab[0, 1:n + 1] = torch.from_numpy(np.asarray(keys, np.uint64).view(np.int64))
        tab[1, 1:n + 1] = torch.from_numpy(np.asarray(counts, np.int64))
        tab[2, 1:n + 1] = torch.from_numpy(np.asarray(wits, np.int64))
    out = torch.zeros(world * 3 * (cap + 1), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, tab.reshape(-1), group=group)
    out = out.cpu().numpy().reshape(world, 3, cap + 1)
    parts = []
    for r in range(world):
        m = int(out[r, 0, 0])
        parts.append((out[r, 0, 1:m + 1].view(np.uint64), out[r, 1, 1:m + 1],
                      out[r, 2, 1:m + 1]))
    k, c, w = merge_tables(parts)
    hh = h.cpu().numpy()
    return [int(x) for x in hh[:-1]], int(hh[-1]), k, c, w


def sweep_sharded(T, start: int, end: int, raw_space: bool = False, classifier=None,
                  group=None):
    """Each rank sweeps its contiguous shard on its own GPU; all ranks return
    the merged SweepReport (identical to a single-GPU ``sweep``)."""
    import torch
    import torch.distributed as dist

    from .classify import Classifier
    from .sweep import _raise_status, report_from_agg

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard(start, end, rank, world)
    c = classifier or Classifier(T, device=torch.cuda.current_device())
    rc, bad, agg = c.native.sweep(raw_space, lo, hi)
    status = torch.tensor([rc, bad if rc else -1], dtype=torch.int64,
                          device=torch.device("cuda", c.device)
                          if dist.get_backend(group) == "nccl" else "cpu")
    hist, total, keys, counts, wits = agg.result()
    dev = status.device
    stats = [torch.zeros_like(status) for _ in range(world)]
    dist.all_gather(stats, status, group=group)
    fails = [(int(s[1]), int(s[0])) for s in stats if int(s[0]) != 0]
    if fails:
        bad, rc = min(fails)
        _raise_status(rc, bad)
    hist, total, keys, counts, wits = allreduce_aggregate(hist, total, keys, counts, wits,
                                                          group, dev)
    params = {"mode": "sweep", "start": start, "end": end, "raw_space": raw_space}
    return report_from_agg(T, raw_space, hist, total, keys, counts, wits, params)
