"""Utterance sharding across GPUs: no collective inside the
step -- utterances are independent (reference decoder.py:455, batch ==
sequential, test_acceptance.py:251-297) -- so every rank decodes its own
length-sorted shard and one host gather restores input order.

* ``plan_shards``: global sort by length, LPT (longest-processing-time-first)
  assignment by estimated cost ~ frames (decode steps ~ T_enc, encoder ~ T),
  then each rank's list sorted by length for tight batches.
* ``decode_corpus_sharded``: runs ``decode_fn`` on the local shard -- whole
  (``batch_size=None``: e.g. ``decode_corpus`` over the length-sorted shard,
  which batches it with a fresh fusion per batch like the reference pipeline,
  pipeline.py:148-149,210-211) or in batches -- and gathers the results to
  every rank (``torch.distributed.all_gather_object``; NCCL or gloo), returning
  them in input order.
"""

from __future__ import annotations

import heapq
from typing import Callable, List, Optional, Sequence


def plan_shards(lengths: Sequence[int], world: int) -> List[List[int]]:
    """Indices per rank; deterministic (ties broken by index)."""
    if world < 1:
        raise ValueError("world size must be positive")
    order = sorted(range(len(lengths)), key=lambda i: (-lengths[i], i))
    heap = [(0, r) for r in range(world)]
    heapq.heapify(heap)
    shards: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + int(lengths[i]), r))
    for s in shards:
        s.sort(key=lambda i: (lengths[i], i))
    return shards


def decode_corpus_sharded(features: Sequence, decode_fn: Callable,
                          batch_size: Optional[int] = None, rank: int = 0, world: int = 1,
                          group=None) -> list:
    """Decode the rank's length-sorted shard with ``decode_fn(list_of_features)
    -> results`` (the whole shard at once, or ``batch_size`` at a time); gather
    and return all results in input order."""
    lengths = [len(f.data) for f in features]
    shards = plan_shards(lengths, world)
    mine = shards[rank]
    local = []
    step = batch_size if batch_size else max(1, len(mine))
    for b in range(0, len(mine), step):
        idx = mine[b:b + step]
        res = decode_fn([features[i] for i in idx])
        if len(res) != len(idx):
            raise ValueError(f"decode_fn returned {len(res)} results for {len(idx)} utterances")
        local.extend(zip(idx, res))
    if world == 1:
        gathered = [local]
    else:
        import torch.distributed as dist
        gathered = [None] * world
        dist.all_gather_object(gathered, local, group=group)
    out = [None] * len(features)
    for part in gathered:
        for i, r in part:
            out[i] = r
    return out
