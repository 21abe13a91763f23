"""Utterance sharding across GPUs (one process per GPU).

Utterances are independent -- batch invariance is a tested property of the
reference (test_decoders.cpp:197-216) and of this decoder -- so the path
shards with no collective inside the decode: each rank decodes its own
utterances, and results are gathered once at the end (host-side, outside any
timed region).  Length balancing: longest-processing-time-first -- utterances
in descending length each go to the rank with the fewest frames so far -- so
every rank gets a similar number of frames.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def shard_indices(lengths: Sequence[int], world: int, rank: int) -> np.ndarray:
    """Indices of the utterances rank `rank` decodes (length-balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    import heapq
    lens = np.asarray(lengths, np.int64)
    order = np.argsort(-lens, kind="stable")
    heap = [(0, r) for r in range(world)]
    mine = []
    for i in order:
        load, r = heapq.heappop(heap)
        if r == rank:
            mine.append(i)
        heapq.heappush(heap, (load + int(lens[i]), r))
    return np.sort(np.asarray(mine, np.int64))


def shard_bounds(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [start, end) of `total` equal-length utterances."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_results(local, indices: np.ndarray, total: int, group=None) -> List:
    """Reassemble per-stream results of every rank in global order on all
    ranks (torch.distributed all_gather_object; gloo or nccl)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    payload = (np.asarray(indices).tolist(), local)
    parts = [None] * world
    dist.all_gather_object(parts, payload, group=group)
    out = [None] * total
    for idx, streams in parts:
        for i, s in zip(idx, streams):
            out[i] = s
    if any(s is None for s in out):
        raise RuntimeError("gather_results: missing streams")
    return out
