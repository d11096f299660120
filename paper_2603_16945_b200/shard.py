"""Record sharding across GPUs.

Each GPU runs an independent pipeline over its own entry walk; there is no
collective on the hot path.  Two partition rules are provided:

* ``slice_shard``  — B200 default: GPU k of g takes the slices {k, k+g, ...}
  (``MetadataEntry.shard_id`` = slice, metadata.cpp:40), so every page is
  decoded by exactly one GPU (no decode amplification).
* ``strided_shard`` — the reference's rule: ``pad_for_shards`` (cyclic
  duplicates of the trailing entries, metadata.cpp:60-74) then entry i goes
  to shard i mod g (distributed.cpp:13-27).  Kept for drop-in parity.

The walk of a shard is the seed-index space of its pipeline, exactly like
``Pipeline(graph, src, shard.size())`` in streaming.cpp:357.
"""
from __future__ import annotations

import json
import os
import struct

import numpy as np


def read_index(primary: str) -> list:
    """(slice, group_id, row) per entry in build_index order (metadata.cpp:20-52),
    parsed from the PcRecord header JSON without touching any page."""
    with open(primary, "rb") as f:
        if f.read(4) != b"PCRC":
            raise ValueError("not a .pcrecord file")
        f.read(2)
        (n,) = struct.unpack("<I", f.read(4))
        h = json.loads(f.read(n))
    groups = sorted(h["group_index"], key=lambda g: g["first_sample"])
    out = []
    for g in groups:
        for r in range(g["sample_count"]):
            out.append((g["slice"], g["group_id"], r))
    return out


def slice_shard(index: list, world: int, rank: int) -> np.ndarray:
    """Entry ids of GPU `rank`: all entries whose slice % world == rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must lie in [0, world)")
    return np.array([i for i, e in enumerate(index) if e[0] % world == rank], dtype=np.uint64)


def pad_for_shards(n: int, world: int) -> np.ndarray:
    """pad_for_shards (metadata.cpp:60-74) on entry ids 0..n-1."""
    if world < 1:
        raise ValueError("num_shards must be >= 1")
    if n == 0:
        return np.zeros(0, np.uint64)
    target = (n + world - 1) // world * world
    ids = list(range(n))
    for i in range(n, target):
        ids.append(n - (target - i - 1) % n - 1)
    return np.array(ids, dtype=np.uint64)


def strided_shard(n: int, world: int, rank: int) -> np.ndarray:
    """shard_index(pad_for_shards(index), {world, rank}) (distributed.cpp:13-27)."""
    if world == 0 or not 0 <= rank < world:
        raise ValueError("shard_id must lie in [0, num_shards)")
    return pad_for_shards(n, world)[rank::world]


def gather_stats(stats: dict, group=None) -> list:
    """End-of-run stats gather (the only collective; off the hot path).
    Uses torch.distributed when initialised (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return [stats]
    keys = sorted(stats)
    t = torch.tensor([float(stats[k]) for k in keys], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    parts = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return [{k: float(v) for k, v in zip(keys, p.cpu().tolist())} for p in parts]


def env_rank() -> tuple:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
