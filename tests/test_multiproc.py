"""CPU, world_size 2 over gloo: the N>1 host path — each rank derives its own
shard walk (no data-path collective) and the end-of-run stats gather (the
only collective) returns every rank's counters in rank order."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, primary, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_16945_b200 import shard
    idx = shard.read_index(primary)
    mine = shard.slice_shard(idx, world, rank)
    stats = {"clouds": len(mine), "rank": rank, "first": int(mine[0]) if len(mine) else -1}
    gathered = shard.gather_stats(stats)
    if rank == 0:
        np.save(out, np.array([[g["clouds"], g["rank"], g["first"]] for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_walks_and_stats_gather(pcp, tmp_path):
    from paper_2603_16945_b200 import shard, synth
    schema, samples = synth.shapenet(40, n_points=16)
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=8, group_size=4)
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), primary, out), nprocs=2, join=True)
    g = np.load(out)
    idx = shard.read_index(primary)
    assert g[:, 1].tolist() == [0, 1]
    assert g[:, 0].sum() == len(idx)
    for r in range(2):
        assert g[r, 0] == len(shard.slice_shard(idx, 2, r))
