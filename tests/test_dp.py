"""Data-parallel consumer (paper_2603_16945_b200/dp.py)
against the compiled reference's simulate_data_parallel
(distributed.cpp:88-164): world-2 over gloo on CPU with batches read by the
reference reader, bit-exact; parameters independent of the device count."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

PARAMS = [0.1, -0.2, 0.3, 0.05, 0.5, -0.4, 0.25]
LR = 0.05
B = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Batch:
    def __init__(self, samples):
        self.samples = samples


def _means(b):
    """Reference axis_means: float coordinates summed into doubles in point
    order (cumsum is sequential), divided by the count."""
    rows = []
    for s in b.samples:
        p = s["data"].view(np.float32).reshape(-1, 3).astype(np.float64)
        rows.append(np.cumsum(p, axis=0)[-1] / len(p))
    return torch.from_numpy(np.array(rows))


def _rank_batches(primary, world, rank, epochs):
    from oracle.ffi import Ref
    from paper_2603_16945_b200.dp import dp_shard
    from paper_2603_16945_b200 import shard
    n = len(shard.read_index(primary))
    ids = dp_shard(n, world, rank)
    smp = Ref().read_samples(primary, ids)
    for _ in range(epochs):
        for k in range(0, len(smp) - len(smp) % B, B):
            yield _Batch(smp[k:k + B])


def _worker(rank, world, port, primary, epochs, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_16945_b200.dp import ToyModel, simulate_data_parallel
    rep = simulate_data_parallel(_rank_batches(primary, world, rank, epochs), ToyModel(PARAMS, LR), world,
                                 rank, means_fn=_means)
    np.save(out + f".{rank}.npy", np.array(rep.params + [rep.max_param_divergence, rep.steps]))
    dist.barrier()
    dist.destroy_process_group()


def _dataset(pcp, tmp_path, n=24):
    from paper_2603_16945_b200 import synth
    schema, samples = synth.shapenet(n, n_points=37)
    return pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=2, group_size=5)


def test_two_ranks_match_reference_simulation(pcp, ref, tmp_path):
    primary = _dataset(pcp, tmp_path)
    out = str(tmp_path / "p")
    mp.spawn(_worker, args=(2, _free_port(), primary, 2, out), nprocs=2, join=True)
    want, div = ref.simulate_dp(primary, 2, 2, B, PARAMS, LR)
    for r in range(2):
        got = np.load(out + f".{r}.npy")
        assert got[-1] == 2 * 24 // (2 * B)  # steps
        assert got[-2] == 0.0 and div == 0.0
        assert got[:-2].tolist() == want  # bit-exact


def test_parameters_do_not_depend_on_device_count(pcp, ref, tmp_path):
    from paper_2603_16945_b200.dp import ToyModel, simulate_data_parallel
    primary = _dataset(pcp, tmp_path)
    # one rank, per_device_batch 2B = the global batch of a 2-device run
    global B
    b0 = B
    try:
        B = 2 * b0
        rep = simulate_data_parallel(_rank_batches(primary, 1, 0, 1), ToyModel(PARAMS, LR), 1, 0, means_fn=_means)
    finally:
        B = b0
    two, _ = ref.simulate_dp(primary, 2, 1, b0, PARAMS, LR)
    one, _ = ref.simulate_dp(primary, 1, 1, 2 * b0, PARAMS, LR)
    assert one == two
    assert rep.params == one
