"""Data-parallel consumer of the device stage (paper §3.2,
Alg. 1): one process per GPU, each rank runs its own pipeline over its shard
of the padded strided index (the reference's shard_index, so rank d's k-th
sample of a step is global position d + k * world of that step's global
batch), computes per-sample toy gradients ON THE DEVICE from the batch's
device views, and the ranks exchange them once per step over
torch.distributed (NCCL on GPUs, gloo on CPU).  Every rank then reduces
them in ascending global sample order and applies the same update, so the
parameters do not depend on the number of devices -- the contract of the
reference's simulate_data_parallel (distributed.cpp:88-164) and
toy_gradient (:73-86), whose CPU threads + std::barrier become processes +
one all_gather per step.

The gradient math is float64 like the reference; per-cloud axis means are
reduced on the device (tree order), so parameters agree with the reference
to ~1e-12 relative rather than bit-exactly.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from ._lib import PcError, K

__all__ = ["ToyModel", "SimReport", "toy_gradient", "allreduce_mean", "axis_means_batch",
           "simulate_data_parallel", "dp_shard"]


@dataclass
class ToyModel:
    params: list
    learning_rate: float = 0.01


@dataclass
class SimReport:
    params: list
    steps: int = 0
    step_seconds: list = field(default_factory=list)
    wall_seconds: float = 0.0
    max_param_divergence: float = 0.0


def allreduce_mean(grads) -> np.ndarray:
    """allreduce_mean (distributed.cpp:29-42): elementwise mean summed in
    list (device-id) order."""
    if len(grads) == 0:
        raise PcError(K["ShapeMismatch"], "no gradients to reduce")
    dim = len(grads[0])
    acc = np.zeros(dim, np.float64)
    for g in grads:
        if len(g) != dim:
            raise PcError(K["ShapeMismatch"], "gradient length mismatch")
        acc += np.asarray(g, np.float64)
    return acc * (1.0 / len(grads))


def toy_gradient(means, params) -> np.ndarray:
    """toy_gradient (distributed.cpp:73-86) from the cloud's axis means, in
    the reference's summation order."""
    x = [float(means[j % 3]) for j in range(len(params))]
    y = 0.0
    for v in x:
        y += v
    pred = 0.0
    for j in range(len(x)):
        pred += x[j] * float(params[j])
    err = pred - y
    return np.array([err * v for v in x], np.float64)


def axis_means_batch(batch, torch):
    """Per-sample float64 axis means of the batch's 'data' field, computed on
    the device from the library's views (no host copy of the clouds)."""
    kind, ptr, nbytes, offs, uniform = batch.fields["data"]
    n = batch.n_samples
    if nbytes == 0:
        raise PcError(K["MissingField"], "'data' is not a non-empty Nx3 float32 blob")
    flat = _device_view(torch, ptr, nbytes // 4)
    out = torch.empty((n, 3), dtype=torch.float64, device=flat.device)
    if uniform:
        pts = flat.view(n, -1, 3).to(torch.float64)
        out[:] = pts.mean(dim=1)
    else:
        for k in range(n):
            a, b = int(offs[k]) // 4, int(offs[k + 1]) // 4
            out[k] = flat[a:b].view(-1, 3).to(torch.float64).mean(dim=0)
    return out


class _Cai:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _device_view(torch, ptr, n_floats):
    """A float32 tensor over library-owned device memory (valid until the
    next next_batch call)."""
    if n_floats == 0:
        return torch.empty(0, dtype=torch.float32, device="cuda")
    return torch.as_tensor(_Cai(ptr, n_floats), device="cuda")


def dp_shard(n_entries: int, world: int, rank: int) -> np.ndarray:
    """The rank's entry list: pad_for_shards + strided shard_index
    (metadata.cpp:60-74, distributed.cpp:13-27)."""
    from .shard import strided_shard
    return strided_shard(n_entries, world, rank)


def simulate_data_parallel(batches, model0: ToyModel, world: int, rank: int, group=None,
                           means_fn=None) -> SimReport:
    """The reference's DP loop over this rank's batch stream.

    ``batches`` yields this rank's per-step batches (per_device_batch samples,
    rank d's k-th sample = global position d + k*world of the step);
    ``means_fn(batch) -> [B, 3] float64 tensor`` gives the per-sample axis
    means (``axis_means_batch`` for device batches).  Per step every rank
    all-gathers the [world, B, dim] per-sample gradients, reduces them in
    ascending global order and applies the mean update."""
    import torch
    import torch.distributed as dist
    if any(not np.isfinite(p) for p in model0.params):
        raise PcError(K["ShapeMismatch"], "non-finite parameter")
    if len(model0.params) == 0:
        raise PcError(K["ShapeMismatch"], "model has no parameters")
    params = np.array(model0.params, np.float64)
    dim = len(params)
    dev = "cuda" if dist.is_initialized() and dist.get_backend(group) == "nccl" else "cpu"
    rep = SimReport(params=list(params))
    t0 = time.perf_counter()
    ts = t0
    for b in batches:
        means = means_fn(b).to("cpu").numpy()
        B = means.shape[0]
        g_local = np.stack([toy_gradient(means[k], params) for k in range(B)])  # [B, dim]
        t = torch.from_numpy(g_local).to(dev)
        if world > 1:
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t, group=group)
            g_all = torch.stack(parts).cpu().numpy()  # [world, B, dim]
        else:
            g_all = g_local[None]
        # ascending global order within the step: position d + k*world
        order = [g_all[d, k] for k in range(B) for d in range(world)]
        mean = np.zeros(dim, np.float64)
        for g in order:
            mean += g
        mean *= 1.0 / (world * B)
        params = params - model0.learning_rate * mean  # params[j] -= lr * mean[j]
        if world > 1:  # divergence check: every rank holds the same parameters
            pt = torch.from_numpy(params.copy()).to(dev)
            mx = pt.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
            mn = pt.clone()
            dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
            rep.max_param_divergence = max(rep.max_param_divergence, float((mx - mn).abs().max()))
        now = time.perf_counter()
        rep.step_seconds.append(now - ts)
        ts = now
        rep.steps += 1
    rep.params = list(params)
    rep.wall_seconds = time.perf_counter() - t0
    return rep
