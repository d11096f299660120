"""Expected outputs for parity tests, built ONLY from the oracles.

* reference ops without extension params run in the compiled reference
  (``Ref.apply_map`` / ``Ref.run_pipeline``);
* App. C ops (fps / voxel / range_crop) and the ``gather`` extension run in
  the C restatement (``Orc.apply_map``), which tests/test_oracle.py pins
  against the reference on every reference op.
"""
from __future__ import annotations

import json

import numpy as np

REF_OPS = {"normalize", "translate", "jitter", "rotate", "random_scale", "flip_yz",
           "color_augment", "random_crop", "downsample"}
TOLERANT = {"jitter", "rotate"}  # glibc cosf/sinf/logf vs CUDA: ulp-level


def map_steps(graph: dict):
    """Expand (possibly fused) map nodes → [(kind, params, seed_op_id)]."""
    steps = []
    for o in graph["ops"]:
        if o["kind"] != "map":
            continue
        if "fused" in o:
            steps += [(f["map"], f.get("params", {}), f["op_id"]) for f in o["fused"]]
        else:
            steps.append((o["map"], o.get("params", {}), o["id"]))
    return steps


def batch_size(graph: dict) -> int:
    return next(o.get("batch_size", 1) for o in graph["ops"] if o["kind"] == "batch")


def expected_run(ref, orc, primary, graph: dict, ids=None, epochs: int = 1):
    """Reference semantics of Pipeline + dataset_source over the walk `ids`."""
    steps = map_steps(graph)
    pure_ref = all(k in REF_OPS and "gather" not in p for k, p, _ in steps)
    if pure_ref:
        return ref.run_pipeline(primary, json.dumps(graph), ids=ids, epochs=epochs)
    index = ref.index(primary)["entries"]
    walk = list(range(len(index))) if ids is None else list(ids)
    raw = ref.read_samples(primary, walk)
    B = batch_size(graph)
    base = graph.get("base_seed", 0)
    drop = graph.get("drop_remainder", True)
    out = []
    for e in range(epochs):
        samples = []
        for k, s in enumerate(raw):
            for kind, params, op_id in steps:
                seed = ref.mix_seed(base, e, k, op_id)
                if kind in REF_OPS and "gather" not in params:
                    s = ref.apply_map(kind, params, s, seed)
                else:
                    s = orc.apply_map(kind, params, s, seed)
            samples.append(s)
        nb = len(samples) // B if drop else -(-len(samples) // B)
        for b in range(nb):
            out.append({"epoch": e, "batch_index": b, "samples": samples[b * B:(b + 1) * B]})
    return out


def tolerant_fields(graph: dict) -> set:
    kinds = {k for k, _, _ in map_steps(graph)}
    f = set()
    if kinds & TOLERANT:
        f |= {"data", "normal"}
    return f


def assert_batches_equal(got: list, want: list, float_fields=(), rtol=1e-5, atol=1e-6):
    assert len(got) == len(want), f"batch count {len(got)} != {len(want)}"
    for bg, bw in zip(got, want):
        assert bg["epoch"] == bw["epoch"] and bg["batch_index"] == bw["batch_index"]
        assert len(bg["samples"]) == len(bw["samples"])
        for k, (sg, sw) in enumerate(zip(bg["samples"], bw["samples"])):
            assert sorted(sg) == sorted(sw), (sorted(sg), sorted(sw))
            for name in sw:
                a, b = sg[name], sw[name]
                if isinstance(b, str):
                    assert a == b
                    continue
                a = np.asarray(a).view(np.uint8)
                b = np.asarray(b).view(np.uint8)
                assert a.size == b.size, (bw["batch_index"], k, name, a.size, b.size)
                if name in float_fields:
                    # rotate/jitter use cosf/sinf/logf, whose last ulp differs
                    # between glibc and CUDA: |a-b| <= rtol*|b| + atol*scale,
                    # scale = the cloud's largest |coordinate| (x*c - y*s can
                    # cancel to ~0 while carrying ulp error of |x|, |y|)
                    fa, fb = a.view(np.float32), b.view(np.float32)
                    scale = max(1.0, float(np.abs(fb).max())) if fb.size else 1.0
                    np.testing.assert_allclose(fa, fb, rtol=rtol, atol=atol * scale,
                                               err_msg=f"batch {bw['batch_index']} sample {k} {name}")
                else:
                    if not np.array_equal(a, b):
                        bad = np.flatnonzero(a != b)
                        raise AssertionError(
                            f"batch {bw['batch_index']} sample {k} field {name}: "
                            f"{bad.size} bytes differ, first at {bad[0]}")
