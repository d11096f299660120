"""CPU: the C-ABI library loads and exports exactly what include/ declares,
host-side logic (writer, graph/options, sharding) matches the reference, and
compute entry points fail loudly (no CPU fallback) without a GPU."""
import filecmp
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "pcpipe_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pcp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(pcp):
    L = pcp.lib()
    names = _declared_functions()
    assert len(names) >= 19
    for n in names:
        assert hasattr(L, n), n
    # and the built .so really contains sm_100a code
    so = open(os.path.join(ROOT, "paper_2603_16945_b200", "libpcpipe_b200.so"), "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so


def test_status_codes_are_errc_plus_one(pcp):
    L = pcp.lib()
    for i, name in enumerate(pcp.ERRC):
        assert L.pcp_errc_name(i).decode() == name
    assert pcp.ERRC[28] == "WorkerPanic" and pcp.ERRC[6] == "ChecksumMismatch"


def test_mix_seed_and_kinds(pcp, ref):
    for args in [(0, 0, 0, 0), (42, 1, 2, 3), (2**64 - 1, 5, 2**40, 7)]:
        assert pcp.mix_seed(*args) == ref.mix_seed(*args)
    assert pcp.map_kind_from_name("downsample") == 8
    assert pcp.map_kind_from_name("fps") == 16
    with pytest.raises(pcp.PcError) as e:
        pcp.map_kind_from_name("blur")
    assert e.value.errc == "UnknownOp"


@pytest.mark.parametrize("gen,kw,G,slices", [
    ("shapenet", {"n_points": 300}, 8, 3),
    ("shapenet", {"n_points": 300, "quantized": True}, 5, 2),
    ("kitti", {"lo": 500, "hi": 900, "quantized": True}, 4, 1),
    ("modelnet", {"n_points": 200}, 64, 4),
])
def test_writer_is_byte_identical_to_reference(pcp, ref, tmp_path, gen, kw, G, slices):
    from paper_2603_16945_b200 import synth
    schema, samples = getattr(synth, gen)(19, **kw)
    a, b = tmp_path / "ref", tmp_path / "ours"
    ref.write_dataset(a, "ds", schema, samples, slice_count=slices, group_size=G)
    pcp.write_dataset(b, "ds", schema, samples, slice_count=slices, group_size=G)
    fa, fb = sorted(os.listdir(a)), sorted(os.listdir(b))
    assert fa == fb
    for f in fa:
        assert filecmp.cmp(a / f, b / f, shallow=False), f


def test_writer_schema_errors(pcp, tmp_path):
    with pytest.raises(pcp.PcError) as e:
        pcp.write_dataset(tmp_path, "x", {"fields": {}}, [{}])
    assert e.value.errc == "EmptySchema"
    schema = {"fields": {"data": {"type": "bytes"}, "label": {"type": "int32"}}}
    with pytest.raises(pcp.PcError) as e:
        pcp.write_dataset(tmp_path, "x", schema, [{"data": np.zeros(12, np.uint8)}])
    assert e.value.errc == "SchemaMismatch"


def test_pipeline_fails_loudly_without_gpu(pcp, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_16945_b200 import synth
    schema, samples = synth.shapenet(4, n_points=64)
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, group_size=2)
    with pytest.raises(pcp.PcError) as e:
        pcp.Pipeline(primary, synth.graph(["normalize"], batch_size=2))
    assert e.value.errc == "IoFailure" and "no CUDA device" in str(e.value)


def test_slice_shard_partitions(pcp, ref, tmp_path):
    from paper_2603_16945_b200 import shard, synth
    schema, samples = synth.shapenet(50, n_points=32)
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=8, group_size=4)
    idx = shard.read_index(primary)
    ri = ref.index(primary)["entries"]
    assert [(e["shard_id"], e["group_id"], e["scalar_meta"]["row"]) for e in ri] == idx
    for world in (1, 2, 4, 8):
        parts = [shard.slice_shard(idx, world, r) for r in range(world)]
        allids = np.sort(np.concatenate(parts))
        assert np.array_equal(allids, np.arange(len(idx)))
        for r, p in enumerate(parts):  # each GPU owns whole slices
            assert {idx[i][0] % world for i in p} <= {r}


@pytest.mark.parametrize("n,world", [(10, 4), (50, 8), (7, 3), (12, 4)])
def test_strided_shard_matches_reference(pcp, ref, tmp_path, n, world):
    """pad_for_shards + shard_index (metadata.cpp:60-74, distributed.cpp:13-27)."""
    from paper_2603_16945_b200 import shard, synth
    schema, samples = synth.shapenet(n, n_points=16)
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=2, group_size=3)
    full = ref.index(primary)["entries"]
    key = lambda e: (e["shard_id"], e["group_id"], e["scalar_meta"]["row"])
    pos = {key(e): i for i, e in enumerate(full)}
    for r in range(world):
        want = [pos[key(e)] for e in ref.index(primary, world, r)["entries"]]
        assert shard.strided_shard(n, world, r).tolist() == want
