"""The device page encoder (pcp_write_dataset_device):
files byte-identical to the reference's write_dataset and to the host
writer, over stored-raw and LZ4 pages, adversarial LZ4 inputs (long
matches, overlapping matches, 255-runs, zero runs) and edge cases."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _files(d):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))}


def _check(pcp, ref, tmp_path, schema, samples, slices, group):
    dev = tmp_path / "dev"
    host = tmp_path / "host"
    refd = tmp_path / "ref"
    pcp.write_dataset(dev, "ds", schema, samples, slice_count=slices, group_size=group, device=0)
    pcp.write_dataset(host, "ds", schema, samples, slice_count=slices, group_size=group)
    ref.write_dataset(refd, "ds", schema, samples, slice_count=slices, group_size=group)
    a, b, c = _files(dev), _files(host), _files(refd)
    assert a.keys() == c.keys()
    for f in c:
        assert a[f] == c[f], f
        assert b[f] == c[f], f


@pytest.mark.parametrize("gen,kw,q,group", [("shapenet", {"n_points": 2048}, False, 16),
                                            ("shapenet", {"n_points": 2048}, True, 16),
                                            ("kitti", {"lo": 3000, "hi": 6000}, True, 3),
                                            ("kitti", {"lo": 3000, "hi": 6000}, False, 3),
                                            ("modelnet", {"n_points": 1000}, True, 5)])
def test_device_writer_matches_reference(pcp, ref, tmp_path, gen, kw, q, group):
    from paper_2603_16945_b200 import synth
    schema, samples = getattr(synth, gen)(24, quantized=q, **kw)
    _check(pcp, ref, tmp_path, schema, samples, slices=3, group=group)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_device_writer_adversarial_lz4(pcp, ref, tmp_path, seed):
    from test_gpu_pipeline import _adversarial_blob
    rng = np.random.default_rng(seed)
    schema = {"fields": {"blob": {"type": "bytes"}, "id": {"type": "int32"}, "name": {"type": "string"}}}
    samples = []
    for i in range(14):
        n = int(rng.choice([0, 1, 5, 11, 12, 13, 100, 4096, 70000, 200000]))
        samples.append({"blob": _adversarial_blob(rng, n) if n else np.zeros(0, np.uint8),
                        "id": np.array([i], np.int32), "name": "s" * int(rng.integers(0, 40))})
    samples.append({"blob": np.zeros(300000, np.uint8), "id": np.array([99], np.int32), "name": ""})
    _check(pcp, ref, tmp_path, schema, samples, slices=2, group=int(rng.integers(1, 5)))
