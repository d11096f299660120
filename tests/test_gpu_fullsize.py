"""GPU parity at the BASELINE configs' own sizes (SURVEY.md §8(d) op chains).

Every bench workload is checked here at the per-cloud size, group size and
batch it is benched at — raw float and quantized (LZ4 pages) variants — on a
handful of clouds, through the C ABI (pcp_pipeline_*), against the oracle
(oracle/_ref = the compiled reference for reference ops, the C restatement for
the App. C ops fps / voxel / grid_subsample / range_crop):

  C1 ModelNet40   10 000 pts, G 32  : normalize → FPS 1024 → rotate → jitter, B 32
  C2 ShapeNet     2 048 pts, G 64   : normalize → downsample 1024 (+seg) → scale → shuffle, B 32
  C3 S3DIS        ~1 M pts,  G 1    : grid 0.04 → random_crop → downsample 4096, B 4
  C4 KITTI        ~120 k pts, G 16  : range crop → voxel 0.05 (+count) → rotate → flip_yz, B 4
  C5 ScanNet      50 k-500 k, G 4   : grid 0.02 → downsample 40 000 → FPS 20 000, B 4

Integer/byte/index outputs are compared bit-exactly; rotate/jitter floats
within |a-b| <= 1e-5|b| + 1e-6 max|coord| (glibc vs CUDA trig/log ulps).
The committed golden datasets (tests/golden/ds_raw, ds_q: reference-written
pages and reference Pipeline batches) run through the GPU path too.
"""
import json
import os

import numpy as np
import pytest

from expect import assert_batches_equal, expected_run, tolerant_fields

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

# (generator, kwargs, clouds, group, batch, chain)
FULL = {
    "modelnet40": ("modelnet", {"n_points": 10000}, 32, 32, 32),
    "shapenet_part": ("shapenet", {"n_points": 2048}, 128, 64, 32),
    "s3dis": ("s3dis", {"mean_points": 1_000_000}, 4, 1, 4),
    "kitti": ("kitti", {}, 16, 16, 4),
    "scannet": ("scannet", {}, 4, 4, 4),
}


def _dataset(pcp, tmp_path, cfg, quantized):
    from paper_2603_16945_b200 import synth
    gen, kw, n, group, _ = FULL[cfg]
    schema, samples = getattr(synth, gen)(n, quantized=quantized, **kw)
    return pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=1, group_size=group)


@pytest.mark.parametrize("quantized", [False, True], ids=["raw", "quantized"])
@pytest.mark.parametrize("cfg", list(FULL))
def test_config_parity_at_bench_size(pcp, ref, orc, tmp_path, cfg, quantized):
    from paper_2603_16945_b200 import synth
    primary = _dataset(pcp, tmp_path, cfg, quantized)
    g = synth.graph(synth.CHAINS[cfg], batch_size=FULL[cfg][4])
    got = pcp.run_pipeline(primary, g)
    want = expected_run(ref, orc, primary, g)
    assert len(want) >= 1
    assert_batches_equal(got, want, float_fields=tolerant_fields(g))


@pytest.mark.parametrize("cfg", ["s3dis", "kitti"])
def test_bench_size_staged_host_batches(pcp, ref, orc, tmp_path, cfg):
    """The e2e leg's mode (pages staged from pinned host memory, batches
    delivered in pinned host memory) at bench size equals the oracle."""
    from paper_2603_16945_b200 import synth
    primary = _dataset(pcp, tmp_path, cfg, False)
    g = synth.graph(synth.CHAINS[cfg], batch_size=FULL[cfg][4])
    want = expected_run(ref, orc, primary, g)
    p = pcp.Pipeline(primary, g, resident=False, host_batches=True)
    got = []
    while True:
        b = p.next_host_batch()
        if b is None:
            break
        got.append(b)
    p.close()
    assert len(got) == len(want)
    for gb, wb in zip(got, want):
        for k, s in enumerate(wb["samples"]):
            for name, v in s.items():
                arr, offs = gb[name]
                raw = arr.view(np.uint8)[offs[k]:offs[k + 1]]
                if name in tolerant_fields(g):
                    a, b = raw.view(np.float32), v.view(np.uint8).view(np.float32)
                    scale = max(1.0, float(np.abs(b).max())) if b.size else 1.0
                    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6 * scale)
                else:
                    assert np.array_equal(raw, v.view(np.uint8)), (name, k)


@pytest.mark.parametrize("name", ["ds_raw", "ds_q"])
def test_golden_datasets_through_gpu(pcp, name):
    """Reference-written pages (tests/golden/<name>/) → GPU pipeline → the
    reference Pipeline's batches committed in <name>.npz (stacked layout)."""
    z = np.load(os.path.join(HERE, "golden", name + ".npz"))
    g = json.loads(bytes(z["graph"]).decode())
    got = pcp.run_pipeline(os.path.join(HERE, "golden", name, "ds.pcrecord"), g)
    assert len(got) == int(z["n_batches"][0])
    for b in got:
        for field in b["samples"][0]:
            stacked = np.concatenate([s[field].view(np.uint8) for s in b["samples"]])
            assert np.array_equal(stacked, z[f"b{b['batch_index']}_{field}"]), (b["batch_index"], field)
