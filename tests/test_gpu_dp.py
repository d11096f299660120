"""Data-parallel consumer on the device stage: per-sample toy gradients from
the pipeline's device views (axis means reduced on the GPU), against the
compiled reference's simulate_data_parallel."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_batches_drive_the_dp_loop(pcp, ref, tmp_path):
    import torch
    from paper_2603_16945_b200 import synth
    from paper_2603_16945_b200.dp import ToyModel, axis_means_batch, dp_shard, simulate_data_parallel
    schema, samples = synth.kitti(24, lo=2000, hi=5000)
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=2, group_size=4)
    params, lr, B = [0.1, -0.2, 0.3, 0.05, 0.5], 0.02, 4
    g = synth.graph([], batch_size=B)
    p = pcp.Pipeline(primary, g, ids=dp_shard(24, 1, 0), epochs=2)
    rep = simulate_data_parallel(iter(p), ToyModel(params, lr), 1, 0,
                                 means_fn=lambda b: axis_means_batch(b, torch))
    p.close()
    want, _ = ref.simulate_dp(primary, 1, 2, B, params, lr)
    assert rep.steps == 2 * 24 // B
    np.testing.assert_allclose(rep.params, want, rtol=1e-12, atol=1e-15)
