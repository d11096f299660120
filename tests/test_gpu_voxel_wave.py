"""Multi-CTA voxel stage (voxel_wave.cu) against the oracle
(App. C restatement + reference ops) and against the one-CTA-per-cloud
op_voxel path (option "vx": false), including the statuses it reports and
the k_cloud fallback for keys too wide for the packed sort."""
import numpy as np
import pytest

from expect import assert_batches_equal, expected_run, tolerant_fields

pytestmark = pytest.mark.gpu


def _ds(pcp, tmp_path, gen, n, group, quantized=False, **kw):
    from paper_2603_16945_b200 import synth
    schema, samples = getattr(synth, gen)(n, quantized=quantized, **kw)
    return pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=1, group_size=group)


CHAINS = {
    "s3dis": ("s3dis", dict(mean_points=40000), 6, 1, None),
    "kitti": ("kitti", dict(lo=9000, hi=15000), 6, 3, None),
    "scannet_fps": ("scannet", dict(lo=20000, hi=30000), 4, 2,
                    [("grid_subsample", {"voxel_size": 0.02}), ("downsample", {"num_points": 12000}),
                     ("fps", {"num_points": 300})]),
    "voxel_gather": ("shapenet", dict(n_points=3000), 6, 3,
                     [("voxel", {"voxel_size": 0.05, "gather": ["seg"]}), "random_scale"]),
    "voxel_only_counts": ("kitti", dict(lo=5000, hi=8000), 4, 2,
                          [("voxel", {"voxel_size": 0.3})]),
    "crop_voxel_fps_cluster": ("scannet", dict(lo=30000, hi=45000), 3, 1,
                               [("grid_subsample", {"voxel_size": 0.01}),
                                ("downsample", {"num_points": 24000}), ("fps", {"num_points": 400}),
                                "rotate"]),
}


@pytest.mark.parametrize("buckets", [True, False], ids=["bucket_mode", "lsd_mode"])
@pytest.mark.parametrize("name", list(CHAINS))
def test_vx_stage_matches_oracle_and_cta_path(pcp, ref, orc, tmp_path, name, buckets):
    from paper_2603_16945_b200 import synth
    gen, kw, n, group, chain = CHAINS[name]
    primary = _ds(pcp, tmp_path, gen, n, group, **kw)
    g = synth.graph(chain or synth.CHAINS[name], batch_size=2, drop_remainder=False)
    p = pcp.Pipeline(primary, g, vx=True, vx_min_points=1, vx_buckets=buckets)
    assert p.stats()["vx"], "the multi-CTA voxel stage should take this chain"
    got = []
    for b in p:
        got.append({"epoch": b.epoch, "batch_index": b.batch_index, "samples": b.samples()})
    p.close()
    want = expected_run(ref, orc, primary, g)
    assert_batches_equal(got, want, float_fields=tolerant_fields(g))
    cta = pcp.run_pipeline(primary, g, vx=False)
    assert_batches_equal(got, cta)


def test_vx_bucket_overflow_takes_lsd(pcp, ref, orc, tmp_path):
    """Few wide voxels: buckets above the shared-memory item capacity send
    the cloud to the global LSD sort; a mixed wave (one cloud of each kind)
    is exact."""
    rng = np.random.default_rng(11)
    schema = {"fields": {"data": {"type": "bytes"}, "intensity": {"type": "bytes"},
                         "label": {"type": "int32"}}}
    samples = []
    for i in range(4):
        side = 1.0 if i % 2 == 0 else 40.0
        p = rng.uniform(0, side, (40000, 3)).astype(np.float32)
        samples.append({"data": p.reshape(-1).view(np.uint8),
                        "intensity": rng.uniform(0, 1, 40000).astype(np.float32).view(np.uint8),
                        "label": np.array([i], np.int32)})
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, group_size=2)
    from paper_2603_16945_b200 import synth
    g = synth.graph([("voxel", {"voxel_size": 0.3}), "flip_yz"], batch_size=2)
    got = pcp.run_pipeline(primary, g, vx=True, vx_min_points=1)
    assert_batches_equal(got, expected_run(ref, orc, primary, g))


def test_vx_fallback_wide_keys(pcp, ref, orc, tmp_path):
    """Keys of 3 x 21 bits + the point index do not fit the packed 64-bit
    word: the cloud falls back to k_cloud's op_voxel, same result."""
    rng = np.random.default_rng(5)
    schema = {"fields": {"data": {"type": "bytes"}, "label": {"type": "int32"}}}
    samples = []
    for i in range(2):
        p = rng.uniform(0, 2000.0, (40000, 3)).astype(np.float32)
        p[:8] = [[0, 0, 0], [2000, 2000, 2000], [0.0005, 0, 0], [0.0015, 0, 0], [0, 0.0009, 0],
                 [1000, 1000, 1000], [1000, 1000, 1000.0004], [1999.9, 0, 1]]
        samples.append({"data": p.reshape(-1).view(np.uint8), "label": np.array([i], np.int32)})
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, group_size=1)
    from paper_2603_16945_b200 import synth
    g = synth.graph([("voxel", {"voxel_size": 0.001})], batch_size=1)
    got = pcp.run_pipeline(primary, g, vx=True, vx_min_points=1)
    assert_batches_equal(got, expected_run(ref, orc, primary, g))


CROP_VOX = [("range_crop", {"lo": [0, 0, 0], "hi": [10, 10, 10]}),
            ("voxel", {"voxel_size": 0.5, "origin": [0.5, 0, 0]}), "flip_yz"]
STATUS_CASES = {
    # mutation of cloud 2, chain, op id named by the WorkerPanic
    "empty_after_crop": ("shift", CROP_VOX, 2),
    "below_origin": ("low_x", CROP_VOX, 2),
    "nan": ("nan", [("grid_subsample", {"voxel_size": 0.5}), "flip_yz"], 1),
    "nan_at_point0": ("nan0", [("grid_subsample", {"voxel_size": 0.5}), "flip_yz"], 1),
    "inf": ("inf", [("grid_subsample", {"voxel_size": 0.5}), "flip_yz"], 1),
    "beyond_key_range": ("far", [("grid_subsample", {"voxel_size": 0.5}), "flip_yz"], 1),
}


@pytest.mark.parametrize("case", list(STATUS_CASES))
def test_vx_statuses_match_cta_path(pcp, tmp_path, case):
    """Failing clouds report the same WorkerPanic (op id, Errc) through the
    vx stage as through op_voxel; the clouds before them are served."""
    mut, chain, op = STATUS_CASES[case]
    rng = np.random.default_rng(9)
    schema = {"fields": {"data": {"type": "bytes"}, "intensity": {"type": "bytes"},
                         "label": {"type": "int32"}}}
    samples = []
    for i in range(4):
        p = rng.uniform(0, 10, (3000, 3)).astype(np.float32)
        p[:, 0] = rng.uniform(0.5, 10, 3000)
        if i == 2:
            if mut == "shift":
                p += 100.0
            elif mut == "nan":
                p[1234, 1] = np.nan
            elif mut == "nan0":
                p[0, 2] = np.nan
            elif mut == "inf":
                p[2500, 2] = np.inf
            elif mut == "far":  # key 2^21 on y: one past the App. C key range
                p[1500, 1] = p[:, 1].min() + 0.5 * 2097152.0 + 10.0
            else:
                p[77, 0] = 0.2
        samples.append({"data": p.reshape(-1).view(np.uint8),
                        "intensity": rng.uniform(0, 1, 3000).astype(np.float32).view(np.uint8),
                        "label": np.array([i], np.int32)})
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, group_size=2)
    from paper_2603_16945_b200 import synth
    g = synth.graph(chain, batch_size=1)
    msgs = []
    for opts in ({"vx": True, "vx_min_points": 1}, {"vx": False}):
        p = pcp.Pipeline(primary, g, **opts)
        assert p.stats()["vx"] == opts["vx"]
        out = [p.next_batch().to_host() for _ in range(2)]
        with pytest.raises(pcp.PcError) as ei:
            p.next_batch()
        msgs.append((str(ei.value), out))
        p.close()
    assert msgs[0][0] == msgs[1][0], msgs
    assert f"op {op}:" in msgs[0][0], msgs[0][0]
    # App. C: an empty cloud after the crop is EmptyCloud; every key outside
    # [0, 2^21) (NaN, inf, below the origin, too far) is OutOfBounds
    # (oracle/pcpipe_oracle.c op_voxel)
    want = "EmptyCloud" if mut == "shift" else "OutOfBounds"
    assert want in msgs[0][0], msgs[0][0]
    for a, b in zip(msgs[0][1], msgs[1][1]):
        for k in b:
            assert np.array_equal(a[k][0].view(np.uint8), b[k][0].view(np.uint8))
