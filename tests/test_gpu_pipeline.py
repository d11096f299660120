"""GPU parity: the B200 pipeline (through the C ABI) against the oracles on
the same PcRecord files, graph JSON, walk and seeds."""
import json
import os

import numpy as np
import pytest

from expect import assert_batches_equal, expected_run, tolerant_fields

pytestmark = pytest.mark.gpu


def _ds(pcp, tmp_path, gen, n, group, slices=1, quantized=False, **kw):
    from paper_2603_16945_b200 import synth
    schema, samples = getattr(synth, gen)(n, quantized=quantized, **kw)
    return pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=slices, group_size=group)


def _run(pcp, primary, graph, **kw):
    return pcp.run_pipeline(primary, graph, **kw)


@pytest.mark.parametrize("quantized,pj", [(False, None), (True, False), (True, True)])
def test_shapenet_chain_parity(pcp, ref, orc, tmp_path, quantized, pj):
    """C2 chain: normalize → downsample 1024 (+seg) → random_scale → shuffle;
    LZ4 pages with either phase-4 path."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 70, group=16, slices=2, quantized=quantized)
    g = synth.graph(synth.CHAINS["shapenet_part"], batch_size=8)
    got = _run(pcp, primary, g, **({} if pj is None else {"lz4_pointer_jumping": pj}))
    want = expected_run(ref, orc, primary, g)
    assert_batches_equal(got, want)


@pytest.mark.parametrize("op", ["normalize", "translate", "jitter", "rotate", "random_scale",
                                "flip_yz", "random_crop", ("downsample", {"num_points": 300}),
                                ("downsample", {"num_points": 1500})])
def test_reference_op_parity(pcp, ref, orc, tmp_path, op):
    """Each reference map kind alone, against the compiled reference Pipeline."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "modelnet", 24, group=8, n_points=1000)
    g = synth.graph([op], batch_size=4)
    got = _run(pcp, primary, g)
    want = expected_run(ref, orc, primary, g)
    assert_batches_equal(got, want, float_fields=tolerant_fields(g))


def test_color_augment_and_crop_parity(pcp, ref, orc, tmp_path):
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "scannet", 6, group=2, lo=3000, hi=9000)
    g = synth.graph(["color_augment", "random_crop", ("downsample", {"num_points": 2048})],
                    batch_size=2)
    assert_batches_equal(_run(pcp, primary, g), expected_run(ref, orc, primary, g))


def test_fps_parity(pcp, ref, orc, tmp_path):
    """C1 chain at reduced size (FPS is App. C; oracle = restatement)."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "modelnet", 8, group=4, n_points=3000)
    g = synth.graph([("normalize", {}), ("fps", {"num_points": 256}), ("rotate", {}), ("jitter", {})],
                    batch_size=4)
    got = _run(pcp, primary, g)
    want = expected_run(ref, orc, primary, g)
    assert_batches_equal(got, want, float_fields=tolerant_fields(g))


def test_kitti_chain_parity(pcp, ref, orc, tmp_path):
    """C4: range crop → voxel 0.05 m (counts) → rotate → flip_yz (CSR batch)."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "kitti", 4, group=2, lo=20000, hi=30000)
    g = synth.graph(synth.CHAINS["kitti"], batch_size=2)
    got = _run(pcp, primary, g)
    want = expected_run(ref, orc, primary, g)
    assert_batches_equal(got, want, float_fields=tolerant_fields(g))


def test_fused_graph_and_epochs(pcp, ref, orc, tmp_path):
    """fuse_maps seeding by original op ids; 3 epochs; remainder kept."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 21, group=5, n_points=600)
    g = synth.graph(["translate", "random_scale", "flip_yz"], batch_size=4, drop_remainder=False)
    fused_map = {"id": 1, "kind": "map", "num_workers": 2, "queue_capacity": 8,
                 "fused": [{"map": "translate", "params": {}, "op_id": 1},
                           {"map": "random_scale", "params": {}, "op_id": 2},
                           {"map": "flip_yz", "params": {}, "op_id": 3}]}
    gf = dict(g, ops=[g["ops"][0], fused_map] + g["ops"][4:])
    want = expected_run(ref, orc, primary, g, epochs=3)
    assert_batches_equal(_run(pcp, primary, g, epochs=3), want)
    assert_batches_equal(_run(pcp, primary, gf, epochs=3), want)


def test_shard_walk(pcp, ref, orc, tmp_path):
    """A GPU's shard = an explicit entry list; seeds use the walk position."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 40, group=8, slices=4, n_points=512)
    ids = [i for i in range(40) if (i // 10) % 2 == 1]  # slices 1 and 3
    g = synth.graph(["normalize", ("downsample", {"num_points": 256})], batch_size=4)
    assert_batches_equal(_run(pcp, primary, g, ids=ids), expected_run(ref, orc, primary, g, ids=ids))


def test_staged_matches_resident(pcp, tmp_path):
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 48, group=8, quantized=True, n_points=700)
    g = synth.graph(synth.CHAINS["shapenet_part"][:2], batch_size=8)
    a = _run(pcp, primary, g, resident=True, wave_batches=2)
    b = _run(pcp, primary, g, resident=False, wave_batches=3)
    assert_batches_equal(a, b)


def test_serial_fisher_yates_path(pcp, ref, orc, tmp_path):
    """The rare Lemire-rejection fallback (serial engine) is exact too."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 16, group=8, n_points=900)
    g = synth.graph([("downsample", {"num_points": 500}), ("downsample", {"num_points": 1200})],
                    batch_size=4)
    want = expected_run(ref, orc, primary, g)
    assert_batches_equal(_run(pcp, primary, g, force_serial_fy=True), want)


def test_preseeded_states_match_in_kernel_seeding(pcp, ref, orc, tmp_path, monkeypatch):
    """k_seed_states (MT19937-64 seeded per sample and RNG op ahead of k_cloud)
    against the in-kernel serial seeding (PCP_NO_PRESEED) and the reference,
    over every RNG op kind in one chain."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "scannet", 6, group=2, lo=3000, hi=9000)
    g = synth.graph(["color_augment", "translate", "flip_yz", "random_scale", "random_crop",
                     ("downsample", {"num_points": 2048}), "rotate", "jitter"], batch_size=2)
    pre = _run(pcp, primary, g)
    monkeypatch.setenv("PCP_NO_PRESEED", "1")
    assert_batches_equal(_run(pcp, primary, g), pre)
    assert_batches_equal(pre, expected_run(ref, orc, primary, g), float_fields=tolerant_fields(g))


def test_corrupt_payload_is_worker_panic(pcp, tmp_path):
    """A flipped payload byte → CRC mismatch → WorkerPanic at that batch."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 32, group=8, n_points=256)
    with open(primary, "rb") as f:
        blob = bytearray(f.read())
    blob[-100] ^= 0x10  # inside the last group's block payload
    with open(primary, "wb") as f:
        f.write(blob)
    g = synth.graph(["normalize"], batch_size=8)
    p = pcp.Pipeline(primary, g)
    for _ in range(3):
        assert p.next_batch() is not None  # groups 0..2 are intact
    with pytest.raises(pcp.PcError) as ei:
        p.next_batch()
    assert ei.value.errc == "WorkerPanic"
    assert "ChecksumMismatch" in str(ei.value)
    p.close()


def test_empty_cloud_and_missing_field(pcp, tmp_path):
    schema = {"fields": {"data": {"type": "bytes"}, "label": {"type": "int32"}}}
    samples = [{"data": np.zeros(0, np.uint8), "label": np.array([1], np.int32)}] * 4
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, group_size=4)
    from paper_2603_16945_b200 import synth
    p = pcp.Pipeline(primary, synth.graph(["normalize"], batch_size=2))
    with pytest.raises(pcp.PcError) as ei:
        p.next_batch()
    assert "EmptyCloud" in str(ei.value) and "op 1" in str(ei.value)
    p.close()


def test_no_map_passthrough_stacks(pcp, ref, orc, tmp_path):
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "kitti", 6, group=3, lo=1000, hi=1000)
    g = synth.graph([], batch_size=3)
    assert_batches_equal(_run(pcp, primary, g), expected_run(ref, orc, primary, g))


@pytest.mark.parametrize("quantized", [False, True])
def test_s3dis_chain_parity(pcp, ref, orc, tmp_path, quantized):
    """C3 at reduced size: grid 0.04 m → random_crop → downsample 4096."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "s3dis", 4, group=1, quantized=quantized, mean_points=60000)
    g = synth.graph(synth.CHAINS["s3dis"], batch_size=2)
    assert_batches_equal(_run(pcp, primary, g), expected_run(ref, orc, primary, g))


def test_scannet_chain_parity(pcp, ref, orc, tmp_path):
    """C5 at reduced size: grid 0.02 m → downsample → FPS."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "scannet", 4, group=2, lo=20000, hi=40000)
    g = synth.graph([("grid_subsample", {"voxel_size": 0.02}), ("downsample", {"num_points": 6000}),
                     ("fps", {"num_points": 500})], batch_size=2)
    assert_batches_equal(_run(pcp, primary, g), expected_run(ref, orc, primary, g))


def test_voxel_gathers_extra_field_and_counts(pcp, ref, orc, tmp_path):
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 6, group=3, n_points=3000)
    g = synth.graph([("voxel", {"voxel_size": 0.1, "gather": ["seg"]}), "random_scale"], batch_size=3)
    assert_batches_equal(_run(pcp, primary, g), expected_run(ref, orc, primary, g))


def test_cluster_fps_chain_parity(pcp, ref, orc, tmp_path):
    """FPS input above one CTA's registers (downsample 24000 -> cluster of 3
    CTAs): chain prefix run redundantly per CTA, FPS split over the cluster."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "scannet", 5, group=2, lo=30000, hi=45000)
    g = synth.graph([("grid_subsample", {"voxel_size": 0.01}), ("downsample", {"num_points": 24000}),
                     ("fps", {"num_points": 700}), "rotate"], batch_size=2, drop_remainder=False)
    got = _run(pcp, primary, g)
    want = expected_run(ref, orc, primary, g)
    assert_batches_equal(got, want, float_fields=tolerant_fields(g))


@pytest.mark.parametrize("slots", [2, 4])
def test_async_d2h_matches_sync(pcp, tmp_path, slots):
    """pcp_memcpy_d2h_async of every batch with one sync at the end equals the
    synchronous copies: small waves and few slots force slot reuse while
    copies of older batches are still queued (the 'served' event guard)."""
    import torch
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 96, group=8, n_points=700)
    g = synth.graph(synth.CHAINS["shapenet_part"][:3], batch_size=4)
    want = [b.to_host() for b in pcp.Pipeline(primary, g, wave_batches=2, slots=slots)]
    L = pcp.lib()
    got, keep = [], []
    p = pcp.Pipeline(primary, g, wave_batches=2, slots=slots)
    for b in p:
        host = {}
        for name, (kind, ptr, nbytes, offs, _) in b.fields.items():
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)  # truly async
            assert L.pcp_memcpy_d2h_async(buf.data_ptr(), ptr, nbytes, b.stream) == 0
            host[name] = (buf, nbytes, offs)
            keep.append(buf)
        got.append(host)
    assert L.pcp_stream_sync(p.stream) == 0
    p.close()
    assert len(got) == len(want)
    for gb, wb in zip(got, want):
        for name in wb:
            buf, nbytes, _ = gb[name]
            assert np.array_equal(buf.numpy()[:nbytes], wb[name][0].view(np.uint8)), name


@pytest.mark.parametrize("kind,resident", [("shapenet", True), ("shapenet", False),
                                           ("kitti", True), ("kitti", False)])
def test_host_batches_match_device_batches(pcp, tmp_path, kind, resident):
    """host_batches (one D2H per field per wave into pinned host memory;
    per-sample copies for ragged fields, e.g. voxel outputs) serves the same
    bytes and offsets as the device batches, across slot reuse."""
    from paper_2603_16945_b200 import synth
    if kind == "shapenet":
        primary = _ds(pcp, tmp_path, "shapenet", 96, group=8, n_points=700)
        g = synth.graph(synth.CHAINS["shapenet_part"], batch_size=4)
    else:
        primary = _ds(pcp, tmp_path, "kitti", 24, group=4, lo=3000, hi=5000)
        g = synth.graph(synth.CHAINS["kitti"], batch_size=2)
    want = [b.to_host() for b in pcp.Pipeline(primary, g, wave_batches=2, slots=2, epochs=2)]
    p = pcp.Pipeline(primary, g, wave_batches=2, slots=2, epochs=2, resident=resident, host_batches=True)
    got = []
    while True:
        b = p.next_host_batch()
        if b is None:
            break
        got.append(b)
    st = p.stats()
    p.close()
    assert len(got) == len(want)
    total = 0
    for gb, wb in zip(got, want):
        assert gb.keys() == wb.keys()
        for name in wb:
            assert np.array_equal(gb[name][1], wb[name][1]), name
            assert np.array_equal(gb[name][0].view(np.uint8), wb[name][0].view(np.uint8)), name
            total += wb[name][0].nbytes
    assert st["d2h_bytes"] == total


def _adversarial_blob(rng, n):
    """Bytes that drive the LZ4 decoder through its corner cases: runs of one
    byte and short-period patterns (self-overlapping matches, offsets 1..8),
    random stretches (literals, some > 64 KB -> long 255-continued lengths),
    repeats of earlier content up to ~60 KB back, and dense small-label
    regions (chains of offset-4 matches)."""
    out, size = [], 0
    while size < n:
        kind = rng.integers(0, 6)
        if kind == 0:
            piece = np.full(int(rng.integers(4, 3000)), rng.integers(0, 256), np.uint8)
        elif kind == 1:
            per = int(rng.integers(2, 9))
            piece = np.tile(rng.integers(0, 256, per, dtype=np.uint8), int(rng.integers(2, 600)))
        elif kind == 2:
            piece = rng.integers(0, 256, int(rng.integers(1, 70000 if rng.random() < 0.15 else 2000)),
                                 dtype=np.uint8)
        elif kind == 3 and out:
            prev = np.concatenate(out)
            back = int(rng.integers(1, min(len(prev), 60000) + 1))
            ln = int(rng.integers(4, 5000))
            piece = np.resize(prev[len(prev) - back:], ln)
        else:
            labels = rng.integers(0, 4, int(rng.integers(16, 800))).astype(np.int32)
            piece = np.repeat(labels, rng.integers(1, 40, len(labels))).view(np.uint8)
        out.append(piece.astype(np.uint8))
        size += len(piece)
    return np.concatenate(out)[:n]


@pytest.mark.parametrize("pj", [False, True])
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_lz4_adversarial_pages_through_pipeline(pcp, ref, tmp_path, seed, pj):
    """Pipeline decode of adversarial LZ4 pages (k_page_decode: skim with
    skipped windows, slow path; phase 4 by k_page_matches' pointer-jumping
    match groups, or page-wide pointer jumping) is byte-exact against the
    reference reader."""
    rng = np.random.default_rng(seed)
    schema = {"fields": {"blob": {"type": "bytes"}, "id": {"type": "int32"}}}
    samples = [{"blob": _adversarial_blob(rng, int(rng.integers(20000, 300000))),
                "id": np.array([i], np.int32)} for i in range(24)]
    primary = pcp.write_dataset(tmp_path, "ds", schema, samples, group_size=6)  # compressible: LZ4 pages
    got = []
    for b in pcp.Pipeline(primary, {"base_seed": 1, "drop_remainder": False, "ops": [
            {"id": 0, "kind": "source", "num_workers": 1, "queue_capacity": 8},
            {"id": 1, "kind": "batch", "batch_size": 4, "num_workers": 1, "queue_capacity": 8},
            {"id": 2, "kind": "sink", "num_workers": 1, "queue_capacity": 8}]}, lz4_pointer_jumping=pj):
        host = b.to_host()
        arr, offs = host["blob"]
        for k in range(b.n_samples):
            got.append(bytes(arr.view(np.uint8)[offs[k]:offs[k + 1]]))
    assert len(got) == len(samples)
    for i, s in enumerate(samples):
        assert got[i] == bytes(s["blob"]), i


@pytest.mark.parametrize("resident", [True, False])
def test_corrupt_payload_host_batches_serves_intact_batches(pcp, tmp_path, resident):
    """host_batches: the batches of a wave before its failing batch are served
    intact from pinned host memory (first wave of the slot, so no stale
    buffers exist), then the failing batch raises WorkerPanic."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 32, group=8, n_points=256)
    g = synth.graph(["normalize"], batch_size=8)
    want = [b.to_host() for b in pcp.Pipeline(primary, g)][:3]
    with open(primary, "rb") as f:
        blob = bytearray(f.read())
    blob[-100] ^= 0x10  # inside the last group's block payload
    with open(primary, "wb") as f:
        f.write(blob)
    p = pcp.Pipeline(primary, g, host_batches=True, resident=resident)
    for k in range(3):
        got = p.next_host_batch()
        assert got is not None
        for name in want[k]:
            assert np.array_equal(got[name][0].view(np.uint8), want[k][name][0].view(np.uint8)), (k, name)
    with pytest.raises(pcp.PcError) as ei:
        p.next_host_batch()
    assert ei.value.errc == "WorkerPanic" and "ChecksumMismatch" in str(ei.value)
    p.close()


def test_lz4_phase4_path_choice(pcp, ref, orc, tmp_path):
    """Auto choice of the LZ4 phase-4 path: pages of >= 32
    clouds on average keep the warp-per-page resolver, pages of few large
    clouds take page-wide pointer jumping; both give the oracle's batches."""
    from paper_2603_16945_b200 import synth
    g = synth.graph(synth.CHAINS["shapenet_part"][:2], batch_size=8)
    for group, want_pj in ((32, False), (4, True)):
        primary = _ds(pcp, tmp_path / f"g{group}", "shapenet", 128, group=group, slices=2, quantized=True)
        p = pcp.Pipeline(primary, g)
        got = [{"epoch": b.epoch, "batch_index": b.batch_index, "samples": b.samples()} for b in p]
        st = p.stats()
        p.close()
        assert st["block_pages_lz4"] > 0
        assert (st["lz4_pj_waves"] > 0) == want_pj, st
        assert_batches_equal(got, expected_run(ref, orc, primary, g))
