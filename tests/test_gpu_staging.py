"""Page staging: shard-local loading and streaming the
slice files through reader threads into the wave slots' pinned buffers
(read → H2D → decode → transform → batch overlapped across waves), against
the oracle and the resident path."""
import os

import numpy as np
import pytest

from expect import assert_batches_equal, expected_run, tolerant_fields

pytestmark = pytest.mark.gpu


def _ds(pcp, tmp_path, gen, n, group, slices, quantized=False, **kw):
    from paper_2603_16945_b200 import synth
    schema, samples = getattr(synth, gen)(n, quantized=quantized, **kw)
    return pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=slices, group_size=group)


def _slice_bytes(primary):
    d = os.path.dirname(primary)
    return sum(os.path.getsize(os.path.join(d, f)) for f in os.listdir(d) if ".pcrecord" in f)


def test_shard_local_loading(pcp, ref, orc, tmp_path):
    """Each rank of a 2-way slice shard loads only its own slices (about half
    of the bytes), and each shard's batches equal the reference run over the
    same entry list (shard-local seeds, streaming.cpp:357)."""
    from paper_2603_16945_b200 import shard, synth
    primary = _ds(pcp, tmp_path, "shapenet", 64, group=8, slices=4, n_points=700)
    g = synth.graph(synth.CHAINS["shapenet_part"][:3], batch_size=4)
    idx = shard.read_index(primary)
    total = _slice_bytes(primary)
    seen = set()
    for rank in range(2):
        ids = shard.slice_shard(idx, 2, rank)
        p = pcp.Pipeline(primary, g, ids=ids)
        st = p.stats()
        assert 0.3 * total < st["loaded_bytes"] < 0.7 * total, (st["loaded_bytes"], total)
        got = [{"epoch": b.epoch, "batch_index": b.batch_index, "samples": b.samples()} for b in p]
        p.close()
        assert_batches_equal(got, expected_run(ref, orc, primary, g, ids=ids))
        seen |= set(int(i) for i in ids)
    assert seen == set(range(len(idx)))


@pytest.mark.parametrize("cfg,threads", [("shapenet_part", 1), ("shapenet_part", 4), ("kitti", 3),
                                         ("s3dis", 8)])
def test_stream_matches_oracle(pcp, ref, orc, tmp_path, cfg, threads):
    """Pages read from the slice files per wave (small waves, 2-3 slots:
    every slot's pinned buffer is refilled several times) give the oracle's
    batches, also with host_batches."""
    from paper_2603_16945_b200 import synth
    if cfg == "shapenet_part":
        primary = _ds(pcp, tmp_path, "shapenet", 96, group=8, slices=3, quantized=threads == 4, n_points=900)
        B = 4
    elif cfg == "kitti":
        primary = _ds(pcp, tmp_path, "kitti", 24, group=2, slices=3, lo=3000, hi=6000)
        B = 2
    else:
        primary = _ds(pcp, tmp_path, "s3dis", 6, group=1, slices=2, mean_points=50000)
        B = 2
    g = synth.graph(synth.CHAINS[cfg], batch_size=B)
    want = expected_run(ref, orc, primary, g, epochs=2)
    p = pcp.Pipeline(primary, g, stream=True, reader_threads=threads, wave_batches=2, slots=2 + threads % 2,
                     epochs=2)
    got = [{"epoch": b.epoch, "batch_index": b.batch_index, "samples": b.samples()} for b in p]
    st = p.stats()
    p.close()
    assert st["stream"] and st["loaded_bytes"] == 0 and st["read_bytes"] > 0
    assert_batches_equal(got, want, float_fields=tolerant_fields(g))
    p = pcp.Pipeline(primary, g, stream=True, reader_threads=threads, host_batches=True, wave_batches=3, epochs=2)
    host = []
    while True:
        b = p.next_host_batch()
        if b is None:
            break
        host.append(b)
    p.close()
    assert len(host) == len(want)
    for hb, wb in zip(host, want):
        for k, smp in enumerate(wb["samples"]):
            for name, v in smp.items():
                arr, offs = hb[name]
                raw = arr.view(np.uint8)[offs[k]:offs[k + 1]]
                if name in tolerant_fields(g):
                    np.testing.assert_allclose(raw.view(np.float32), v.view(np.uint8).view(np.float32),
                                               rtol=1e-5, atol=1e-6 * max(1.0, float(np.abs(v.view(np.uint8).view(np.float32)).max())))
                else:
                    assert np.array_equal(raw, v.view(np.uint8)), (name, k)


def test_stream_read_failure_is_io_failure(pcp, tmp_path):
    """A slice file truncated after open: the reader's short read surfaces
    from next_batch as IoFailure (no hang, no stale data)."""
    from paper_2603_16945_b200 import synth
    primary = _ds(pcp, tmp_path, "shapenet", 64, group=8, slices=2, n_points=500)
    g = synth.graph(["normalize"], batch_size=8)
    p = pcp.Pipeline(primary, g, stream=True, wave_batches=1, slots=2)
    cont = primary + "1"
    with open(cont, "r+b") as f:
        f.truncate(100)
    with pytest.raises(pcp.PcError) as ei:
        for _ in p:
            pass
    assert ei.value.errc == "IoFailure"
    p.close()


def test_caller_supplied_pages_like_stream_dataset(pcp, ref, orc, tmp_path):
    """pcp_pipeline_open_source driven like stream_dataset's SourceFn
    (streaming.cpp:324-351): slices 'download' in the background, the page
    source blocks until the requested slice is present, consumption is
    reported per wave.  Output = the reference run over the same shard."""
    import threading
    import time
    from paper_2603_16945_b200 import shard, synth
    primary = _ds(pcp, tmp_path, "shapenet", 96, group=8, slices=4, n_points=600)
    g = synth.graph(synth.CHAINS["shapenet_part"], batch_size=4)
    with open(primary, "rb") as f:
        head = f.read(10)
        (jl,) = np.frombuffer(head[6:10], np.uint32)
        header = head + f.read(int(jl))
    d = os.path.dirname(primary)
    names = sorted(f for f in os.listdir(d) if ".pcrecord" in f)
    files = {}
    for i, name in enumerate(["ds.pcrecord"] + [f"ds.pcrecord{k}" for k in range(1, len(names))]):
        with open(os.path.join(d, name), "rb") as f:
            files[i] = f.read()[len(header) if i == 0 else 0:]
    present, cv = set(), threading.Condition()

    def downloader():
        for sl in (3, 1, 0, 2):
            time.sleep(0.05)
            with cv:
                present.add(sl)
                cv.notify_all()

    def read(sl, off, n):
        with cv:
            cv.wait_for(lambda: sl in present, timeout=30)
        return files[sl][off:off + n]

    consumed = []
    idx = shard.read_index(primary)
    ids = shard.strided_shard(len(idx), 2, 1)  # the reference's padded strided rule
    t = threading.Thread(target=downloader)
    t.start()
    p = pcp.Pipeline.from_source(header, g, read, lambda e, f, n: consumed.append((e, f, n)), ids=ids,
                                 epochs=2, wave_batches=2, slots=2)
    got = [{"epoch": b.epoch, "batch_index": b.batch_index, "samples": b.samples()} for b in p]
    p.close()
    t.join()
    assert_batches_equal(got, expected_run(ref, orc, primary, g, ids=ids, epochs=2))
    per_epoch = {}
    for e, f, n in consumed:
        per_epoch[e] = per_epoch.get(e, 0) + n
    assert per_epoch == {0: len(ids) // 4 * 4, 1: len(ids) // 4 * 4}
