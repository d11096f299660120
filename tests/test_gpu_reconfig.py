"""Live reconfiguration of the device stage (pcp_pipeline_update_config,
the update_op_config analogue) and autotuning over it: batches, their order
and their seeds never change (test_pipeline.cpp:336-367's property)."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ds(pcp, tmp_path, n=160, group=8, slices=2):
    from paper_2603_16945_b200 import synth
    schema, samples = synth.shapenet(n, n_points=600)
    return pcp.write_dataset(tmp_path, "ds", schema, samples, slice_count=slices, group_size=group)


def _key(b):
    return b.epoch, b.batch_index


def test_update_config_keeps_content(pcp, tmp_path):
    from paper_2603_16945_b200 import autotune, synth
    primary = _ds(pcp, tmp_path)
    g = synth.graph(synth.CHAINS["shapenet_part"], batch_size=4, drop_remainder=False)
    want = {_key(b): b.to_host() for b in pcp.Pipeline(primary, g, epochs=3, wave_batches=3, slots=4)}
    p = pcp.Pipeline(primary, g, epochs=3, wave_batches=3, slots=4)
    got = []
    plan = {7: {"slots": 2, "wave_batches": 1}, 30: {"slots": 6, "wave_batches": 7},
            61: {"wave_batches": 2}, 90: {"slots": 3}}
    k = 0
    while True:
        if k in plan:
            autotune.update_config(p, **plan[k])
        b = p.next_batch()
        if b is None:
            break
        got.append((_key(b), b.to_host()))
        k += 1
    m = autotune.metrics(p)
    p.close()
    # updates that arrive while an earlier one is still draining merge into it
    assert 3 <= m["reconfigs"] <= 4 and m["slots"] == 3 and m["wave_batches"] == 2
    assert [x[0] for x in got] == list(want)
    for key, host in got:
        for name in want[key]:
            assert np.array_equal(host[name][0].view(np.uint8), want[key][name][0].view(np.uint8)), (key, name)
    assert m["batches_emitted"] == len(want) and m["items_emitted"] == 3 * 160
    kinds = [o["kind"] for o in m["ops"]]
    assert kinds[0] == "source" and "map" in kinds and kinds[-1] == "batch"


def test_update_config_rejects_bad_knobs(pcp, tmp_path):
    from paper_2603_16945_b200 import autotune, synth
    primary = _ds(pcp, tmp_path, n=32)
    g = synth.graph(["normalize"], batch_size=4)
    p = pcp.Pipeline(primary, g)
    for bad, errc in (({"slots": 1}, "OutOfBounds"), ({"slots": 9}, "OutOfBounds"),
                      ({"wave_batches": 0}, "OutOfBounds"), ({"workers": 3}, "UnknownOp")):
        with pytest.raises(pcp.PcError) as ei:
            autotune.update_config(p, **bad)
        assert ei.value.errc == errc, (bad, ei.value)
    p.close()
    ps = pcp.Pipeline(primary, g, stream=True)
    with pytest.raises(pcp.PcError):
        autotune.update_config(ps, slots=3)
    ps.close()


def test_autotune_live_pipeline(pcp, tmp_path):
    """autotune evaluates candidates on the live pipeline (draining batches),
    leaves the best applied, and the batches that follow are unchanged."""
    from paper_2603_16945_b200 import autotune, synth
    primary = _ds(pcp, tmp_path, n=256)
    g = synth.graph(synth.CHAINS["shapenet_part"], batch_size=4)
    epochs = 400
    p = pcp.Pipeline(primary, g, epochs=epochs, wave_batches=4)
    best, hist = autotune.autotune(p, autotune.SearchSpace(slots=(2, 3, 4), wave_batches=(1, 4, 16)),
                                   iterations=4, seed_phase=2, eval_window_ms=40)
    assert len(hist) >= 2 and best.objective == max(h.objective for h in hist) > 0
    tail = []
    while True:  # the final update lands at a wave boundary: drain until it shows
        b = p.next_batch()
        if b is None:
            break
        tail.append((_key(b), b.to_host()))  # views live until the next next_batch
        m = autotune.metrics(p)
        if len(tail) >= 40 and m["slots"] == best.slots and m["wave_batches"] == best.wave_batches:
            break
        if len(tail) == 600:
            break
    m = autotune.metrics(p)
    assert m["slots"] == best.slots and m["wave_batches"] == best.wave_batches
    keys = [k for k, _ in tail]
    ref = pcp.Pipeline(primary, g, epochs=epochs)
    want = {}
    for b in ref:
        if _key(b) in keys:
            want[_key(b)] = b.to_host()
        if len(want) == len(keys):
            break
    ref.close()
    for k, h in tail:
        for name in h:
            assert np.array_equal(h[name][0].view(np.uint8), want[k][name][0].view(np.uint8))
    p.close()
