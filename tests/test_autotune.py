"""Autotune control plane (paper_2603_16945_b200/autotune.py) on CPU:
proposal phases, GP refinement, exhaustion, the bottleneck rule and the
persisted config format (autotune.cpp:76-88,198-359)."""
import numpy as np
import pytest

from paper_2603_16945_b200 import PcError
from paper_2603_16945_b200.autotune import (MetricsSample, SearchSpace, SurrogateState, TuneConfig,
                                            detect_bottleneck, load_best, persist_best, propose_config)


def test_seed_phase_proposes_unobserved_and_exhausts():
    space = SearchSpace(slots=(2, 3), wave_batches=(1, 2))
    rng = np.random.default_rng(0)
    st = SurrogateState()
    seen = set()
    for _ in range(4):
        c = propose_config(st, space, "seed", rng)
        assert (c.slots, c.wave_batches) not in seen
        seen.add((c.slots, c.wave_batches))
        c.objective = 1.0
        st.observed.append(c)
    with pytest.raises(PcError) as ei:
        propose_config(st, space, "seed", rng)
    assert ei.value.errc == "OutOfRange"


def test_refine_phase_follows_the_surrogate():
    """Objective rising with slots and falling with wave size: expected
    improvement picks an unobserved point towards the improving corner."""
    space = SearchSpace(slots=(2, 3, 4, 5, 6), wave_batches=(1, 2, 4, 8, 16))
    st = SurrogateState()
    for s, w in [(2, 16), (3, 8), (4, 4), (2, 1), (6, 16)]:
        st.observed.append(TuneConfig(s, w, objective=10.0 * s - np.log2(w)))
    c = propose_config(st, space, "refine", np.random.default_rng(3))
    assert c.slots >= 5 and c.wave_batches < 16, c


def test_detect_bottleneck_rule():
    def window(empty_per_poll):
        return [MetricsSample(i * 0.01, [], 10 * i, int(10 * i * empty_per_poll), 0.0, 0) for i in range(30)]
    assert detect_bottleneck(window(0.5)) == "data_side"
    assert detect_bottleneck(window(0.1)) == "consumer_side"
    with pytest.raises(PcError):
        detect_bottleneck(window(0.5)[:29])


def test_persist_and_load(tmp_path):
    p = tmp_path / "best.json"
    persist_best(TuneConfig(5, 8, objective=123.0), p)
    c = load_best(p)
    assert (c.slots, c.wave_batches, c.objective) == (5, 8, 123.0)
    p.write_text('{"version": 2}')
    with pytest.raises(PcError) as ei:
        load_best(p)
    assert ei.value.errc == "SchemaMismatch"
    with pytest.raises(PcError) as ei:
        load_best(tmp_path / "missing.json")
    assert ei.value.errc == "IoFailure"
