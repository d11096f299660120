"""Live reconfiguration and autotuning of the device stage's knobs
(SURVEY.md §8(f)3), with the reference's control-plane contract
(proj/core/include/pcpipe/autotune.hpp:35-127, src/autotune.cpp:19-409):

* ``collect_metrics`` / ``detect_bottleneck``: MetricsSnapshot samples
  (``pcp_pipeline_metrics``) and the sink empty-poll ratio rule (data side
  when > threshold over >= 30 samples, autotune.cpp:76-88).
* ``SearchSpace`` / ``propose_config``: random seeding, then a Gaussian-
  process surrogate (isotropic squared exponential on min-max normalised
  dimensions) maximising expected improvement over 512 random candidates
  (autotune.cpp:122-283).  The knobs are the device stage's: wave slots
  (waves in flight = streams) and wave size in batches -- the GPU analogue of
  the reference's (workers, queue capacity) per map operator.
* ``measure_throughput`` / ``apply_and_measure``: items/s after a one-window
  warm-up on the live pipeline, draining batches like the reference's
  SinkDrainer; knobs applied through ``pcp_pipeline_update_config`` (the
  update_op_config analogue: content, order and seeds do not change).
* ``persist_best`` / ``load_best``: the versioned JSON file
  (autotune.cpp:313-359).

Host-side control plane only; every batch is still produced by the CUDA
stage.
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from ._lib import PcError, K, lib, _check

__all__ = ["MetricsSample", "collect_metrics", "detect_bottleneck", "SearchSpace", "TuneConfig",
           "SurrogateState", "propose_config", "measure_throughput", "apply_and_measure",
           "persist_best", "load_best", "autotune", "metrics", "update_config"]


def metrics(pipeline) -> dict:
    """Pipeline::metrics() (pipeline.cpp:734-766) of the device stage."""
    return json.loads(lib().pcp_pipeline_metrics(pipeline._h).decode())


def update_config(pipeline, **knobs) -> None:
    """Pipeline::update_op_config (pipeline.cpp:691-732) for the device knobs
    (slots, wave_batches); applied at the next wave boundary."""
    _check(lib().pcp_pipeline_update_config(pipeline._h, json.dumps(knobs).encode()))


@dataclass
class MetricsSample:
    timestamp_s: float
    ops: list
    sink_polls: int
    sink_empty_polls: int
    sink_empty_ratio: float
    items_emitted: int


def _drain(pipeline, until: float) -> int:
    """Pull batches until the monotonic deadline; returns batches drained
    (the reference's SinkDrainer keeps the sink flowing the same way)."""
    n = 0
    while time.monotonic() < until:
        if pipeline.next_batch_raw() is None:
            raise PcError(K["Shutdown"], "pipeline drained during measurement")
        n += 1
    return n


def collect_metrics(pipeline, interval_ms: int, count: int) -> list:
    """count samples, one per interval, while draining batches
    (collect_metrics, autotune.cpp:19-74)."""
    out = []
    t0 = time.monotonic()
    m0 = metrics(pipeline)
    prev_p, prev_e = m0["sink_polls"], m0["sink_empty_polls"]
    for _ in range(count):
        _drain(pipeline, time.monotonic() + interval_ms / 1e3)
        m = metrics(pipeline)
        dp, de = m["sink_polls"] - prev_p, m["sink_empty_polls"] - prev_e
        ops = [{"op_id": o["op_id"],
                "delay_ms": 1e3 * o["busy_seconds"] / o["items"] if o["items"] else 0.0,
                "queue_utilization": min(1.0, o["out_queue_size"] / o["out_queue_capacity"])
                if o["out_queue_capacity"] else 0.0} for o in m["ops"]]
        out.append(MetricsSample(time.monotonic() - t0, ops, m["sink_polls"], m["sink_empty_polls"],
                                 de / dp if dp else 0.0, m["items_emitted"]))
        prev_p, prev_e = m["sink_polls"], m["sink_empty_polls"]
    return out


def detect_bottleneck(window: list, threshold: float = 0.3) -> str:
    """'data_side' iff the sink empty ratio over the window exceeds the
    threshold, else 'consumer_side' (autotune.cpp:76-88: needs >= 30 samples)."""
    if len(window) < 30:
        raise PcError(K["OutOfBounds"], f"need >= 30 samples, got {len(window)}")
    polls = window[-1].sink_polls - window[0].sink_polls
    empty = window[-1].sink_empty_polls - window[0].sink_empty_polls
    ratio = empty / polls if polls else 0.0
    return "data_side" if ratio > threshold else "consumer_side"


@dataclass
class SearchSpace:
    slots: tuple = (2, 3, 4, 5, 6)
    wave_batches: tuple = (1, 2, 4, 8, 16, 32, 64)

    def validate(self):
        if not self.slots or not self.wave_batches:
            raise PcError(K["OutOfBounds"], "empty search space")
        if min(self.slots) < 2 or max(self.slots) > 8:
            raise PcError(K["OutOfBounds"], "slots outside [2, 8]")
        if min(self.wave_batches) < 1:
            raise PcError(K["OutOfBounds"], "wave_batches must be >= 1")

    def cardinality(self) -> int:
        return len(self.slots) * len(self.wave_batches)

    def point(self, cfg) -> np.ndarray:
        """min-max normalised coordinates (slots, log2 wave_batches)."""
        s0, s1 = min(self.slots), max(self.slots)
        w0, w1 = math.log2(min(self.wave_batches)), math.log2(max(self.wave_batches))
        return np.array([(cfg.slots - s0) / max(1, s1 - s0),
                         (math.log2(cfg.wave_batches) - w0) / max(1e-9, w1 - w0)])


@dataclass
class TuneConfig:
    slots: int
    wave_batches: int
    objective: float = 0.0

    def same_assignment(self, o) -> bool:
        return self.slots == o.slots and self.wave_batches == o.wave_batches


@dataclass
class SurrogateState:
    observed: list = field(default_factory=list)
    length_scale: float = 0.35
    signal_variance: float = 1.0
    noise: float = 1e-3

    def best_objective(self) -> float:
        return max((c.objective for c in self.observed), default=0.0)


def _gp_posterior(state: SurrogateState, space: SearchSpace, cand: np.ndarray):
    X = np.array([space.point(c) for c in state.observed])
    y = np.array([c.objective for c in state.observed], dtype=np.float64)
    mu0, sd0 = y.mean(), y.std() or 1.0
    yn = (y - mu0) / sd0

    def k(a, b):
        d2 = ((a[:, None, :] - b[None, :, :]) ** 2).sum(-1)
        return state.signal_variance * np.exp(-0.5 * d2 / state.length_scale ** 2)

    Kxx = k(X, X) + state.noise * np.eye(len(X))
    L = np.linalg.cholesky(Kxx)
    alpha = np.linalg.solve(L.T, np.linalg.solve(L, yn))
    Ks = k(cand, X)
    mu = Ks @ alpha
    v = np.linalg.solve(L, Ks.T)
    var = np.maximum(state.signal_variance - (v * v).sum(0), 1e-12)
    return mu * sd0 + mu0, np.sqrt(var) * sd0


def propose_config(state: SurrogateState, space: SearchSpace, phase: str, rng: np.random.Generator):
    """'seed': a uniformly random unobserved assignment; 'refine': argmax
    expected improvement over 512 random unobserved candidates
    (propose_config, autotune.cpp:198-283).  OutOfRange when exhausted."""
    space.validate()
    seen = {(c.slots, c.wave_batches) for c in state.observed}
    free = [(s, w) for s in space.slots for w in space.wave_batches if (s, w) not in seen]
    if not free:
        raise PcError(K["OutOfRange"], "search space exhausted")
    if phase == "seed" or len(state.observed) < 2:
        s, w = free[int(rng.integers(len(free)))]
        return TuneConfig(s, w)
    pick = [free[int(i)] for i in rng.integers(len(free), size=min(512, 4 * len(free)))]
    cands = [TuneConfig(s, w) for s, w in dict.fromkeys(pick)]
    P = np.array([space.point(c) for c in cands])
    mu, sd = _gp_posterior(state, space, P)
    best = state.best_objective()
    z = (mu - best) / sd
    cdf = 0.5 * (1.0 + np.vectorize(math.erf)(z / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * z * z) / math.sqrt(2 * math.pi)
    ei = (mu - best) * cdf + sd * pdf
    return cands[int(np.argmax(ei))]


def measure_throughput(pipeline, window_ms: int) -> float:
    """Mean items/s over one window after a one-window warm-up
    (measure_throughput, autotune.cpp:285-297)."""
    _drain(pipeline, time.monotonic() + window_ms / 1e3)
    i0 = metrics(pipeline)["items_emitted"]
    t0 = time.monotonic()
    _drain(pipeline, t0 + window_ms / 1e3)
    dt = time.monotonic() - t0
    return (metrics(pipeline)["items_emitted"] - i0) / dt if dt > 0 else 0.0


def apply_and_measure(pipeline, cfg: TuneConfig, window_ms: int) -> float:
    update_config(pipeline, slots=cfg.slots, wave_batches=cfg.wave_batches)
    return measure_throughput(pipeline, window_ms)


def persist_best(cfg: TuneConfig, path) -> None:
    doc = {"version": 1, "knobs": {"slots": cfg.slots, "wave_batches": cfg.wave_batches},
           "objective": cfg.objective, "timestamp": int(time.time())}
    try:
        with open(path, "w") as f:
            json.dump(doc, f, indent=2)
    except OSError as e:
        raise PcError(K["IoFailure"], f"cannot write {path}: {e}")


def load_best(path) -> TuneConfig:
    try:
        with open(path) as f:
            doc = json.load(f)
    except OSError as e:
        raise PcError(K["IoFailure"], f"cannot read {path}: {e}")
    except ValueError as e:
        raise PcError(K["SchemaMismatch"], f"config file: {e}")
    if doc.get("version") != 1 or "knobs" not in doc:
        raise PcError(K["SchemaMismatch"], "unsupported config version")
    return TuneConfig(int(doc["knobs"]["slots"]), int(doc["knobs"]["wave_batches"]),
                      float(doc.get("objective", 0.0)))


def autotune(pipeline, space: SearchSpace | None = None, iterations: int = 6, seed_phase: int = 3,
             eval_window_ms: int = 300, seed: int = 0):
    """Evaluate candidates on the live pipeline and leave the best applied
    (autotune, autotune.cpp:364-409).  Returns (best, history)."""
    space = space or SearchSpace()
    space.validate()
    rng = np.random.default_rng(seed)
    m = metrics(pipeline)
    cur = TuneConfig(int(m["slots"]), int(m["wave_batches"]))
    cur.objective = measure_throughput(pipeline, eval_window_ms)
    state = SurrogateState(observed=[cur])
    best, history = cur, [cur]
    for _ in range(iterations):
        phase = "seed" if len(state.observed) < seed_phase else "refine"
        try:
            cand = propose_config(state, space, phase, rng)
        except PcError as e:
            if e.errc == "OutOfRange":
                break
            raise
        cand.objective = apply_and_measure(pipeline, cand, eval_window_ms)
        state.observed.append(cand)
        history.append(cand)
        if cand.objective > best.objective:
            best = cand
    update_config(pipeline, slots=best.slots, wave_batches=best.wave_batches)
    return best, history
