"""Drop-in ``run`` / ``Simulator`` backed by the CUDA scheduler.

Same names, arguments, return types and error behaviour as the reference's
``semsched.engine`` (``/root/reference/pkg/src/semsched/engine.py:40-450``):

* ``run(cfg, arrivals=None) -> Trace`` generates the workload when
  ``arrivals`` is None, runs the predictor pipeline on the host, then runs
  every scheduler round of the trace on the GPU (``ss_run_traces_host``)
  and rebuilds the reference's ``Trace`` -- records in arrival order, the
  time-sorted event list (ARRIVAL, PREDICTION_READY, ITERATION_END with the
  reference payload, RUN_END), ``unservable`` and ``eviction_count`` -- and
  writes the final per-request state back into the caller's ``Request``
  objects as the reference does.
* ``run_many(cfg, traces)`` is the batched entry the GPU exists for: any
  number of independent traces in one launch, returning per-trace statistics
  (and optionally per-request records).

There is no CPU path: without the extension or a GPU these raise
``NativeUnavailable``.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Any, Dict, List, Optional, Sequence

import numpy as np

from . import _abi as A
from .batching import Batch, BatchKind
from .costs import GpuProfile, decode_step_time, get_profile, prefill_time, reload_time
from .predictors import PredictorConfig
from .requests import Request, Stage
from .workload import WorkloadSpec, generate


class Policy(enum.Enum):
    SEMANTIC = "semantic"
    FCFS = "fcfs"
    SJF = "sjf"
    HPJF = "hpjf"


class EventKind(enum.Enum):
    ARRIVAL = "arrival"
    PREDICTION_READY = "prediction_ready"
    ITERATION_END = "iteration_end"
    RUN_END = "run_end"


_EVENT_ORDER = {EventKind.ARRIVAL: 0, EventKind.PREDICTION_READY: 1, EventKind.ITERATION_END: 2,
                EventKind.RUN_END: 3}


@dataclass
class Event:
    time: float
    kind: EventKind
    payload: Dict[str, Any] = field(default_factory=dict)

    def to_json_obj(self) -> Dict[str, Any]:
        return {"t": round(self.time, 9), "kind": self.kind.value, **self.payload}


@dataclass
class RequestRecord:
    id: int
    arrival_time: float
    prediction_ready: Optional[float]
    first_scheduled: Optional[float]
    finish_time: Optional[float]
    generated_tokens: int
    evictions: int
    true_urgency: int
    predicted_urgency: Optional[int]
    prompt_len: int


@dataclass
class Trace:
    records: List[RequestRecord] = field(default_factory=list)
    events: List[Event] = field(default_factory=list)
    unservable: List[int] = field(default_factory=list)
    eviction_count: int = 0

    def completed_records(self) -> List[RequestRecord]:
        return [r for r in self.records if r.finish_time is not None]


@dataclass(frozen=True)
class ScenarioConfig:
    """engine.py:89-111."""

    policy: Policy = Policy.SEMANTIC
    profile: str = "a100_qwen7b"
    profile_override: Optional[GpuProfile] = None
    batch_size: int = 16
    memory_capacity: int = 10**9
    workload: WorkloadSpec = field(default_factory=WorkloadSpec)
    predictor: PredictorConfig = field(default_factory=PredictorConfig)
    seed: int = 0
    dependency_rule: bool = True
    decode_batch_cost: str = "max"

    def __post_init__(self) -> None:
        if self.batch_size < 1:
            raise ValueError("batch size must be >= 1")
        if self.memory_capacity < 1:
            raise ValueError("memory capacity must be >= 1")
        if self.decode_batch_cost not in ("max", "sum"):
            raise ValueError("decode_batch_cost must be 'max' or 'sum'")

    def gpu_profile(self) -> GpuProfile:
        return self.profile_override or get_profile(self.profile)


def batch_duration(batch: Batch, p: GpuProfile, decode_cost: str = "max") -> float:
    """Host restatement of one round's virtual duration (engine.py:126-149);
    the device computes the same float64 chain per round."""
    if len(batch) == 0:
        raise ValueError("empty batch has no duration")
    total = 0.0
    steps: List[float] = []
    for r in batch.members:
        if r.stage is Stage.DECODING:
            steps.append(decode_step_time(r.prompt_len + r.decoded_tokens + 1, 1, p))
        else:
            total += reload_time(r.kv_host_tokens, p)
            total += prefill_time(r.prompt_len - r.prefilled_tokens, p)
    if steps:
        total += max(steps) if decode_cost == "max" else sum(steps)
    return total


def scenario_params(cfg: ScenarioConfig, flags: int = A.SS_FLAG_DIGEST, max_rounds: int = 0):
    from .results import make_params

    return make_params(cfg.gpu_profile(), cfg.batch_size, cfg.memory_capacity,
                       policy=cfg.policy.value, dependency_rule=cfg.dependency_rule,
                       decode_batch_cost=cfg.decode_batch_cost, levels=cfg.workload.levels,
                       flags=flags, max_rounds=max_rounds)


class TraceError(RuntimeError):
    """A trace the device could not finish (livelock, anomaly, ...)."""

    def __init__(self, status: int):
        super().__init__(f"trace ended with status {A.TRACE_STATUS_NAMES.get(status, status)}")
        self.status = status


_STAGE_BACK = {A.SS_STAGE_WAITING: Stage.WAITING, A.SS_STAGE_DECODING: Stage.DECODING,
               A.SS_STAGE_COMPLETED: Stage.COMPLETED}


class Simulator:
    """Single-run simulation; ``run(cfg)`` is the usual entry (engine.py:152-243)."""

    def __init__(self, cfg: ScenarioConfig, events: bool = True):
        self.cfg = cfg
        self.profile = cfg.gpu_profile()
        self.trace = Trace()
        self.clock = 0.0
        self.requests: List[Request] = []
        self.events = events
        self.last_result = None

    def run(self, arrivals: Optional[List[Request]] = None) -> Trace:
        from . import native
        from .soa import prepare_trace

        cfg = self.cfg
        if arrivals is None:
            arrivals = generate(cfg.workload)
        self.requests = arrivals
        batch, ready = prepare_trace(arrivals, cfg)
        params = scenario_params(cfg)
        res = native.run_host(params, batch, want_log=self.events)
        self.last_result = res
        st = int(res.stats["status"][0])
        if st != A.SS_TRACE_OK:
            raise TraceError(st)
        self.clock = float(res.stats["final_clock"][0])
        tr = self.trace
        tr.eviction_count = int(res.stats["evictions"][0])
        pend = [r for _, r in ready]
        tr.unservable = [pend[int(s)].id for s in res.unservable[0]]
        # write the final state back into the caller's Request objects
        for i, r in enumerate(pend):
            fin = float(res.finish_time[i])
            first = float(res.first_scheduled[i])
            code = int(res.state[i])
            r.finish_time = None if np.isnan(fin) else fin
            r.first_scheduled_time = None if np.isnan(first) else first
            r.decoded_tokens = int(res.generated[i])
            r.evictions = int(res.evictions[i])
            r.f_t = float(res.f_t[i])
            stg = code & 255
            pf = (code >> 8) & 1
            r.prefilled_tokens = r.prompt_len if pf else 0
            if stg in _STAGE_BACK:
                r.stage = _STAGE_BACK[stg]
            elif stg == A.SS_STAGE_UNSERVABLE:
                # _mark_unservable (engine.py:402-412) keeps the stage and the host KV and
                # releases the device KV; bit 9 says the request was DECODING then
                r.stage = Stage.DECODING if (code >> 9) & 1 else Stage.WAITING
                r.kv_device_tokens = 0
                r.kv_host_tokens = 0 if r.stage is Stage.DECODING else r.prefilled_tokens + r.decoded_tokens
                continue
            if r.stage is Stage.DECODING:
                r.kv_device_tokens, r.kv_host_tokens = r.prefilled_tokens + r.decoded_tokens, 0
            elif r.stage is Stage.WAITING:
                r.kv_device_tokens, r.kv_host_tokens = 0, r.prefilled_tokens + r.decoded_tokens
            else:
                r.kv_device_tokens, r.kv_host_tokens = 0, (0 if r.stage is Stage.COMPLETED else r.kv_host_tokens)
        if self.events:
            tr.events = _events(arrivals, ready, pend, res, self.clock)
        else:
            tr.events = [Event(self.clock, EventKind.RUN_END, {})]
        for r in arrivals:
            tr.records.append(RequestRecord(
                id=r.id, arrival_time=r.arrival_time, prediction_ready=r.prediction_ready_time,
                first_scheduled=r.first_scheduled_time, finish_time=r.finish_time,
                generated_tokens=r.decoded_tokens, evictions=r.evictions,
                true_urgency=r.true_urgency.rank, predicted_urgency=r.f_e.rank if r.f_e else None,
                prompt_len=r.prompt_len))
        return tr


def _events(arrivals, ready, pend, res, clock) -> List[Event]:
    ev: List[Event] = [Event(r.arrival_time, EventKind.ARRIVAL, {"ids": [r.id]}) for r in arrivals]
    ev += [Event(t, EventKind.PREDICTION_READY, {"ids": [r.id]}) for t, r in ready]
    for rec in res.rounds(0):
        decisions = [{"victim": pend[d[0]].id, "prefill_action": "offload" if d[1] == 0 else "discard",
                      "decode_saved": d[2], "decode_discarded": d[3], "freed_slots": d[4],
                      "f_t_before": round(d[5], 9), "f_t_after": round(d[6], 9)} for d in rec.decisions]
        if rec.kind == A.SS_KIND_NONE:
            payload = {"ids": [], "mem_used": rec.mem_used, "evictions": decisions}
        else:
            payload = {"ids": sorted(pend[int(s)].id for s in rec.granted),
                       "kind_detail": "decode" if rec.kind == A.SS_KIND_DECODE else "prefill",
                       "mem_used": rec.mem_used,
                       "completed": [pend[int(s)].id for s in rec.completed],
                       "evictions": decisions}
        ev.append(Event(rec.time, EventKind.ITERATION_END, payload))
    ev.append(Event(clock, EventKind.RUN_END, {}))
    ev.sort(key=lambda e: (e.time, _EVENT_ORDER[e.kind]))
    return ev


def run(cfg: ScenarioConfig, arrivals: Optional[List[Request]] = None) -> Trace:
    """Simulate a scenario to completion and return its trace (engine.py:444-450)."""
    return Simulator(cfg).run(arrivals)


@dataclass
class ManyResult:
    """Per-trace outcome of ``run_many``."""

    stats: np.ndarray                 # structured ss_trace_stats per trace
    kernel_ms: float
    result: Any = None                # RunResult when records were requested

    @property
    def decisions(self) -> int:
        return int(self.stats["rounds"].sum())

    def average_waiting_time(self) -> np.ndarray:
        return self.stats["sum_wait"] / np.maximum(self.stats["completed"], 1)

    def overall_normalized_waiting_time(self) -> np.ndarray:
        return self.stats["sum_norm_wait"] / np.maximum(self.stats["completed"], 1)

    def normalized_waiting_time(self, level: int) -> np.ndarray:
        c = self.stats["level_count"][:, level]
        return np.where(c > 0, self.stats["level_norm_sum"][:, level] / np.maximum(c, 1), np.nan)


def run_many(cfg: ScenarioConfig, traces: Sequence, records: bool = False) -> ManyResult:
    """Run many independent traces in one device call.

    ``traces`` is a ``TraceBatch`` (already laid out) or a sequence of
    arrival lists / ``WorkloadSpec``s; each is prepared with ``cfg``'s
    predictor settings."""
    from . import native
    from .soa import TraceBatch, prepare_trace

    if isinstance(traces, TraceBatch):
        batch = traces
    else:
        parts = []
        for tr in traces:
            arr = generate(tr) if isinstance(tr, WorkloadSpec) else tr
            parts.append(prepare_trace(arr, cfg)[0])
        batch = TraceBatch.concat(parts)
    res = native.run_host(scenario_params(cfg), batch, want_log=False)
    return ManyResult(stats=res.stats, kernel_ms=res.kernel_ms, result=res if records else None)
