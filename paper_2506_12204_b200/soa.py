"""Structure-of-arrays trace layout shared by the host shim and the device.

A ``TraceBatch`` holds any number of independent traces back to back. Inside
a trace, rows are in the reference's *pending* order — sorted by
(prediction-ready time, arrival time, id) exactly as ``predictor_pipeline``
returns them (``predictors.py:148``) — so admission on the device is a
cursor walk. ``tie`` is each request's rank in (arrival time, id) order, the
tail of the dispatch key (``requests.py:81-91``); ``record_pos`` maps a row
back to the request's position in the caller's arrival list (the order of
``Trace.records``, ``engine.py:228-242``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from ._abi import SS_MAX_TRACE_REQS

FIELDS = ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie")
DTYPES = {"ready": np.float64, "arrival": np.float64, "prompt": np.uint32,
          "true_out": np.uint32, "pred_len": np.uint32, "pred_urg": np.uint8,
          "true_urg": np.uint8, "tie": np.uint32, "ids": np.int64, "record_pos": np.int64}


@dataclass
class TraceBatch:
    offsets: np.ndarray          # int64 [T+1]
    ready: np.ndarray
    arrival: np.ndarray
    prompt: np.ndarray
    true_out: np.ndarray
    pred_len: np.ndarray
    pred_urg: np.ndarray
    true_urg: np.ndarray
    tie: np.ndarray
    ids: np.ndarray              # reference request ids (int64)
    record_pos: np.ndarray       # row -> index in the trace's arrival list

    @property
    def n_traces(self) -> int:
        return len(self.offsets) - 1

    @property
    def n_requests(self) -> int:
        return int(self.offsets[-1])

    def trace_slice(self, t: int) -> slice:
        return slice(int(self.offsets[t]), int(self.offsets[t + 1]))

    def nbytes_inputs(self) -> int:
        """Bytes the device path reads as inputs (the H2D payload)."""
        return int(self.offsets.nbytes + sum(getattr(self, f).nbytes for f in FIELDS))

    def validate(self) -> None:
        sizes = np.diff(self.offsets)
        if (sizes < 0).any():
            raise ValueError("trace offsets must be nondecreasing")
        if sizes.size and sizes.max() >= SS_MAX_TRACE_REQS:
            raise ValueError(f"a trace exceeds {SS_MAX_TRACE_REQS - 1} requests")
        if (self.prompt < 1).any() or (self.true_out < 1).any():
            raise ValueError("lengths must be >= 1")

    def subset(self, traces: Sequence[int]) -> "TraceBatch":
        """A new batch holding the listed traces, in that order."""
        parts = []
        for t in traces:
            s = self.trace_slice(int(t))
            kw = {f: getattr(self, f)[s] for f in FIELDS + ("ids", "record_pos")}
            parts.append(TraceBatch(offsets=np.array([0, s.stop - s.start], np.int64), **kw))
        return TraceBatch.concat(parts)

    @staticmethod
    def concat(batches: Sequence["TraceBatch"]) -> "TraceBatch":
        offs = [np.zeros(1, np.int64)]
        base = 0
        for b in batches:
            offs.append(b.offsets[1:] + base)
            base += b.n_requests
        kw = {f: np.concatenate([getattr(b, f) for b in batches]) for f in FIELDS + ("ids", "record_pos")}
        return TraceBatch(offsets=np.concatenate(offs), **kw)


def tie_ranks(arrival: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """Rank of (arrival, id) within one trace."""
    order = np.lexsort((ids, arrival))
    tie = np.empty(len(order), np.uint32)
    tie[order] = np.arange(len(order), dtype=np.uint32)
    return tie


def from_prepared(arrivals: Sequence, ready: Sequence[Tuple[float, object]]) -> TraceBatch:
    """One trace from ``Request`` objects after ``predictor_pipeline``.

    ``arrivals`` is the caller's list (record order); ``ready`` the
    pipeline's (ready_time, request) list (pending order)."""
    pos = {id(r): i for i, r in enumerate(arrivals)}
    n = len(ready)
    rd = np.fromiter((t for t, _ in ready), np.float64, n)
    reqs = [r for _, r in ready]
    arr = np.fromiter((r.arrival_time for r in reqs), np.float64, n)
    ids = np.fromiter((r.id for r in reqs), np.int64, n)
    tb = TraceBatch(
        offsets=np.array([0, n], np.int64),
        ready=rd,
        arrival=arr,
        prompt=np.fromiter((r.prompt_len for r in reqs), np.uint32, n),
        true_out=np.fromiter((r.true_output_len for r in reqs), np.uint32, n),
        pred_len=np.fromiter((r.predicted_bucket.representative_len for r in reqs), np.uint32, n),
        pred_urg=np.fromiter((r.f_e.rank for r in reqs), np.uint8, n),
        true_urg=np.fromiter((r.true_urgency.rank for r in reqs), np.uint8, n),
        tie=tie_ranks(arr, ids),
        ids=ids,
        record_pos=np.fromiter((pos[id(r)] for r in reqs), np.int64, n),
    )
    return tb


def empty_batch() -> TraceBatch:
    z = {f: np.zeros(0, DTYPES[f]) for f in FIELDS + ("ids", "record_pos")}
    return TraceBatch(offsets=np.zeros(1, np.int64), **z)


def prepare_trace(arrivals: List, cfg) -> Tuple[TraceBatch, list]:
    """Run the reference-semantics predictor pipeline on ``arrivals`` (which
    it mutates, like the reference) and lay the trace out as SoA."""
    import random

    from .predictors import predictor_pipeline

    rng = random.Random(cfg.seed)
    ready = predictor_pipeline(arrivals, cfg.predictor, rng, levels=cfg.workload.levels,
                               buckets=cfg.workload.buckets,
                               max_output_len=cfg.workload.max_output_len)
    return from_prepared(arrivals, ready), ready
