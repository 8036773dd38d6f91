"""Run parameters and result containers shared by every backend caller.

``make_params`` marshals a ``ScenarioConfig``-like description into the POD
``ss_params`` of the C-ABI; ``RunResult`` holds the structure-of-arrays that
come back; ``parse_log`` decodes the per-round ITERATION_END records whose
layout is defined in ``include/semsched_b200.h``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi as A


def make_params(profile, batch_size: int, memory_capacity: int, policy: str = "semantic",
                dependency_rule: bool = True, decode_batch_cost: str = "max", levels: int = 5,
                flags: int = A.SS_FLAG_DIGEST, max_rounds: int = 0, bulk_min: int = 0,
                epilogue_min: int = 0) -> A.ss_params:
    """``profile`` is any object with alpha1..beta_save attributes or a dict."""
    g = (lambda k: profile[k]) if isinstance(profile, dict) else (lambda k: getattr(profile, k))
    if decode_batch_cost not in ("max", "sum"):
        raise ValueError("decode_batch_cost must be 'max' or 'sum'")
    if batch_size < 1:
        raise ValueError("batch size must be >= 1")
    if memory_capacity < 1:
        raise ValueError("memory capacity must be >= 1")
    p = A.ss_params()
    p.profile = A.ss_profile(g("alpha1"), g("alpha2"), g("gamma1"), g("gamma2"),
                             g("beta_load"), g("beta_save"))
    p.memory_capacity = int(memory_capacity)
    p.batch_size = int(batch_size)
    p.policy = A.SS_POLICY[policy] if isinstance(policy, str) else int(policy)
    p.dependency_rule = 1 if dependency_rule else 0
    p.decode_cost_sum = 1 if decode_batch_cost == "sum" else 0
    p.levels = int(levels)
    p.flags = int(flags)
    p.max_rounds = int(max_rounds)
    p.bulk_min = int(bulk_min)
    p.epilogue_min = int(epilogue_min)
    return p


@dataclass
class RoundRecord:
    kind: int                   # SS_KIND_*
    granted: np.ndarray         # trace-local slots, batch order
    completed: np.ndarray       # granted order
    mem_used: int
    time: float
    decisions: list             # [victim, action, saved, discarded, freed, ftb, fta]


def parse_log(words: np.ndarray) -> List[RoundRecord]:
    w = np.asarray(words, dtype=np.uint32)
    out: List[RoundRecord] = []
    i = 0
    n = len(w)
    f64 = lambda lo, hi: float(np.array([int(lo) | (int(hi) << 32)], np.uint64).view(np.float64)[0])
    while i < n:
        kind, m, c, v = (int(x) for x in w[i:i + 4])
        mem = int(w[i + 4]) | (int(w[i + 5]) << 32)
        t = f64(w[i + 6], w[i + 7])
        i += A.SS_LOG_HEADER_WORDS
        decs = []
        for _ in range(v):
            d = w[i:i + A.SS_LOG_DECISION_WORDS]
            decs.append([int(d[0]), int(d[1]), int(d[2]), int(d[3]), int(d[4]),
                         f64(d[5], d[6]), f64(d[7], d[8])])
            i += A.SS_LOG_DECISION_WORDS
        g = w[i:i + m].astype(np.int64)
        i += m
        cc = w[i:i + c].astype(np.int64)
        i += c
        out.append(RoundRecord(kind, g, cc, mem, t, decs))
    return out


@dataclass
class RunResult:
    first_scheduled: np.ndarray
    finish_time: np.ndarray
    generated: np.ndarray
    evictions: np.ndarray
    f_t: np.ndarray
    state: np.ndarray
    stats: np.ndarray                       # structured, stats_dtype()
    unservable: List[np.ndarray]            # per trace, trace-local slots
    logs: Optional[List[np.ndarray]] = None  # per trace, uint32 words
    kernel_ms: Optional[float] = None
    extra: dict = field(default_factory=dict)

    def rounds(self, t: int) -> List[RoundRecord]:
        if self.logs is None:
            raise ValueError("run had no round log (SS_FLAG_ROUND_LOG)")
        return parse_log(self.logs[t])


def log_capacity_words(batch, params, scale: int = 1) -> np.ndarray:
    """Per-trace round-log capacity (offsets), generous first guess."""
    sizes = np.diff(batch.offsets).astype(np.int64)
    tokens = np.zeros(len(sizes), np.int64)
    if len(sizes):
        idx = np.repeat(np.arange(len(sizes)), sizes)
        tokens = np.bincount(idx, weights=batch.true_out.astype(np.float64), minlength=len(sizes)).astype(np.int64)
    # rounds <= tokens + prefills (+ eviction rework); each round logs a header,
    # its granted and completed slots; evictions are rare next to that.
    per = (A.SS_LOG_HEADER_WORDS + 2) * (tokens + 2 * sizes) + 64 * sizes + 64
    off = np.zeros(len(sizes) + 1, np.int64)
    np.cumsum(per * scale, out=off[1:])
    return off


def alloc_host_outputs(n_req: int, n_traces: int):
    return dict(
        first_scheduled=np.full(n_req, np.nan), finish_time=np.full(n_req, np.nan),
        generated=np.zeros(n_req, np.uint32), evictions=np.zeros(n_req, np.uint32),
        f_t=np.zeros(n_req, np.float64), state=np.zeros(n_req, np.uint32),
        stats=np.zeros(n_traces, A.stats_dtype()), unservable=np.zeros(max(n_req, 1), np.uint32),
    )


def collect(batch, outs, log=None, log_off=None, kernel_ms=None) -> RunResult:
    st = outs["stats"]
    unserv = []
    for t in range(batch.n_traces):
        o = int(batch.offsets[t])
        unserv.append(outs["unservable"][o:o + int(st["unservable"][t])].astype(np.int64))
    logs = None
    if log is not None:
        logs = [log[int(log_off[t]):int(log_off[t]) + int(st["log_words"][t])] for t in range(batch.n_traces)]
    return RunResult(first_scheduled=outs["first_scheduled"], finish_time=outs["finish_time"],
                     generated=outs["generated"], evictions=outs["evictions"], f_t=outs["f_t"],
                     state=outs["state"], stats=st, unservable=unserv, logs=logs, kernel_ms=kernel_ms)
