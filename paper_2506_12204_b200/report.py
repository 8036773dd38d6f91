"""Run reports and CSV rows (the reference's ``metrics.py:94-230`` API).

Two producers feed the same ``RunReport``:

* ``build_report(trace, ...)`` -- from one drop-in ``Trace`` (records on the
  host, the Eq. 2 audit on the device), as the reference builds it;
* ``reports_from_stats(...)`` -- from the device's fused per-trace
  statistics (``ss_trace_stats``: CPython-3.12 Neumaier sums in pending
  order, which is record order for generated traces) plus one batched audit
  launch, with no per-request data on the host. ``sweeps.sweep`` uses it.

Both divide the same sums by the same counts, so a sweep row equals the row
the reference writes for that scenario, ``repr`` for ``repr``.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass, field
from typing import Any, Dict, List, Optional

import numpy as np

from .engine import Trace


@dataclass
class RunReport:
    policy: str
    profile: str
    seed: int
    per_urgency_norm_wait: Dict[int, float]
    avg_wait_s: float
    overall_norm_wait_request_avg: float
    overall_norm_wait_level_avg: float
    violations: int
    violation_rate: float
    evictions: int
    unservable: int
    config: Dict[str, Any] = field(default_factory=dict)

    def to_json_obj(self) -> Dict[str, Any]:
        obj = {name: getattr(self, name) for name in self.__dataclass_fields__}
        obj["per_urgency_norm_wait"] = {str(lv): v for lv, v in sorted(self.per_urgency_norm_wait.items())}
        return obj


def _mean(total: float, n: int) -> float:
    return total / n if n else 0.0


def _level_avg(per_level: Dict[int, float]) -> float:
    # Python sum over the levels in ascending order, as the reference's dict
    return _mean(sum(per_level.values()), len(per_level))


def build_report(trace: Trace, policy: str, profile: str, seed: int, config: Optional[Dict[str, Any]] = None,
                 audit_ranking: str = "true") -> RunReport:
    """One run's report (``metrics.py:137-163``)."""
    from .metrics import _completed, constraint_audit, normalized_waiting_time

    done = _completed(trace, require_all=False)
    per_level = {lv: normalized_waiting_time(trace, lv) for lv in sorted({r.true_urgency for r in done})}
    pairs, rate = constraint_audit(trace, audit_ranking)
    waits = [r.finish_time - r.arrival_time for r in done]
    return RunReport(policy=policy, profile=profile, seed=seed, per_urgency_norm_wait=per_level,
                     avg_wait_s=_mean(sum(waits), len(done)),
                     overall_norm_wait_request_avg=_mean(sum(w / r.generated_tokens for w, r in zip(waits, done)),
                                                         len(done)),
                     overall_norm_wait_level_avg=_level_avg(per_level), violations=len(pairs),
                     violation_rate=rate, evictions=trace.eviction_count, unservable=len(trace.unservable),
                     config=config or {})


def reports_from_stats(stats: np.ndarray, violations: np.ndarray, comparable: np.ndarray,
                       meta: List[Dict[str, Any]]) -> List[RunReport]:
    """One report per trace of a batched run: ``stats`` the structured
    ``ss_trace_stats`` rows, ``violations`` / ``comparable`` the audit counts,
    ``meta[t]`` the policy / profile / seed / config echo of trace t."""
    out = []
    for t, m in enumerate(meta):
        st = stats[t]
        n = int(st["completed"])
        per_level = {lv: float(st["level_norm_sum"][lv]) / int(st["level_count"][lv])
                     for lv in range(len(st["level_count"])) if int(st["level_count"][lv])}
        v, c = int(violations[t]), int(comparable[t])
        out.append(RunReport(policy=m["policy"], profile=m["profile"], seed=m["seed"],
                             per_urgency_norm_wait=per_level, avg_wait_s=_mean(float(st["sum_wait"]), n),
                             overall_norm_wait_request_avg=_mean(float(st["sum_norm_wait"]), n),
                             overall_norm_wait_level_avg=_level_avg(per_level), violations=v,
                             violation_rate=v / c if c else 0.0, evictions=int(st["evictions"]),
                             unservable=int(st["unservable"]), config=m.get("config") or {}))
    return out


# CSV: (column, value of a row given the report, the level and the axis)
_COLUMNS = (
    ("policy", lambda r, lv, ax, av: r.policy),
    ("profile", lambda r, lv, ax, av: r.profile),
    ("axis", lambda r, lv, ax, av: ax),
    ("axis_value", lambda r, lv, ax, av: av),
    ("urgency", lambda r, lv, ax, av: lv),
    ("norm_wait_s_per_tok", lambda r, lv, ax, av: repr(r.per_urgency_norm_wait[lv])),
    ("avg_wait_s", lambda r, lv, ax, av: repr(r.avg_wait_s)),
    ("violations", lambda r, lv, ax, av: r.violations),
    ("evictions", lambda r, lv, ax, av: r.evictions),
    ("seed", lambda r, lv, ax, av: r.seed),
)
CSV_HEADER = [name for name, _ in _COLUMNS]
_PARSE = {"urgency": int, "norm_wait_s_per_tok": float, "avg_wait_s": float, "violations": int,
          "evictions": int, "seed": int}


def report_rows(report: RunReport, axis: str = "", axis_value: str = "") -> List[Dict[str, Any]]:
    """One row per urgency level present in the run (``metrics.py:180-200``)."""
    return [{name: get(report, lv, axis, axis_value) for name, get in _COLUMNS}
            for lv in sorted(report.per_urgency_norm_wait)]


def emit_csv(rows: List[Dict[str, Any]]) -> str:
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=CSV_HEADER, lineterminator="\n")
    w.writeheader()
    w.writerows(rows)
    return buf.getvalue()


def parse_csv(text: str) -> List[Dict[str, Any]]:
    return [{k: _PARSE.get(k, str)(row[k]) for k in CSV_HEADER} for row in csv.DictReader(io.StringIO(text))]
