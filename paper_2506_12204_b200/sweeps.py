"""Scenario runs and axis sweeps (the reference's ``sweeps.py:13-47`` API).

``run_scenario(cfg)`` is the drop-in single run: ``engine.run`` (every round
on the GPU) plus ``build_report``.

``sweep(base, axis, values)`` keeps the reference's signature and results
but not its loop of one simulation per value. Every value's scenario is
prepared up front (``apply_axis``, native trace generation); scenarios whose
scheduler parameters (``ss_params``: policy, profile, batch size, KV budget,
dependency rule, batch-cost mode, levels) coincide share ONE device launch
-- an axis that only changes trace inputs (seed, ``workload.*``,
``predictor.*``) is a single launch for the whole sweep -- followed by one
batched Eq. 2 audit launch per group. Reports come from the kernel's fused
per-trace statistics, so no per-request data is needed on the host.
"""

from __future__ import annotations

from typing import Any, Dict, List, Sequence, Tuple

import numpy as np

from .config import ConfigError, apply_axis, scenario_to_dict
from .engine import ScenarioConfig, TraceError, run, scenario_params
from .report import RunReport, build_report, report_rows, reports_from_stats


def run_scenario(cfg: ScenarioConfig) -> Tuple[RunReport, Any]:
    trace = run(cfg)
    report = build_report(trace, policy=cfg.policy.value, profile=cfg.profile, seed=cfg.seed,
                          config=scenario_to_dict(cfg))
    return report, trace


def _prepare(cfg: ScenarioConfig):
    from .tracegen import generate_batch

    return generate_batch(cfg.workload, [cfg.workload.seed], cfg.predictor, pred_seeds=[cfg.seed], threads=1)


def _host_sums(stats, res, batch, t: int) -> None:
    """Replace trace t's waiting-time sums by sums in RECORD order over the
    per-request outputs: the kernel's fused sums follow pending order, which
    differs from record order only for hand-made arrival lists."""
    sl = batch.trace_slice(t)
    order = np.argsort(batch.record_pos[sl], kind="stable")
    fin = res.finish_time[sl][order]
    done = ~np.isnan(fin)
    wait = (fin - batch.arrival[sl][order])[done]
    norm = wait / res.generated[sl][order][done].astype(np.float64)
    lv = batch.true_urg[sl][order][done]
    stats["sum_wait"][t] = sum(wait.tolist())  # CPython sum, as the reference
    stats["sum_norm_wait"][t] = sum(norm.tolist())
    for level in range(stats["level_count"].shape[1]):
        stats["level_norm_sum"][t, level] = sum(norm[lv == level].tolist())


def run_scenarios(cfgs: Sequence[ScenarioConfig]) -> List[RunReport]:
    """Reports for many scenarios, one device launch per distinct ss_params."""
    from . import native
    from .metrics import audit_batch
    from .soa import TraceBatch

    groups: Dict[bytes, List[int]] = {}
    params = {}
    for i, cfg in enumerate(cfgs):
        p = scenario_params(cfg)
        key = bytes(p)
        groups.setdefault(key, []).append(i)
        params[key] = p
    reports: List[RunReport] = [None] * len(cfgs)  # type: ignore[list-item]
    for key, idx in groups.items():
        batch = TraceBatch.concat([_prepare(cfgs[i]) for i in idx])
        res = native.run_host(params[key], batch, want_log=False)
        for t in range(len(idx)):
            st = int(res.stats["status"][t])
            if st != 0:
                raise TraceError(st)
        viol, comp = audit_batch(batch, res.finish_time)
        stats = res.stats.copy()
        for t in range(len(idx)):
            sl = batch.trace_slice(t)
            if not np.array_equal(batch.record_pos[sl], np.arange(sl.stop - sl.start)):
                _host_sums(stats, res, batch, t)
        meta = [{"policy": cfgs[i].policy.value, "profile": cfgs[i].profile, "seed": cfgs[i].seed,
                 "config": scenario_to_dict(cfgs[i])} for i in idx]
        for i, rep in zip(idx, reports_from_stats(stats, viol, comp, meta)):
            reports[i] = rep
    return reports


def sweep(base: ScenarioConfig, axis: str, values: Sequence[Any],
          seed_per_value: bool = False) -> Tuple[List[RunReport], List[Dict[str, Any]]]:
    """Run the base scenario once per axis value; with ``seed_per_value``
    run i uses seed + i, otherwise every run shares the base seed."""
    if not values:
        raise ConfigError("sweep needs at least one axis value")
    cfgs = []
    for i, v in enumerate(values):
        cfg = apply_axis(base, axis, str(v))
        if seed_per_value:
            cfg = apply_axis(cfg, "seed", str(base.seed + i))
        cfgs.append(cfg)
    reports = run_scenarios(cfgs)
    rows = [row for v, rep in zip(values, reports) for row in report_rows(rep, axis=axis, axis_value=str(v))]
    return reports, rows
