"""Eq. 2 constraint audit and report assembly vs the reference
(``golden_audit.json.gz`` from ``tests/golden/make_golden_audit.py``).

The pair sweep runs on the device (``ss_audit_host``); pairs (in the
reference's order), rates, ``build_report`` and the CSV rows must match the
reference exactly."""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_2506_12204_b200.engine import RequestRecord, Trace

AUDIT = load_golden("audit")["cases"]


def _trace(case) -> Trace:
    recs = [RequestRecord(id=d[0], arrival_time=d[1], prediction_ready=d[2], first_scheduled=d[3], finish_time=d[4],
                          generated_tokens=d[5], evictions=d[6], true_urgency=d[7], predicted_urgency=d[8],
                          prompt_len=d[9]) for d in case["records"]]
    return Trace(records=recs, unservable=list(case["unservable"]), eviction_count=case["eviction_count"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", AUDIT, ids=[c["name"] for c in AUDIT])
def test_audit_and_report_match_reference(case):
    from paper_2506_12204_b200.metrics import build_report, constraint_audit, emit_csv, report_rows

    tr = _trace(case)
    for rk in ("true", "predicted"):
        pairs, rate = constraint_audit(tr, rk)
        assert [list(p) for p in pairs] == case[f"audit_{rk}"]["pairs"], rk
        assert rate == case[f"audit_{rk}"]["rate"], rk
    rep = build_report(tr, case["report"]["policy"], case["report"]["profile"], case["report"]["seed"],
                       config={"n": len(tr.records)})
    assert json.dumps(rep.to_json_obj()) == json.dumps(case["report"])
    assert emit_csv(report_rows(rep, "b", "16")) == case["csv"]


@pytest.mark.gpu
def test_audit_batch_matches_single_trace_audits():
    """The batched audit over a run_many result equals per-trace audits."""
    from paper_2506_12204_b200.engine import ScenarioConfig, run
    from paper_2506_12204_b200.metrics import audit_batch, constraint_audit
    from paper_2506_12204_b200.soa import TraceBatch, prepare_trace
    from paper_2506_12204_b200.workload import WorkloadSpec, generate
    from paper_2506_12204_b200 import native
    from paper_2506_12204_b200.engine import scenario_params

    parts, traces = [], []
    for s in range(12):
        cfg = ScenarioConfig(seed=s, workload=WorkloadSpec(total_requests=250, seed=s, levels=3))
        parts.append(prepare_trace(generate(cfg.workload), cfg)[0])
        traces.append(run(cfg))
    batch = TraceBatch.concat(parts)
    res = native.run_host(scenario_params(cfg), batch)
    for rk in ("true", "predicted"):
        viol, comp = audit_batch(batch, res.finish_time, rk)
        for t, tr in enumerate(traces):
            pairs, rate = constraint_audit(tr, rk)
            assert viol[t] == len(pairs)
            assert (len(pairs) / comp[t] if comp[t] else 0.0) == rate


def test_audit_rejects_bad_ranking():
    from paper_2506_12204_b200.metrics import constraint_audit

    with pytest.raises(ValueError):
        constraint_audit(Trace(), "bogus")
    assert constraint_audit(Trace(), "true") == ([], 0.0)


@pytest.mark.parametrize("case", AUDIT, ids=[c["name"] for c in AUDIT])
def test_oracle_audit_counts_match_reference(case):
    """The C restatement (bench CPU baseline) gives the reference's counts."""
    from oracle_binding import audit_oracle

    recs = [d for d in case["records"] if d[4] is not None]
    for rk, col in (("true", 7), ("predicted", 8)):
        v, c = audit_oracle([0, len(recs)], [d[4] for d in recs], [d[1] for d in recs], [d[col] for d in recs])
        assert int(v[0]) == len(case[f"audit_{rk}"]["pairs"])
        assert (int(v[0]) / int(c[0]) if c[0] else 0.0) == case[f"audit_{rk}"]["rate"]
