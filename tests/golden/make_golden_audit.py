"""Golden fixtures for the constraint audit (Eq. 2) and report assembly,
produced by the REFERENCE (build container only: needs /root/reference).

    python tests/golden/make_golden_audit.py

Traces come from the reference's own ``run`` (all policies, ample and tight
memory, predictor errors so predicted and true ranks differ) and from
synthetic record sets with tied finish times and unfinished requests. Each
case stores the records and the reference's ``constraint_audit`` (both
rankings) and ``build_report`` results.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from semsched.engine import Policy, RequestRecord, ScenarioConfig, Trace, run  # noqa: E402
from semsched.metrics import build_report, constraint_audit, emit_csv, report_rows  # noqa: E402
from semsched.predictors import PredictorConfig  # noqa: E402
from semsched.workload import WorkloadSpec  # noqa: E402


def rec_dump(r):
    return [r.id, r.arrival_time, r.prediction_ready, r.first_scheduled, r.finish_time, r.generated_tokens,
            r.evictions, r.true_urgency, r.predicted_urgency, r.prompt_len]


def case(name, trace, policy="semantic", profile="a100_qwen7b", seed=0):
    out = {"name": name, "records": [rec_dump(r) for r in trace.records], "unservable": list(trace.unservable),
           "eviction_count": trace.eviction_count}
    for rk in ("true", "predicted"):
        v, rate = constraint_audit(trace, rk)
        out[f"audit_{rk}"] = {"pairs": [list(p) for p in v], "rate": rate}
    rep = build_report(trace, policy, profile, seed, config={"n": len(trace.records)})
    out["report"] = rep.to_json_obj()
    out["csv"] = emit_csv(report_rows(rep, "b", "16"))
    return out


def main():
    cases = []
    for i, (pol, cap, err) in enumerate([(Policy.SEMANTIC, 10**9, 0.0), (Policy.SEMANTIC, 1200, 0.3),
                                         (Policy.FCFS, 10**9, 0.0), (Policy.SJF, 1500, 0.2),
                                         (Policy.HPJF, 10**9, 0.4), (Policy.SEMANTIC, 900, 0.5), (Policy.SEMANTIC, 2000, 0.3),
                                         (Policy.SJF, 10**9, 0.5)]):
        cfg = ScenarioConfig(policy=pol, memory_capacity=cap, seed=i,
                             workload=WorkloadSpec(total_requests=300 + 100 * i, seed=i, levels=3),
                             predictor=PredictorConfig(urgency_error=err, length_error=err))
        try:
            tr = run(cfg)
        except Exception as exc:  # the reference's own stale-entry failures
            print("skip", pol, cap, err, type(exc).__name__)
            continue
        cases.append(case(f"run_{pol.value}_{cap}_{err}", tr, pol.value, "a100_qwen7b", i))
    rng = random.Random(7)
    for i in range(8):
        n = rng.choice([1, 2, 10, 60, 400])
        recs = []
        for k in range(n):
            arr = round(rng.random() * 10, 3)
            fin = None if rng.random() < 0.1 else arr + rng.choice([1.0, 2.0, 2.5, rng.random() * 5])
            recs.append(RequestRecord(id=1000 + k, arrival_time=arr, prediction_ready=arr, first_scheduled=arr,
                                      finish_time=fin, generated_tokens=rng.randint(1, 50), evictions=0,
                                      true_urgency=rng.randrange(4), predicted_urgency=rng.randrange(4),
                                      prompt_len=10))
        tr = Trace(records=recs, unservable=[r.id for r in recs if r.finish_time is None])
        cases.append(case(f"synthetic_{i}_{n}", tr))
    out = os.path.join(HERE, "golden_audit.json.gz")
    with gzip.open(out, "wt", encoding="utf-8") as fh:
        json.dump({"cases": cases}, fh)
    print(out, [(c["name"], len(c["audit_true"]["pairs"])) for c in cases])


if __name__ == "__main__":
    main()
