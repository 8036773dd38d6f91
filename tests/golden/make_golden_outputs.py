"""Golden OUTPUT fixtures: what the reference's metrics, report, CSV and
trace.jsonl writers produce for the golden cases, plus reference sweeps.

Run in the build container (needs /root/reference; the GPU box only reads
the committed fixture):

    python tests/golden/make_golden_outputs.py

For every case of golden_{small,large,anomaly}.json.gz that the reference
finishes, it re-runs the UNMODIFIED reference ``run(cfg, arrivals)`` (no
hooks, fresh process state) and records

* the waiting-time metrics (``metrics.py:35-56``) and ``build_report(...)``
  serialised exactly as ``cli.py:23-25`` writes report.json;
* for traces of at most 300 requests, ``results.csv`` and the sha256 / line
  count of ``trace.jsonl`` as ``cli._write_outputs`` (``cli.py:21-49``)
  writes them (the full text for a few cases, for diagnostics);

and, for a handful of scenario dicts, the outputs of the reference CLI's
``simulate`` and ``sweep`` commands (``cli.py:52-85``; ``sweeps.py:25-47``;
``config.py:119-146``), byte for byte.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import tempfile
import time
from pathlib import Path

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import semsched  # noqa: E402
from semsched import cli as ref_cli  # noqa: E402
from semsched.config import scenario_to_dict  # noqa: E402
from semsched.costs import GpuProfile, BUILTIN_PROFILES  # noqa: E402
from semsched.engine import Policy, ScenarioConfig, run  # noqa: E402
from semsched.metrics import (average_waiting_time, build_report, constraint_audit,  # noqa: E402
                              normalized_waiting_time, overall_normalized_waiting_time)
from semsched.predictors import PredictorConfig, Strategy  # noqa: E402
from semsched.requests import Request, UrgencyLevel  # noqa: E402
from semsched.workload import WorkloadSpec  # noqa: E402

SMALL_MAX = 300
KEEP_TEXT = ("default_200", "mem_a100", "anom_c700_s0")


def cfg_from_params(p):
    wl, pc = p["workload"], p["predictor"]
    prof = p["profile_name"]
    override = None
    if prof not in BUILTIN_PROFILES:
        override = GpuProfile(prof, **p["profile"])
    return ScenarioConfig(
        policy=Policy(p["policy"]), profile=prof, profile_override=override, batch_size=p["batch_size"],
        memory_capacity=p["memory_capacity"],
        workload=WorkloadSpec(total_requests=wl["total_requests"], gap_s=wl["gap_s"], concurrent=wl["concurrent"],
                              concurrent_mode=wl["concurrent_mode"], levels=wl["levels"],
                              prompt_len_range=tuple(wl["prompt_len_range"]),
                              output_len_range=tuple(wl["output_len_range"]), buckets=wl["buckets"],
                              max_output_len=wl["max_output_len"], seed=wl["seed"]),
        predictor=PredictorConfig(latency_s=pc["latency_s"], batch_size=pc["batch_size"],
                                  strategy=Strategy(pc["strategy"]), urgency_error=pc["urgency_error"],
                                  length_error=pc["length_error"]),
        seed=p["seed"], dependency_rule=p["dependency_rule"], decode_batch_cost=p["decode_batch_cost"])


def arrivals_of(case, levels):
    return [Request(id=i, arrival_time=a, prompt_len=pl, true_output_len=o, true_urgency=UrgencyLevel(u, levels))
            for i, a, pl, o, u in case["arrivals"]]


def written(report, trace, rows):
    with tempfile.TemporaryDirectory() as d:
        ref_cli._write_outputs(Path(d), report, trace, rows)
        return {f: (Path(d) / f).read_text() for f in ("report.json", "results.csv", "trace.jsonl")}


def case_outputs(case, group):
    cfg = cfg_from_params(case["params"])
    t0 = time.perf_counter()
    trace = run(cfg, arrivals_of(case, cfg.workload.levels))
    recs = trace.completed_records()
    levels = sorted({r.true_urgency for r in recs})
    viol, rate = constraint_audit(trace)
    report = build_report(trace, policy=cfg.policy.value, profile=cfg.profile, seed=cfg.seed,
                          config=scenario_to_dict(cfg))
    out = {"name": case["name"], "group": group,
           "metrics": {"average_waiting_time": average_waiting_time(trace) if recs else None,
                       "overall_normalized_waiting_time": overall_normalized_waiting_time(trace) if recs else None,
                       "normalized_waiting_time": {str(lv): normalized_waiting_time(trace, lv) for lv in levels},
                       "violations": len(viol), "violation_rate": rate},
           "report_json": json.dumps(report.to_json_obj(), indent=2, sort_keys=True) + "\n"}
    if len(case["arrivals"]) <= SMALL_MAX:
        from semsched.metrics import report_rows

        files = written(report, trace, report_rows(report))
        out["results_csv"] = files["results.csv"]
        out["trace_jsonl_sha256"] = hashlib.sha256(files["trace.jsonl"].encode()).hexdigest()
        out["trace_jsonl_lines"] = files["trace.jsonl"].count("\n")
        if case["name"] in KEEP_TEXT:
            out["trace_jsonl"] = files["trace.jsonl"]
    print(f"{group:8s} {case['name']:28s} {time.perf_counter() - t0:6.2f}s", flush=True)
    return out


# scenario dicts: the reference CLI test's base config, acceptance criterion
# 10's config, a tight-memory one and a mixed custom profile
SCENARIOS = {
    "cli_base": {"policy": "semantic", "profile": "a100_qwen7b", "batch_size": 8, "seed": 3,
                 "workload": {"total_requests": 40, "gap_s": 0.2, "concurrent": 4, "output_len_range": [1, 60]},
                 "predictor": {"latency_s": 0.01}},
    "criterion10": {"policy": "semantic", "profile": "a100_qwen7b", "batch_size": 8, "seed": 11,
                    "workload": {"total_requests": 120, "gap_s": 0.2, "concurrent": 5,
                                 "output_len_range": [1, 120]},
                    "predictor": {"latency_s": 0.01, "urgency_error": 0.3, "length_error": 0.3}},
    "tight": {"policy": "semantic", "profile": "a5000_qwen7b", "batch_size": 16, "seed": 5,
              "memory_capacity": 1200,
              "workload": {"total_requests": 150, "gap_s": 0.1, "concurrent": 8, "levels": 3}},
    "custom": {"policy": "semantic", "profile": "lab_gpu", "batch_size": 4, "seed": 2, "memory_capacity": 900,
               "custom_profile": {"alpha1": 5e-5, "alpha2": 1e-4, "gamma1": 1e-5, "gamma2": 1e-3,
                                  "beta_load": 5e-3, "beta_save": 5e-3},
               "workload": {"total_requests": 60, "concurrent": 3, "output_len_range": [1, 80]}},
}

SWEEPS = [
    ("cli_base", "predictor.urgency_error", ["0.0", "0.3", "0.6"], False),
    ("cli_base", "memory_capacity", ["1000000000", "600", "300"], False),
    ("cli_base", "policy", ["semantic", "fcfs", "sjf", "hpjf"], False),
    ("criterion10", "seed", ["11", "12", "13"], True),
    ("tight", "workload.total_requests", ["50", "100", "150"], False),
    ("custom", "batch_size", ["1", "4", "32"], False),
    ("custom", "decode_batch_cost", ["max", "sum"], False),
]


def cli_outputs(argv):
    with tempfile.TemporaryDirectory() as d:
        import contextlib
        import io

        out = Path(d) / "out"
        cfgp = Path(d) / "scenario.json"
        cfgp.write_text(json.dumps(argv[0]))
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = ref_cli.main([argv[1], "--config", str(cfgp), *argv[2:], "--out", str(out)])
        files = {p.name: p.read_text() for p in out.iterdir()} if out.exists() else {}
        res = {"rc": rc, "stdout": buf.getvalue()}
        for f, txt in files.items():
            if f == "trace.jsonl":
                res["trace_jsonl_sha256"] = hashlib.sha256(txt.encode()).hexdigest()
                res["trace_jsonl_lines"] = txt.count("\n")
            else:
                res[f] = txt
        return res


def main():
    out = {"reference": "semsched " + semsched.__version__, "python": sys.version.split()[0], "cases": [],
           "simulate": {}, "sweeps": []}
    for group in ("small", "large", "anomaly"):
        with gzip.open(os.path.join(HERE, f"golden_{group}.json.gz"), "rt") as fh:
            cases = json.load(fh)["cases"]
        for c in cases:
            if "ref_error" in c["expected"]:
                continue
            out["cases"].append(case_outputs(c, group))
    for name, d in SCENARIOS.items():
        out["simulate"][name] = {"config": d, **cli_outputs([d, "simulate"])}
    for name, axis, values, spv in SWEEPS:
        extra = ["--axis", axis, "--values", ",".join(values)] + (["--seed-per-value"] if spv else [])
        res = cli_outputs([SCENARIOS[name], "sweep", *extra])
        out["sweeps"].append({"scenario": name, "config": SCENARIOS[name], "axis": axis, "values": values,
                              "seed_per_value": spv, **res})
        print(f"sweep {name} {axis}: rc {res['rc']}", flush=True)
    path = os.path.join(HERE, "golden_outputs.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(out, fh)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
