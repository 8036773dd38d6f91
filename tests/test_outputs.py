"""Reports, CSV rows, trace.jsonl, config overrides, sweeps and the CLI
against the REFERENCE's own outputs (tests/golden/make_golden_outputs.py
ran the unmodified semsched package on the golden cases and scenarios).

CPU tests pin the host-side writers (config echo, report rows, CSV) from the
fixture alone; GPU tests run every case through the device path and compare
the files byte for byte, and the fused device statistics within 1e-6
relative (north_star's floating-point tolerance; they are in fact equal)."""

from __future__ import annotations

import gzip
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import HERE, golden_cases
from paper_2506_12204_b200.config import ConfigError, apply_axis, load_scenario, scenario_from_dict, scenario_to_dict
from paper_2506_12204_b200.report import RunReport, emit_csv, parse_csv, report_rows

STATS_RTOL = 1e-6

with gzip.open(os.path.join(HERE, "golden", "golden_outputs.json.gz"), "rt", encoding="utf-8") as _fh:
    OUT = json.load(_fh)
CASES = {c["name"]: c for g in ("small", "large", "anomaly") for c in golden_cases(g)}
OUT_CASES = OUT["cases"]
SMALL_OUT = [c for c in OUT_CASES if "results_csv" in c]


def my_cfg(params):
    from paper_2506_12204_b200.costs import BUILTIN_PROFILES, GpuProfile
    from paper_2506_12204_b200.engine import Policy, ScenarioConfig
    from paper_2506_12204_b200.predictors import PredictorConfig, Strategy
    from paper_2506_12204_b200.workload import WorkloadSpec

    wl, pc = params["workload"], params["predictor"]
    name = params["profile_name"]
    override = None if name in BUILTIN_PROFILES else GpuProfile(name, **params["profile"])
    return ScenarioConfig(
        policy=Policy(params["policy"]), profile=name, profile_override=override, batch_size=params["batch_size"],
        memory_capacity=params["memory_capacity"],
        workload=WorkloadSpec(**{**wl, "prompt_len_range": tuple(wl["prompt_len_range"]),
                                 "output_len_range": tuple(wl["output_len_range"])}),
        predictor=PredictorConfig(latency_s=pc["latency_s"], batch_size=pc["batch_size"],
                                  strategy=Strategy(pc["strategy"]), urgency_error=pc["urgency_error"],
                                  length_error=pc["length_error"]),
        seed=params["seed"], dependency_rule=params["dependency_rule"],
        decode_batch_cost=params["decode_batch_cost"])


def my_arrivals(case, levels):
    from paper_2506_12204_b200 import Request, UrgencyLevel

    return [Request(id=i, arrival_time=a, prompt_len=pl, true_output_len=o, true_urgency=UrgencyLevel(u, levels))
            for i, a, pl, o, u in case["arrivals"]]


def report_of_json(text):
    d = json.loads(text)
    d["per_urgency_norm_wait"] = {int(k): v for k, v in d["per_urgency_norm_wait"].items()}
    return RunReport(**d)


# ---------------------------------------------------------------- CPU -----

@pytest.mark.parametrize("case", OUT_CASES, ids=[c["name"] for c in OUT_CASES])
def test_config_echo_matches_reference(case):
    """scenario_to_dict(cfg) is the report's config echo (config.py:67-113)."""
    want = json.loads(case["report_json"])["config"]
    cfg = my_cfg(CASES[case["name"]]["params"])
    assert json.loads(json.dumps(scenario_to_dict(cfg))) == want
    # and the dict round-trips (the workload seed is the scenario seed)
    again = scenario_from_dict(scenario_to_dict(cfg))
    assert scenario_to_dict(again) == scenario_to_dict(cfg)


@pytest.mark.parametrize("case", SMALL_OUT, ids=[c["name"] for c in SMALL_OUT])
def test_report_rows_and_csv_match_reference(case):
    rep = report_of_json(case["report_json"])
    assert json.dumps(rep.to_json_obj(), indent=2, sort_keys=True) + "\n" == case["report_json"]
    text = emit_csv(report_rows(rep))
    assert text == case["results_csv"]
    rows = parse_csv(text)
    assert [r["urgency"] for r in rows] == sorted(rep.per_urgency_norm_wait)


@pytest.mark.parametrize("sw", OUT["sweeps"], ids=[f"{s['scenario']}-{s['axis']}" for s in OUT["sweeps"]])
def test_apply_axis_matches_reference_echo(sw):
    base = scenario_from_dict(sw["config"])
    reports = json.loads(sw["report.json"])
    assert len(reports) == len(sw["values"])
    for i, (v, want) in enumerate(zip(sw["values"], reports)):
        cfg = apply_axis(base, sw["axis"], v)
        if sw["seed_per_value"]:
            cfg = apply_axis(cfg, "seed", str(base.seed + i))
        assert json.loads(json.dumps(scenario_to_dict(cfg))) == want["config"]


def test_config_errors(tmp_path):
    from paper_2506_12204_b200.cli import main

    base = scenario_from_dict(OUT["simulate"]["cli_base"]["config"])
    with pytest.raises(ConfigError):
        apply_axis(base, "turbo.mode", "1")
    with pytest.raises(ConfigError):
        apply_axis(base, "workload.prompt_len_range", "3")
    with pytest.raises(ConfigError):
        apply_axis(base, "workload.urgency_weights.x", "3")
    with pytest.raises(ValueError):
        apply_axis(base, "batch_size", "many")
    assert apply_axis(base, "dependency_rule", "false").dependency_rule is False
    assert apply_axis(base, "workload.gap_s", "0.5").workload.gap_s == 0.5
    with pytest.raises(ConfigError):
        scenario_from_dict({"policy": "lifo"})
    with pytest.raises(ConfigError):
        scenario_from_dict({"workload": {"gap_s": -1}})
    with pytest.raises(ConfigError):
        scenario_from_dict({"custom_profile": {"alpha1": 1}})
    p = scenario_from_dict({"profile": "lab_gpu", "custom_profile": {"alpha1": 1e-9, "alpha2": 1e-4, "gamma1": 1e-8,
                                                                    "gamma2": 1e-2, "beta_load": 1e-4}}).gpu_profile()
    assert p.name == "lab_gpu" and p.gamma2 == 1e-2 and p.beta_save == 1e-4
    bad = tmp_path / "bad.json"
    bad.write_text('{"policy": "lifo"}')
    assert main(["simulate", "--config", str(bad), "--out", str(tmp_path / "o")]) == 1
    assert main(["simulate", "--config", str(tmp_path / "nope.json"), "--out", str(tmp_path / "o")]) == 1
    lst = tmp_path / "list.json"
    lst.write_text("[1, 2]")
    with pytest.raises(ConfigError):
        load_scenario(str(lst))
    good = tmp_path / "s.json"
    good.write_text(json.dumps(OUT["simulate"]["cli_base"]["config"]))
    assert main(["sweep", "--config", str(good), "--axis", "turbo.mode", "--values", "1",
                 "--out", str(tmp_path / "o")]) == 1


# ---------------------------------------------------------------- GPU -----

def _sha(path):
    return hashlib.sha256(path.read_bytes()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("case", OUT_CASES, ids=[c["name"] for c in OUT_CASES])
def test_dropin_report_and_files_match_reference(case, tmp_path):
    """engine.run -> build_report -> report.json byte-identical; the
    metrics functions equal the reference's; small traces: results.csv and
    trace.jsonl (every event payload, 9-dp decisions, records) byte-identical
    (criterion 10, tests/test_acceptance.py:312-337; cli.py:21-49)."""
    from paper_2506_12204_b200 import metrics
    from paper_2506_12204_b200.cli import write_outputs
    from paper_2506_12204_b200.engine import run
    from paper_2506_12204_b200.report import build_report

    gc = CASES[case["name"]]
    cfg = my_cfg(gc["params"])
    trace = run(cfg, my_arrivals(gc, cfg.workload.levels))
    rep = build_report(trace, policy=cfg.policy.value, profile=cfg.profile, seed=cfg.seed,
                       config=scenario_to_dict(cfg))
    assert json.dumps(rep.to_json_obj(), indent=2, sort_keys=True) + "\n" == case["report_json"]
    m = case["metrics"]
    if m["average_waiting_time"] is not None:
        assert metrics.average_waiting_time(trace) == m["average_waiting_time"]
        assert metrics.overall_normalized_waiting_time(trace) == m["overall_normalized_waiting_time"]
    for lv, v in m["normalized_waiting_time"].items():
        assert metrics.normalized_waiting_time(trace, int(lv)) == v
    if "results_csv" in case:
        write_outputs(tmp_path, rep, trace, report_rows(rep))
        assert (tmp_path / "results.csv").read_text() == case["results_csv"]
        got = (tmp_path / "trace.jsonl").read_text()
        if "trace_jsonl" in case and got != case["trace_jsonl"]:
            a, b = got.splitlines(), case["trace_jsonl"].splitlines()
            k = next(i for i, (x, y) in enumerate(zip(a + [""], b + [""])) if x != y)
            pytest.fail(f"trace.jsonl line {k}: {a[k] if k < len(a) else None!r} != {b[k] if k < len(b) else None!r}")
        assert got.count("\n") == case["trace_jsonl_lines"]
        assert _sha(tmp_path / "trace.jsonl") == case["trace_jsonl_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", OUT_CASES, ids=[c["name"] for c in OUT_CASES])
def test_fused_device_stats_match_reference_metrics(case):
    """The kernel's fused end-of-trace statistics (ss_trace_stats, through
    run_many) against the reference's metrics.py:35-56 on the same trace:
    average waiting time, overall normalized waiting time, per-level
    normalized waiting time and the level average, rel 1e-6."""
    from paper_2506_12204_b200.engine import run_many

    gc = CASES[case["name"]]
    cfg = my_cfg(gc["params"])
    res = run_many(cfg, [my_arrivals(gc, cfg.workload.levels)])
    m = case["metrics"]
    want = json.loads(case["report_json"])
    assert int(res.stats["status"][0]) == 0
    assert int(res.stats["evictions"][0]) == want["evictions"]
    assert int(res.stats["unservable"][0]) == want["unservable"]
    if m["average_waiting_time"] is None:
        assert int(res.stats["completed"][0]) == 0
        return
    np.testing.assert_allclose(res.average_waiting_time()[0], m["average_waiting_time"], rtol=STATS_RTOL, atol=0)
    np.testing.assert_allclose(res.overall_normalized_waiting_time()[0], m["overall_normalized_waiting_time"],
                               rtol=STATS_RTOL, atol=0)
    per = {int(k): v for k, v in m["normalized_waiting_time"].items()}
    for lv in range(16):
        got = res.normalized_waiting_time(lv)[0]
        if lv in per:
            np.testing.assert_allclose(got, per[lv], rtol=STATS_RTOL, atol=0)
        else:
            assert np.isnan(got)
    lvl = [res.normalized_waiting_time(lv)[0] for lv in sorted(per)]
    np.testing.assert_allclose(sum(lvl) / len(lvl), want["overall_norm_wait_level_avg"], rtol=STATS_RTOL, atol=0)


def _cli(tmp_path, config, *argv):
    from paper_2506_12204_b200.cli import main

    cfgp = tmp_path / "scenario.json"
    cfgp.write_text(json.dumps(config))
    out = tmp_path / "out"
    rc = main([argv[0], "--config", str(cfgp), *argv[1:], "--out", str(out)])
    return rc, out


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(OUT["simulate"]))
def test_cli_simulate_files_match_reference(name, tmp_path, capsys):
    want = OUT["simulate"][name]
    rc, out = _cli(tmp_path, want["config"], "simulate")
    assert rc == want["rc"]
    assert capsys.readouterr().out == want["stdout"]
    assert (out / "report.json").read_text() == want["report.json"]
    assert (out / "results.csv").read_text() == want["results.csv"]
    assert _sha(out / "trace.jsonl") == want["trace_jsonl_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("sw", OUT["sweeps"], ids=[f"{s['scenario']}-{s['axis']}" for s in OUT["sweeps"]])
def test_batched_sweep_matches_reference(sw, tmp_path, capsys):
    """sweep() = one launch per distinct ss_params (a trace-input axis is a
    single launch): results.csv and report.json byte-identical to the
    reference's sequential sweep (sweeps.py:25-47)."""
    extra = ["--axis", sw["axis"], "--values", ",".join(sw["values"])] + (["--seed-per-value"] if sw["seed_per_value"]
                                                                          else [])
    rc, out = _cli(tmp_path, sw["config"], "sweep", *extra)
    assert rc == sw["rc"]
    assert (out / "results.csv").read_text() == sw["results.csv"]
    assert (out / "report.json").read_text() == sw["report.json"]


@pytest.mark.gpu
def test_sweep_groups_launches():
    from paper_2506_12204_b200 import native
    from paper_2506_12204_b200.sweeps import sweep

    base = scenario_from_dict(OUT["simulate"]["cli_base"]["config"])
    calls = []
    orig = native.run_host
    native.run_host = lambda p, b, **kw: calls.append(b.n_traces) or orig(p, b, **kw)
    try:
        sweep(base, "predictor.urgency_error", ["0.0", "0.3", "0.6"])
        assert calls == [3]
        calls.clear()
        sweep(base, "memory_capacity", ["1000000000", "600", "600"])
        assert sorted(calls) == [1, 2]
    finally:
        native.run_host = orig


@pytest.mark.gpu
def test_cli_audit_roundtrip(tmp_path, capsys):
    from paper_2506_12204_b200.cli import main

    rc, out = _cli(tmp_path, OUT["simulate"]["cli_base"]["config"], "simulate")
    capsys.readouterr()
    assert main(["audit", "--trace", str(out / "trace.jsonl")]) == 0
    assert "violations=" in capsys.readouterr().out
    lines = [{"kind": "request_record", "id": 0, "arrival": 0.0, "finish": 5.0, "generated_tokens": 5,
              "true_urgency": 3, "predicted_urgency": 3},
             {"kind": "request_record", "id": 1, "arrival": 0.0, "finish": 9.0, "generated_tokens": 5,
              "true_urgency": 0, "predicted_urgency": 0}]
    p = tmp_path / "t.jsonl"
    p.write_text("\n".join(json.dumps(x) for x in lines) + "\n")
    assert main(["audit", "--trace", str(p)]) == 0
    assert "violations=1" in capsys.readouterr().out
