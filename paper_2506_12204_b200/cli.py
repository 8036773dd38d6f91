"""Command line and output files (the reference's ``cli.py``).

    python -m paper_2506_12204_b200 simulate --config scenario.json --out DIR
    python -m paper_2506_12204_b200 sweep --config scenario.json --axis predictor.urgency_error \\
        --values 0.0,0.3 [--seed-per-value] --out DIR
    python -m paper_2506_12204_b200 audit --trace DIR/trace.jsonl [--ranking predicted]

Same subcommands, flags, files and exit codes as ``cli.py:1-151`` (0 ok,
1 configuration error, 2 unservable requests): ``report.json``,
``results.csv`` and ``trace.jsonl`` are byte-identical to the reference's
for the same scenario (``tests/test_outputs.py``). The simulation and the
sweep run on the GPU (``sweeps.py``); the audit's pair sweep too
(``metrics.constraint_audit``).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path
from typing import Iterator, List, Optional

from .config import ConfigError, apply_axis, load_scenario
from .engine import RequestRecord, Trace
from .report import emit_csv, report_rows

# trace.jsonl request_record line: JSON key -> RequestRecord attribute
_RECORD_KEYS = (("id", "id"), ("arrival", "arrival_time"), ("prediction_ready", "prediction_ready"),
                ("first_scheduled", "first_scheduled"), ("finish", "finish_time"),
                ("generated_tokens", "generated_tokens"), ("evictions", "evictions"),
                ("true_urgency", "true_urgency"), ("predicted_urgency", "predicted_urgency"),
                ("prompt_len", "prompt_len"))


def trace_lines(trace: Trace) -> Iterator[str]:
    """trace.jsonl: every event, then one ``request_record`` per record."""
    for ev in trace.events:
        yield json.dumps(ev.to_json_obj(), sort_keys=True)
    for rec in trace.records:
        obj = {key: getattr(rec, attr) for key, attr in _RECORD_KEYS}
        obj["kind"] = "request_record"
        yield json.dumps(obj, sort_keys=True)


def write_outputs(out_dir: Path, report, trace: Trace, rows) -> None:
    """report.json, results.csv and trace.jsonl of one run (``cli.py:21-49``)."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    (out_dir / "report.json").write_text(json.dumps(report.to_json_obj(), indent=2, sort_keys=True) + "\n")
    (out_dir / "results.csv").write_text(emit_csv(rows))
    with open(out_dir / "trace.jsonl", "w", encoding="utf-8") as fh:
        fh.writelines(line + "\n" for line in trace_lines(trace))


def read_trace_records(path: str) -> Trace:
    """The request records of a trace.jsonl (other lines skipped)."""
    trace = Trace()
    optional = {"prediction_ready": None, "first_scheduled": None, "finish": None, "evictions": 0,
                "predicted_urgency": None, "prompt_len": 1}
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            obj = json.loads(line)
            if obj.get("kind") != "request_record":
                continue
            kw = {attr: (obj.get(key, optional[key]) if key in optional else obj[key]) for key, attr in _RECORD_KEYS}
            trace.records.append(RequestRecord(**kw))
    return trace


def _simulate(args) -> int:
    from .sweeps import run_scenario

    cfg = load_scenario(args.config)
    for axis, value in (("policy", args.policy), ("seed", args.seed), ("profile", args.profile)):
        if value is not None and value != "":
            cfg = apply_axis(cfg, axis, str(value))
    report, trace = run_scenario(cfg)
    write_outputs(Path(args.out), report, trace, report_rows(report))
    print(f"policy={report.policy} avg_wait={report.avg_wait_s:.4f}s "
          f"norm_wait={report.overall_norm_wait_request_avg:.4f}s/tok violations={report.violations} "
          f"evictions={report.evictions} unservable={report.unservable}")
    return 2 if report.unservable else 0


def _sweep(args) -> int:
    from .sweeps import sweep

    cfg = load_scenario(args.config)
    reports, rows = sweep(cfg, args.axis, [v for v in args.values.split(",") if v],
                          seed_per_value=args.seed_per_value)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    (out / "results.csv").write_text(emit_csv(rows))
    (out / "report.json").write_text(json.dumps([r.to_json_obj() for r in reports], indent=2, sort_keys=True) + "\n")
    print(f"{len(reports)} runs, {len(rows)} rows -> {out / 'results.csv'}")
    return 2 if any(r.unservable for r in reports) else 0


def _audit(args) -> int:
    from .metrics import constraint_audit

    pairs, rate = constraint_audit(read_trace_records(args.trace), ranking=args.ranking)
    print(f"violations={len(pairs)} rate={rate:.6f}")
    for i, j in pairs[:20]:
        print(f"  finished-first={i} outranked-by={j}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="semsched", description="Priority-aware LLM-serving scheduling simulator")
    sub = ap.add_subparsers(dest="command", required=True)
    s = sub.add_parser("simulate", help="run one scenario")
    s.add_argument("--config", required=True)
    s.add_argument("--policy", choices=["semantic", "fcfs", "sjf", "hpjf"])
    s.add_argument("--seed", type=int)
    s.add_argument("--profile")
    s.add_argument("--out", required=True)
    s.set_defaults(func=_simulate)
    w = sub.add_parser("sweep", help="run a scenario across an axis")
    w.add_argument("--config", required=True)
    w.add_argument("--axis", required=True)
    w.add_argument("--values", required=True, help="comma-separated values")
    w.add_argument("--seed-per-value", action="store_true")
    w.add_argument("--out", required=True)
    w.set_defaults(func=_sweep)
    a = sub.add_parser("audit", help="audit a trace.jsonl for ordering violations")
    a.add_argument("--trace", required=True)
    a.add_argument("--ranking", choices=["true", "predicted"], default="true")
    a.set_defaults(func=_audit)
    return ap


def main(argv: Optional[List[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
