"""Generate golden fixtures by running the REFERENCE scheduler.

Run in the build container (needs /root/reference, which does not exist on
the GPU box):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src,
runs each case through the reference's own ``Simulator.run`` and records,
per case: the prepared inputs (after the reference's predictor pipeline, in
pending order), every RequestRecord, the unservable list, the eviction
count, the number of scheduler rounds, the schedule digest (the same
definition as include/semsched_b200.h, computed here from the reference's
own ITERATION_END events) and, for small cases, the full per-round log.

The only runtime hook is a ``Simulator`` subclass that observes
``_schedule``/``_execute`` and a full-precision replacement of the engine's
JSON helper ``_decision_obj`` (the reference rounds f_t to 9 digits for its
trace.jsonl, engine.py:432-441); no reference file is modified.
"""

from __future__ import annotations

import gzip
import json
import os
import struct
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import semsched  # noqa: E402  (the reference)
from semsched import engine as ref_engine  # noqa: E402
from semsched.costs import GpuProfile as RefProfile  # noqa: E402
from semsched.engine import EventKind, Policy, ScenarioConfig, Simulator  # noqa: E402
from semsched.predictors import PredictorConfig, Strategy  # noqa: E402
from semsched.requests import Request as RefRequest, UrgencyLevel as RefUrg  # noqa: E402
from semsched.workload import WorkloadSpec, generate  # noqa: E402

M64 = (1 << 64) - 1


def mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def term(rnd, tag, idx, v):
    salt = ((((rnd << 24) ^ (tag << 20) ^ idx) & M64) * 0x9E3779B97F4A7C15) & M64
    return mix64((v & M64) ^ salt)


def grant_term(pos, slot):
    return mix64((slot ^ (((pos + 1) * 0xD6E8FEB86659FD93) & M64)) & M64)


def round_mul(rnd):
    return ((2 * rnd + 1) * 0xA0761D6478BD642F) & M64


def decision_term(rnd, d, w0, w1, w2, w3, w4):
    # include/semsched_b200.h ss_decision_term
    wt = mix64((((rnd << 24) ^ d) * 0x8CB92BA72F3D8DD7) & M64) | 1
    v = (0xC2B2AE3D27D4EB4F * (w0 ^ 0x165667B19E3779F9) + 0x27D4EB2F165667C5 * (w1 ^ 0x85EBCA77C2B2AE63)
         + 0x9E3779B185EBCA87 * (w2 ^ 0xFF51AFD7ED558CCD) + 0xC4CEB9FE1A85EC53 * (w3 ^ 0x62A9D9ED799705F5)
         + 0x4CF5AD432745937F * (w4 ^ 0x1B873593CC9E2D51))
    return (wt * v) & M64


def round_fields(rnd, hdr, mem, tbits):
    # include/semsched_b200.h ss_round_fields
    v = (0xD1B54A32D192ED03 * (hdr ^ 0x5851F42D4C957F2D) + 0xAEF17502108EF2D9 * (mem ^ 0x14057B7EF767814F)
         + 0xF1357AEA2E62A9C5 * (tbits ^ 0x2545F4914F6CDD1D))
    return ((2 * rnd + 1) * v) & M64


def fbits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def full_decision(d):
    return {"victim": d.victim_id, "prefill_action": d.prefill_action,
            "decode_saved": d.decode_saved, "decode_discarded": d.decode_discarded,
            "freed_slots": d.freed_slots, "f_t_before": d.f_t_before, "f_t_after": d.f_t_after}


ref_engine._decision_obj = full_decision

# The granted list is local to Simulator._execute; the engine passes it to the
# module-level batch_duration (engine.py:346-347), so observe it there.
_orig_batch_duration = ref_engine.batch_duration
_last_granted = []


def _observing_batch_duration(batch, p, decode_cost="max"):
    _last_granted[:] = [r.id for r in batch.members]
    return _orig_batch_duration(batch, p, decode_cost)


ref_engine.batch_duration = _observing_batch_duration


class Capture(Simulator):
    """Observe every scheduler round of the unmodified engine."""

    def __init__(self, cfg, max_rounds=None):
        super().__init__(cfg)
        self.rounds = []
        self.max_rounds = max_rounds

    def _schedule(self):
        b = super()._schedule()
        self._members = list(b.members)
        self._kind = b.kind
        return b

    def _execute(self, batch):
        n0 = len(self.trace.events)
        _last_granted.clear()
        super()._execute(batch)
        new = self.trace.events[n0:]
        if new:
            ev = new[0]
            granted = list(_last_granted) if ev.payload["ids"] else []
            assert sorted(granted) == ev.payload["ids"]
            self.rounds.append({
                "kind": (0 if ev.payload.get("kind_detail") == "decode" else 1) if granted else 2,
                "granted": granted,
                "completed": list(ev.payload.get("completed", [])),
                "mem_used": ev.payload["mem_used"],
                "time": ev.time,
                "decisions": ev.payload["evictions"],
                "logged": True,
            })
        else:
            self.rounds.append({"kind": 2, "granted": [], "completed": [], "mem_used": self.mem.used,
                                "time": self.clock, "decisions": [], "logged": False})
        if self.max_rounds and len(self.rounds) > self.max_rounds:
            raise RuntimeError("round cap hit (livelock?)")


def profile_dict(p):
    return {k: getattr(p, k) for k in ("alpha1", "alpha2", "gamma1", "gamma2", "beta_load", "beta_save")}


def _params(cfg):
    wl = cfg.workload
    return {
        "policy": cfg.policy.value,
        "profile": profile_dict(cfg.gpu_profile()),
        "profile_name": cfg.profile,
        "batch_size": cfg.batch_size,
        "memory_capacity": cfg.memory_capacity,
        "dependency_rule": cfg.dependency_rule,
        "decode_batch_cost": cfg.decode_batch_cost,
        "levels": wl.levels,
        "seed": cfg.seed,
        "workload": {"total_requests": wl.total_requests, "gap_s": wl.gap_s,
                     "concurrent": wl.concurrent, "concurrent_mode": wl.concurrent_mode,
                     "levels": wl.levels, "prompt_len_range": list(wl.prompt_len_range),
                     "output_len_range": list(wl.output_len_range), "buckets": wl.buckets,
                     "max_output_len": wl.max_output_len, "seed": wl.seed},
        "predictor": {"latency_s": cfg.predictor.latency_s, "batch_size": cfg.predictor.batch_size,
                      "strategy": cfg.predictor.strategy.value,
                      "urgency_error": cfg.predictor.urgency_error,
                      "length_error": cfg.predictor.length_error},
    }


def _inputs(pending, recpos):
    return {
        "ready": [r.prediction_ready_time for r in pending],
        "arrival": [r.arrival_time for r in pending],
        "prompt": [r.prompt_len for r in pending],
        "true_out": [r.true_output_len for r in pending],
        "pred_len": [r.predicted_bucket.representative_len for r in pending],
        "pred_urg": [r.f_e.rank for r in pending],
        "true_urg": [r.true_urgency.rank for r in pending],
        "ids": [r.id for r in pending],
        "record_pos": [recpos[r.id] for r in pending],
    }


def run_case(name, cfg, arrivals_fn, keep_log):
    arrivals = arrivals_fn()
    sim = Capture(cfg, max_rounds=2_000_000)
    t0 = time.perf_counter()
    try:
        trace = sim.run(arrivals)
    except Exception as exc:  # the reference itself fails on this trace
        err = f"{type(exc).__name__}: {exc}"
        dt = time.perf_counter() - t0
        reqs = sim.requests
        pending = sorted(reqs, key=lambda r: (r.prediction_ready_time, r.arrival_time, r.id))
        print(f"{name:28s} REFERENCE RAISED {err} after {len(sim.rounds)} rounds", flush=True)
        return {
            "name": name, "params": _params(cfg),
            "arrivals": [[r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.true_urgency.rank] for r in reqs],
            "inputs": _inputs(pending, {r.id: i for i, r in enumerate(reqs)}),
            "expected": {"ref_error": err, "rounds_before_error": len(sim.rounds)},
            "ref_seconds": dt,
        }
    dt = time.perf_counter() - t0
    reqs = sim.requests
    pending = sorted(reqs, key=lambda r: (r.prediction_ready_time, r.arrival_time, r.id))
    slot = {r.id: i for i, r in enumerate(pending)}
    recpos = {r.id: i for i, r in enumerate(reqs)}
    digest = 0
    log = []
    for k, rd in enumerate(sim.rounds):
        g = [slot[i] for i in rd["granted"]]
        c = [slot[i] for i in rd["completed"]]
        decs = rd["decisions"]
        d = round_fields(k, rd["kind"] | (len(g) << 8) | (len(c) << 24) | (len(decs) << 40), rd["mem_used"],
                         fbits(rd["time"]))
        gh = 0
        for j, s in enumerate(g):
            gh += grant_term(j, s)
        d += (gh & M64) * round_mul(k)
        for j, s in enumerate(c):
            d += term(k, 5, j, s)
        dl = []
        for j, e in enumerate(decs):
            act = 0 if e["prefill_action"] == "offload" else 1
            v = slot[e["victim"]]
            d += decision_term(k, j, v | (act << 32), e["decode_saved"] | (e["decode_discarded"] << 32),
                               e["freed_slots"], fbits(e["f_t_before"]), fbits(e["f_t_after"]))
            dl.append([v, act, e["decode_saved"], e["decode_discarded"], e["freed_slots"],
                       e["f_t_before"], e["f_t_after"]])
        digest = (digest + d) & M64
        if keep_log and rd["logged"]:
            log.append({"kind": rd["kind"], "granted": g, "completed": c, "mem_used": rd["mem_used"],
                        "time": rd["time"], "decisions": dl})
    ends = [e for e in trace.events if e.kind is EventKind.ITERATION_END]
    peak = max((e.payload["mem_used"] for e in ends), default=0)
    wl = cfg.workload
    case = {
        "name": name,
        "params": _params(cfg),
        "arrivals": [[r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.true_urgency.rank]
                     for r in reqs],
        "inputs": _inputs(pending, recpos),
        "expected": {
            "records": [[rec.id, rec.first_scheduled, rec.finish_time, rec.generated_tokens,
                         rec.evictions, rec.prediction_ready] for rec in trace.records],
            "unservable": list(trace.unservable),
            "eviction_count": trace.eviction_count,
            "rounds": len(sim.rounds),
            "digest": format(digest, "016x"),
            "final_clock": sim.clock,
            "mem_used_peak": peak,
            "final_f_t": [r.f_t for r in reqs],
            "final_stage": [r.stage.value for r in reqs],
            "n_events": len(trace.events),
            "log": log if keep_log else None,
        },
        "ref_seconds": dt,
    }
    print(f"{name:28s} rounds={len(sim.rounds):7d} evictions={trace.eviction_count:5d} "
          f"unservable={len(trace.unservable):3d} peak={peak:7d} {dt:6.2f}s", flush=True)
    return case


def scen(**kw):
    base = dict(policy=Policy.SEMANTIC, profile="a100_qwen7b", batch_size=16,
                workload=WorkloadSpec(total_requests=0), predictor=PredictorConfig())
    base.update(kw)
    return ScenarioConfig(**base)


def gen_arrivals(cfg):
    return lambda: generate(cfg.workload)


def explicit(rows):
    def f():
        return [RefRequest(id=i, arrival_time=a, prompt_len=p, true_output_len=o,
                           true_urgency=RefUrg(u)) for i, a, p, o, u in rows]
    return f


def medical(seed=0, n=1000):
    from paper_2506_12204_b200.scenarios import medical_arrivals

    def f():
        return [RefRequest(id=r.id, arrival_time=r.arrival_time, prompt_len=r.prompt_len,
                           true_output_len=r.true_output_len,
                           true_urgency=RefUrg(r.true_urgency.rank, r.true_urgency.levels))
                for r in medical_arrivals(seed=seed, n=n)]
    return f


def ample_peak(cfg, arrivals_fn):
    import dataclasses

    sim = Simulator(dataclasses.replace(cfg, memory_capacity=10**9))
    tr = sim.run(arrivals_fn())
    return max(e.payload["mem_used"] for e in tr.events if e.kind is EventKind.ITERATION_END)


MIXED = RefProfile("mixed", alpha1=5e-5, alpha2=1e-4, gamma1=1e-5, gamma2=1e-3,
                   beta_load=5e-3, beta_save=5e-3)


def cases_small():
    out = []
    wl200 = WorkloadSpec(total_requests=200, seed=1)
    c = scen(workload=wl200, seed=1)
    out.append(("default_200", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=200, seed=1, output_len_range=(1, 200)), batch_size=1, seed=1)
    out.append(("b1_200", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=120, seed=6, output_len_range=(1, 120)), batch_size=4,
             predictor=PredictorConfig(latency_s=0.01, urgency_error=0.3, length_error=0.3), seed=11)
    out.append(("b4_pred_errors", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=160, gap_s=0.5, concurrent=5, concurrent_mode="fixed",
                                   seed=3, output_len_range=(1, 100)),
             predictor=PredictorConfig(latency_s=0.01, batch_size=16, strategy=Strategy.FULL_BATCHING), seed=3)
    out.append(("full_batching", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=160, gap_s=0.5, concurrent=5, concurrent_mode="fixed",
                                   seed=3, output_len_range=(1, 100)),
             predictor=PredictorConfig(latency_s=0.1, batch_size=4), seed=3)
    out.append(("immediate_chunks", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=200, seed=2), batch_size=8, decode_batch_cost="sum")
    out.append(("decode_sum", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=300, seed=9, levels=3), batch_size=32)
    out.append(("b32_levels3", c, gen_arrivals(c), True))
    for pol in (Policy.FCFS, Policy.SJF, Policy.HPJF):
        c = scen(policy=pol, workload=wl200, seed=1)
        out.append((f"policy_{pol.value}", c, gen_arrivals(c), True))
    # reference engine tests (tests/test_engine.py)
    c = scen(batch_size=4, predictor=PredictorConfig(latency_s=0.05))
    out.append(("single_request", c, explicit([(0, 1.0, 80, 12, 2)]), True))
    c = scen(batch_size=1)
    out.append(("preempt_semantic", c, explicit([(0, 0.0, 50, 400, 4), (1, 0.5, 50, 20, 0)]), True))
    c = scen(batch_size=1, policy=Policy.FCFS)
    out.append(("preempt_fcfs", c, explicit([(0, 0.0, 50, 400, 4), (1, 0.5, 50, 20, 0)]), True))
    c = scen(batch_size=4, memory_capacity=200)
    out.append(("oversized_unservable", c, explicit([(0, 0.0, 500, 5, 0), (1, 0.0, 50, 5, 1)]), True))
    c = scen(batch_size=2, memory_capacity=200)
    out.append(("runtime_unservable", c,
                explicit([(0, 0.0, 50, 199, 1), (1, 0.0, 30, 5, 2), (2, 0.3, 40, 10, 0)]), True))
    c = scen(workload=WorkloadSpec(total_requests=80, seed=7, output_len_range=(1, 200)),
             memory_capacity=2000, batch_size=8)
    out.append(("mem_2000", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=60, seed=8, concurrent=10, gap_s=0.05,
                                   prompt_len_range=(64, 128), output_len_range=(50, 200)),
             memory_capacity=1500, batch_size=8)
    out.append(("pressure_1500", c, gen_arrivals(c), True))
    c = scen(workload=WorkloadSpec(total_requests=0))
    out.append(("empty", c, gen_arrivals(c), True))
    # criterion 11 spike at 50% of peak, and at 25%
    spike_wl = WorkloadSpec(total_requests=200, gap_s=0.1, concurrent=20, concurrent_mode="fixed",
                            seed=4, prompt_len_range=(64, 128), output_len_range=(20, 150))
    c = scen(workload=spike_wl, seed=4)
    pk = ample_peak(c, gen_arrivals(c))
    for div in (2, 4):
        import dataclasses
        cc = dataclasses.replace(c, memory_capacity=max(pk // div, 128 + 250))
        out.append((f"spike_peak_div{div}", cc, gen_arrivals(cc), True))
    # memory-constrained (config D shape, small) under three profiles, +no dependency rule
    wl = WorkloadSpec(total_requests=300, seed=5, levels=3)
    c = scen(workload=wl, seed=5)
    pk = ample_peak(c, gen_arrivals(c))
    cap = max(pk // 4, 578)
    import dataclasses
    for tag, kw in (("a100", dict(profile="a100_qwen7b")), ("a5000", dict(profile="a5000_qwen7b")),
                    ("mixed", dict(profile="mixed", profile_override=MIXED)),
                    ("a5000_nodep", dict(profile="a5000_qwen7b", dependency_rule=False)),
                    ("mixed_nodep_sum", dict(profile="mixed", profile_override=MIXED,
                                             dependency_rule=False, decode_batch_cost="sum"))):
        cc = dataclasses.replace(c, memory_capacity=cap, **kw)
        out.append((f"mem_{tag}", cc, gen_arrivals(cc), True))
    # burst (criterion 6 shape, smaller)
    c = scen(profile="a100_qwen4b_adjusted",
             workload=WorkloadSpec(total_requests=300, gap_s=0.1, concurrent=100, concurrent_mode="fixed",
                                   seed=2, output_len_range=(1, 300)), seed=2)
    out.append(("burst_300", c, gen_arrivals(c), True))
    return out


def cases_large():
    import dataclasses
    out = []
    c = scen(workload=WorkloadSpec(total_requests=1000, levels=3), memory_capacity=4096)
    out.append(("A_medical", c, medical(0, 1000), False))
    c = scen(workload=WorkloadSpec(total_requests=1000, seed=0), seed=0)
    out.append(("B_seed0", c, gen_arrivals(c), False))
    c = scen(workload=WorkloadSpec(total_requests=1000, seed=1, levels=3), seed=1)
    pk = ample_peak(c, gen_arrivals(c))
    cap = max(pk // 4, 578)
    for tag, kw in (("a100", dict(profile="a100_qwen7b")), ("a5000", dict(profile="a5000_qwen7b")),
                    ("mixed", dict(profile="mixed", profile_override=MIXED))):
        cc = dataclasses.replace(c, memory_capacity=cap, **kw)
        out.append((f"D_{tag}", cc, gen_arrivals(cc), False))
    c = scen(workload=WorkloadSpec(total_requests=2000, seed=0), seed=0)
    out.append(("E_seed0", c, gen_arrivals(c), False))
    c = scen(profile="a100_qwen4b_adjusted",
             workload=WorkloadSpec(total_requests=1000, gap_s=0.1, concurrent=100, concurrent_mode="fixed",
                                   seed=2, output_len_range=(1, 300)), seed=2)
    out.append(("criterion6_burst", c, gen_arrivals(c), False))
    c = scen(workload=WorkloadSpec(total_requests=2000, seed=3, output_len_range=(1, 200)), batch_size=32,
             predictor=PredictorConfig(urgency_error=0.5), seed=3)
    out.append(("criterion4_b32_err", c, gen_arrivals(c), False))
    return out


def cases_anomaly():
    """Tight-memory traces where an admission that fails after evicting
    leaves a victim that is a later batch member; granting it keeps a stale
    heap entry (duplicates, stale keys) and sometimes crashes the reference."""
    out = []
    for cap, seeds in ((700, (0, 1, 2, 3, 7, 9, 12, 14, 17, 21)), (1500, (8, 20, 32))):
        for sd in seeds:
            c = scen(workload=WorkloadSpec(total_requests=300, seed=sd, levels=3), seed=sd, memory_capacity=cap)
            out.append((f"anom_c{cap}_s{sd}", c, gen_arrivals(c), sd < 4))
    # baseline policies evicting by their own keys under the same pressure
    for pol in (Policy.FCFS, Policy.SJF, Policy.HPJF):
        for b, sd in ((16, 500), (5, 501), (16, 522), (16, 529)):
            c = scen(policy=pol, batch_size=b, workload=WorkloadSpec(total_requests=250, seed=sd, levels=3),
                     seed=sd, memory_capacity=900)
            out.append((f"anom_{pol.value}_b{b}_s{sd}", c, gen_arrivals(c), sd == 500))
    return out


def main():
    which = sys.argv[1:] or ["small", "large", "anomaly"]
    groups = {"small": cases_small, "large": cases_large, "anomaly": cases_anomaly}
    for group in which:
        cases = groups[group]()
        fixtures = [run_case(*c) for c in cases]
        path = os.path.join(HERE, f"golden_{group}.json.gz")
        with gzip.open(path, "wt", encoding="utf-8") as fh:
            json.dump({"reference": "semsched " + semsched.__version__,
                       "python": sys.version.split()[0], "cases": fixtures}, fh)
        print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
