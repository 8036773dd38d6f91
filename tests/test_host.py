"""CPU-side checks: host types, trace preparation, the C-ABI library surface,
cost-model known answers. No GPU needed."""

import math
import os
import re

import numpy as np
import pytest

from conftest import REPO, case_batch, golden_cases, has_reference
from paper_2506_12204_b200 import costs as C
from paper_2506_12204_b200.engine import Policy, ScenarioConfig
from paper_2506_12204_b200.predictors import PredictorConfig, Strategy
from paper_2506_12204_b200.requests import LengthBucket, Request, Stage, UrgencyLevel
from paper_2506_12204_b200.soa import TraceBatch, prepare_trace
from paper_2506_12204_b200.workload import WorkloadSpec, bucketize, generate


# ---- known answers from the reference's own tests (tests/test_costs.py, test_kvcache.py)
def test_cost_known_answers():
    a100 = C.get_profile("a100_qwen7b")
    syn = C.GpuProfile("syn", alpha1=0.0, alpha2=1e-4, gamma1=0.01, gamma2=0.05, beta_load=0.5, beta_save=0.5)
    assert C.prefill_time(100, a100) == pytest.approx(0.019945, rel=1e-9)
    assert C.decode_step_time(100, 1, a100) == pytest.approx(0.0133013, rel=1e-4)
    assert C.decode_total_time(10, 5, syn) == pytest.approx(0.9, rel=1e-12)
    a5000 = C.get_profile("a5000_qwen7b")
    assert not C.should_cache_prefill(1000, a5000)
    assert C.should_cache_prefill(100, a100)
    # Eq. 6 interior optimum lies in {15, 16} for the synthetic profile (test_costs.py:140-143)
    assert C.optimal_save_tokens(10, 50, syn) in (15, 16)


def test_optimal_save_matches_bruteforce_and_oracle():
    from oracle_binding import lib
    import ctypes as Ct
    from paper_2506_12204_b200 import _abi as A

    import random

    rng = random.Random(20240817)
    profiles = list(C.BUILTIN_PROFILES.values()) + [
        C.GpuProfile("syn", 0.0, 1e-4, 0.01, 0.05, 0.5, 0.5),
        C.GpuProfile("flat", 0.0, 1e-4, 0.0, 0.05, 0.2, 0.2),
    ]
    L = lib()
    for _ in range(1000):
        p = rng.choice(profiles)
        n, m = rng.randint(0, 512), rng.randint(0, 512)
        best, best_cost = 0, math.inf
        for s in range(m + 1):
            c = C.resume_cost(n, m, s, p)
            if c <= best_cost:
                best, best_cost = s, c
        assert C.optimal_save_tokens(n, m, p) == best
        sp = A.ss_profile(p.alpha1, p.alpha2, p.gamma1, p.gamma2, p.beta_load, p.beta_save)
        assert L.so_optimal_save_tokens(n, m, Ct.byref(sp)) == best
        for f in ("prefill_time", "decode_total_time"):
            pass
        assert L.so_prefill_time(n, Ct.byref(sp)) == C.prefill_time(n, p)
        assert L.so_decode_total_time(n, m, Ct.byref(sp)) == C.decode_total_time(n, m, p)


def test_python_sum_is_neumaier_in_oracle():
    from oracle_binding import lib

    xs = np.array([1e16, 1.0, -1e16, 0.1, 0.2, 3.3e-5], np.float64)
    assert lib().so_pysum(xs.ctypes.data, len(xs)) == sum(xs.tolist())
    rng = np.random.default_rng(0)
    for _ in range(50):
        ys = rng.standard_normal(rng.integers(1, 300)) * 10.0 ** rng.integers(-5, 6)
        assert lib().so_pysum(ys.ctypes.data, len(ys)) == sum(ys.tolist())


# ---- host types mirror the reference's validation
def test_config_validation():
    with pytest.raises(ValueError):
        ScenarioConfig(batch_size=0)
    with pytest.raises(ValueError):
        ScenarioConfig(decode_batch_cost="median")
    with pytest.raises(ValueError):
        ScenarioConfig(memory_capacity=0)
    with pytest.raises(ValueError):
        Request(id=0, arrival_time=0.0, prompt_len=0, true_output_len=1, true_urgency=UrgencyLevel(0))
    with pytest.raises(ValueError):
        UrgencyLevel(5, 5)


def test_bucketize_matches_reference_values():
    assert [bucketize(x, 5, 500).representative_len for x in (0, 99, 100, 250, 499, 500)] == [50, 50, 150, 250, 450, 450]


# ---- trace preparation reproduces the reference's inputs exactly
@pytest.mark.parametrize("group", ["small", "large"])
def test_prepare_trace_matches_golden_inputs(group):
    for case in golden_cases(group):
        p = case["params"]
        if case["name"].startswith("A_") or case["params"]["workload"]["total_requests"] == 0:
            continue
        if case["arrivals"] and case["name"] in ("single_request", "preempt_semantic", "preempt_fcfs",
                                                 "oversized_unservable", "runtime_unservable"):
            arrivals = [Request(id=i, arrival_time=a, prompt_len=pl, true_output_len=o,
                                true_urgency=UrgencyLevel(u, p["levels"])) for i, a, pl, o, u in case["arrivals"]]
        else:
            w = dict(p["workload"])
            w["prompt_len_range"] = tuple(w["prompt_len_range"])
            w["output_len_range"] = tuple(w["output_len_range"])
            arrivals = generate(WorkloadSpec(**w))
        pc = p["predictor"]
        cfg = ScenarioConfig(workload=WorkloadSpec(levels=p["levels"]), seed=p["seed"],
                             predictor=PredictorConfig(latency_s=pc["latency_s"], batch_size=pc["batch_size"],
                                                       strategy=Strategy(pc["strategy"]),
                                                       urgency_error=pc["urgency_error"],
                                                       length_error=pc["length_error"]))
        got, _ = prepare_trace(arrivals, cfg)
        want = case_batch(case)
        for f in ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie", "ids",
                  "record_pos"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), (case["name"], f)


def test_native_generator_matches_python():
    import dataclasses

    from paper_2506_12204_b200.tracegen import generate_batch

    for wkw, pc in ((dict(total_requests=300), PredictorConfig()),
                    (dict(total_requests=150, levels=3, concurrent=7, urgency_weights=[0.5, 0.3, 0.2]),
                     PredictorConfig(latency_s=0.01, urgency_error=0.3, length_error=0.4, batch_size=3)),
                    (dict(total_requests=120, concurrent=9, concurrent_mode="fixed", output_len_range=(1, 120)),
                     PredictorConfig(latency_s=0.05, batch_size=16, strategy=Strategy.FULL_BATCHING,
                                     length_error=0.9))):
        spec = WorkloadSpec(**wkw)
        seeds = list(range(12)) + [2**31 + 5, 2**40 + 3]
        b = generate_batch(spec, seeds, pc)
        parts = []
        for s in seeds:
            cfg = ScenarioConfig(workload=dataclasses.replace(spec, seed=s), predictor=pc, seed=s)
            parts.append(prepare_trace(generate(cfg.workload), cfg)[0])
        ref = TraceBatch.concat(parts)
        for f in ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie", "ids",
                  "record_pos"):
            assert np.array_equal(getattr(b, f), getattr(ref, f)), f


@pytest.mark.skipif(not has_reference(), reason="reference not mounted (GPU box)")
def test_generate_matches_reference_package():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from semsched.workload import WorkloadSpec as RW, generate as rgen

    for seed in (0, 1, 7, 123):
        for kw in (dict(total_requests=200), dict(total_requests=90, levels=3, concurrent=12,
                                                      concurrent_mode="fixed", urgency_weights=[1, 2, 3])):
            mine = generate(WorkloadSpec(seed=seed, **kw))
            ref = rgen(RW(seed=seed, **kw))
            assert [(r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.true_urgency.rank) for r in mine] == \
                   [(r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.true_urgency.rank) for r in ref]


@pytest.mark.skipif(not has_reference(), reason="reference not mounted (GPU box)")
def test_predictors_match_reference_package():
    """Native predictor draws on the caller's Random: same predictions, same
    ready times and the caller's stream left where the reference leaves it."""
    import random
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from semsched import predictors as RP
    from semsched.requests import UrgencyLevel as RU
    from semsched.workload import WorkloadSpec as RW, generate as rgen
    from paper_2506_12204_b200 import predictors as MP

    for seed, kw in ((3, dict(urgency_error=0.4, length_error=0.3)),
                     (5, dict(latency_s=0.05, batch_size=3, strategy="full_batching", urgency_error=1.0)),
                     (9, dict(latency_s=0.3, batch_size=2, length_error=0.9))):
        spec = dict(total_requests=150, seed=seed, levels=4, concurrent=6)
        mine, ref = generate(WorkloadSpec(**spec)), rgen(RW(**spec))
        mk = {**kw, "strategy": Strategy(kw.get("strategy", "immediate"))}
        rk = {**kw, "strategy": RP.Strategy(kw.get("strategy", "immediate"))}
        r1, r2 = random.Random(seed), random.Random(seed)
        a = MP.predictor_pipeline(mine, PredictorConfig(**mk), r1, levels=4)
        b = RP.predictor_pipeline(ref, RP.PredictorConfig(**rk), r2, levels=4)
        assert [(t, r.id, r.f_e.rank, r.predicted_bucket.index, r.predicted_bucket.representative_len)
                for t, r in a] == [(t, r.id, r.f_e.rank, r.predicted_bucket.index,
                                    r.predicted_bucket.representative_len) for t, r in b]
        assert r1.getstate() == r2.getstate()
    # the single-request API
    r1, r2 = random.Random(11), random.Random(11)
    for k in range(300):
        em_m, em_r = MP.ErrorModel(0.5, 5), RP.ErrorModel(0.5, 5)
        assert MP.predict_urgency(UrgencyLevel(k % 5, 5), em_m, r1).rank == \
            RP.predict_urgency(RU(k % 5, 5), em_r, r2).rank
    assert r1.getstate() == r2.getstate()
    r1, r2 = random.Random(12), random.Random(12)
    for k in range(300):
        x = MP.predict_length_bucket(k, MP.ErrorModel(0.3, 400), r1, 7)
        y = RP.predict_length_bucket(k, RP.ErrorModel(0.3, 400), r2, 7)
        assert (x.index, x.representative_len) == (y.index, y.representative_len)
    assert r1.getstate() == r2.getstate()


@pytest.mark.skipif(not has_reference(), reason="reference not mounted (GPU box)")
def test_load_dataset_matches_reference_package(tmp_path):
    import json
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from semsched.workload import WorkloadSpec as RW, load_dataset as rload
    from paper_2506_12204_b200.workload import load_dataset

    lines = [json.dumps({"id": i, "prompt_tokens": 10 + i, "urgency": i % 3, "output_tokens": 5 + i}) for i in range(40)]
    lines[3] = "{not json"
    lines[7] = json.dumps({"id": 7, "urgency": 9, "output_tokens": 4, "prompt_tokens": 3})
    lines[9] = json.dumps({"id": 9, "urgency": 1, "output_tokens": 4, "prompt": "a b c d"})
    lines[11] = json.dumps({"id": 11, "urgency": 1, "output_tokens": 4})
    lines[12] = json.dumps({"urgency": 1, "output_tokens": 4})
    lines[13] = json.dumps({"id": 13, "urgency": 1, "output_tokens": 0, "prompt_tokens": 2})
    lines[14] = ""
    p = tmp_path / "d.jsonl"
    p.write_text("\n".join(lines) + "\n")
    for kw in (dict(levels=3, seed=4), dict(levels=3, seed=5, concurrent=3, concurrent_mode="fixed", gap_s=0.5)):
        a, ea = load_dataset(str(p), WorkloadSpec(**kw))
        b, eb = rload(str(p), RW(**kw))
        assert ea == eb
        assert [(r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.true_urgency.rank) for r in a] == \
               [(r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.true_urgency.rank) for r in b]


# ---- the C-ABI library: loads without a GPU and exports every declared symbol
def _declared_symbols():
    syms = set()
    for h in os.listdir(os.path.join(REPO, "include")):
        txt = open(os.path.join(REPO, "include", h)).read()
        syms |= set(re.findall(r"^\s*(?:int|const char\*|double|int64_t)\s+(ss_\w+)\s*\(", txt, re.M))
    return syms


def test_library_exports_every_declared_symbol():
    from paper_2506_12204_b200 import native

    L = native.lib()
    declared = _declared_symbols()
    assert {"ss_run_traces", "ss_run_traces_host", "ss_generate_traces"} <= declared
    for s in declared:
        assert hasattr(L, s), s


def test_no_cpu_fallback_without_device():
    import torch

    from paper_2506_12204_b200 import native
    from paper_2506_12204_b200.engine import run

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(native.NativeUnavailable):
        native.device_info()
    with pytest.raises((native.NativeUnavailable, native.SchedulerError)):
        run(ScenarioConfig(workload=WorkloadSpec(total_requests=5)))
