"""CUDA scheduler vs the reference (golden fixtures) and vs the oracle.

Bit-exact: schedules (per-round logs), eviction decisions, unservable lists,
per-request first_scheduled / finish_time (float64 bit patterns),
generated tokens, eviction counts, final f_t, round counts and digests."""

import numpy as np
import pytest

from conftest import case_batch, case_params, golden_cases
from parity_helpers import check_against_golden, compare_with_oracle as _compare_with_oracle
from paper_2506_12204_b200 import _abi as A

pytestmark = pytest.mark.gpu

SMALL = golden_cases("small")
LARGE = golden_cases("large")
ANOM = golden_cases("anomaly")
# both scheduler variants (chunked stretches / one round per step) on every case
VARIANTS = {"chunked": A.SS_FLAG_FORCE_CHUNKED, "perround": A.SS_FLAG_FORCE_PERROUND}
variants = pytest.mark.parametrize("variant", list(VARIANTS))


@pytest.fixture(scope="module")
def native():
    from paper_2506_12204_b200 import native as nat

    nat.device_info()  # raises if no GPU / no extension
    return nat


@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
@variants
def test_gpu_matches_reference_small(native, case, variant):
    batch = case_batch(case)
    res = native.run_host(case_params(case, A.SS_FLAG_DIGEST | VARIANTS[variant]), batch, want_log=True)
    check_against_golden(res, case, batch=batch)


@pytest.mark.parametrize("case", LARGE, ids=[c["name"] for c in LARGE])
@variants
def test_gpu_matches_reference_large(native, case, variant):
    batch = case_batch(case)
    res = native.run_host(case_params(case, A.SS_FLAG_DIGEST | VARIANTS[variant]), batch, want_log=False)
    check_against_golden(res, case, batch=batch)


@pytest.mark.parametrize("case", ANOM, ids=[c["name"] for c in ANOM])
@variants
def test_gpu_matches_reference_stale_entries(native, case, variant):
    batch = case_batch(case)
    res = native.run_host(case_params(case, A.SS_FLAG_DIGEST | VARIANTS[variant]), batch, want_log=True)
    if "ref_error" in case["expected"]:
        assert int(res.stats["status"][0]) == A.SS_TRACE_REF_ERROR
        assert int(res.stats["rounds"][0]) == case["expected"]["rounds_before_error"] + 1
    else:
        check_against_golden(res, case, batch=batch)


def _seeded_batch(n_traces, total, cfg_kw=None, seed0=0):
    from paper_2506_12204_b200.engine import ScenarioConfig
    from paper_2506_12204_b200.soa import TraceBatch, prepare_trace
    from paper_2506_12204_b200.workload import WorkloadSpec, generate

    parts = []
    cfg = None
    for s in range(seed0, seed0 + n_traces):
        cfg = ScenarioConfig(workload=WorkloadSpec(total_requests=total, seed=s, **(cfg_kw or {})), seed=s)
        parts.append(prepare_trace(generate(cfg.workload), cfg)[0])
    return TraceBatch.concat(parts), cfg


@pytest.mark.parametrize("capacity", [10**9, 1500, 700])
@variants
def test_gpu_many_traces_vs_oracle(native, capacity, variant):
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.results import make_params

    batch, cfg = _seeded_batch(96, 300, dict(levels=3))
    p = lambda f=0: make_params(cfg.gpu_profile(), 16, capacity, levels=3, flags=A.SS_FLAG_DIGEST | f)
    gpu = native.run_host(p(VARIANTS[variant]), batch)
    cpu = run_oracle(p(), batch, threads=8)
    assert _compare_with_oracle(gpu, cpu, batch) >= batch.n_traces // 2


@variants
def test_gpu_config_d_sample_vs_oracle(native, variant):
    """Config D at bench shape (1,000 requests, 3 levels, 2,295 slots): heavy
    eviction, lost decisions, stale heap entries and reference exceptions.
    Status and rounds must agree on every trace, everything else where the
    trace finished."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.dist import shard_seeds
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    batch = generate_batch(WorkloadSpec(total_requests=1000, levels=3), shard_seeds(64, 0), pinned=False)
    p = lambda f=0: make_params(get_profile("a100_qwen7b"), 16, 2295, levels=3, flags=A.SS_FLAG_DIGEST | f)
    gpu = native.run_host(p(VARIANTS[variant]), batch)
    cpu = run_oracle(p(), batch, threads=8)
    assert (cpu.stats["status"] == A.SS_TRACE_REF_ERROR).any()  # the sample covers an exception
    _compare_with_oracle(gpu, cpu, batch)


@pytest.mark.parametrize("policy", ["fcfs", "sjf", "hpjf"])
@pytest.mark.parametrize("capacity", [10**9, 900])
def test_gpu_baseline_policies_vs_oracle(native, policy, capacity):
    """FCFS / SJF / HPJF (engine.py:114-123, 256-285), including eviction by
    each policy's key, against the oracle on many traces."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.results import make_params

    batch, cfg = _seeded_batch(48, 250, dict(levels=3), seed0=500)
    for b in (1, 5, 16):
        p = lambda: make_params(cfg.gpu_profile(), b, capacity, policy=policy, levels=3, flags=A.SS_FLAG_DIGEST)
        gpu = native.run_host(p(), batch)
        cpu = run_oracle(p(), batch, threads=8)
        _compare_with_oracle(gpu, cpu, batch)


@pytest.mark.parametrize("prof", ["a100_qwen7b", "a5000_qwen7b", "mixed"])
@pytest.mark.parametrize("b", [1, 7, 16, 32])
def test_gpu_batch_sizes_profiles_vs_oracle(native, prof, b):
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.scenarios import MIXED_PROFILE

    pr = MIXED_PROFILE if prof == "mixed" else get_profile(prof)
    batch, _ = _seeded_batch(24, 200, dict(levels=4, output_len_range=(1, 300)), seed0=100 + b)
    for dep, cost in ((True, "max"), (False, "sum")):
        p = lambda: make_params(pr, b, 800, levels=4, dependency_rule=dep, decode_batch_cost=cost,
                                flags=A.SS_FLAG_DIGEST)
        gpu = native.run_host(p(), batch)
        cpu = run_oracle(p(), batch, threads=8)
        _compare_with_oracle(gpu, cpu, batch)


def test_gpu_round_logs_vs_oracle(native):
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.results import make_params

    batch, cfg = _seeded_batch(8, 150, dict(levels=3))
    gpu = native.run_host(make_params(cfg.gpu_profile(), 8, 600, levels=3), batch, want_log=True)
    cpu = run_oracle(make_params(cfg.gpu_profile(), 8, 600, levels=3, flags=A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG),
                     batch)
    for t in range(batch.n_traces):
        if cpu.stats["status"][t] == 0:
            assert np.array_equal(gpu.logs[t], cpu.logs[t]), t


def test_run_dropin_matches_golden(native):
    """engine.run() rebuilds the reference Trace (records, events, unservable)."""
    from paper_2506_12204_b200 import Request, UrgencyLevel
    from paper_2506_12204_b200.engine import EventKind, Policy, ScenarioConfig, run
    from paper_2506_12204_b200.costs import GpuProfile
    from paper_2506_12204_b200.predictors import PredictorConfig, Strategy
    from paper_2506_12204_b200.workload import WorkloadSpec

    for case in SMALL:
        p = case["params"]
        prof = GpuProfile("x", **p["profile"])
        wl = WorkloadSpec(**{**p["workload"], "prompt_len_range": tuple(p["workload"]["prompt_len_range"]),
                             "output_len_range": tuple(p["workload"]["output_len_range"])})
        pc = p["predictor"]
        cfg = ScenarioConfig(policy=Policy(p["policy"]), profile_override=prof, batch_size=p["batch_size"],
                             memory_capacity=p["memory_capacity"], workload=wl,
                             predictor=PredictorConfig(latency_s=pc["latency_s"], batch_size=pc["batch_size"],
                                                       strategy=Strategy(pc["strategy"]),
                                                       urgency_error=pc["urgency_error"],
                                                       length_error=pc["length_error"]),
                             seed=p["seed"], dependency_rule=p["dependency_rule"],
                             decode_batch_cost=p["decode_batch_cost"])
        arrivals = [Request(id=i, arrival_time=a, prompt_len=pl, true_output_len=o,
                            true_urgency=UrgencyLevel(u, wl.levels)) for i, a, pl, o, u in case["arrivals"]]
        tr = run(cfg, arrivals)
        exp = case["expected"]
        assert len(tr.events) == exp["n_events"], case["name"]
        assert tr.unservable == exp["unservable"]
        assert tr.eviction_count == exp["eviction_count"]
        for rec, want in zip(tr.records, exp["records"]):
            assert rec.id == want[0]
            assert rec.first_scheduled == want[1] and rec.finish_time == want[2], case["name"]
            assert rec.generated_tokens == want[3] and rec.evictions == want[4]
        ends = [e for e in tr.events if e.kind is EventKind.ITERATION_END]
        assert len(ends) == len(exp["log"])
        # the caller's Request objects end in the reference's final stage (runtime
        # unservable requests keep the stage they had when marked, engine.py:402-412)
        assert [r.stage.value for r in arrivals] == exp["final_stage"], case["name"]


# ---- bulk admission: grid-wide radix sort + sorted RUN (ss_prepass.cu) ------

@pytest.mark.parametrize("policy", ["semantic", "fcfs", "sjf", "hpjf"])
@pytest.mark.parametrize("capacity", [10**9, 1500, 700])
def test_gpu_bulk_run_forced_vs_oracle(native, policy, capacity):
    """bulk_min = 1 routes every trace's first admission through the sorted
    RUN (tiny groups, later arrivals interleaving with the RUN, evictions and
    stale entries re-queued next to it); results must not change."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.results import make_params

    batch, cfg = _seeded_batch(64, 300, dict(levels=3), seed0=900)
    p = lambda bm: make_params(cfg.gpu_profile(), 16, capacity, policy=policy, levels=3, flags=A.SS_FLAG_DIGEST,
                               bulk_min=bm)
    gpu = native.run_host(p(1), batch)
    cpu = run_oracle(p(0), batch, threads=8)
    _compare_with_oracle(gpu, cpu, batch)


def _burst_batch(n_traces, n, seed0, levels=5, **kw):
    """Traces whose requests all arrive at t = 0 (config C's shape, small)."""
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    spec = WorkloadSpec(total_requests=n, concurrent=n, concurrent_mode="fixed", levels=levels, **kw)
    return generate_batch(spec, list(range(seed0, seed0 + n_traces)))


@pytest.mark.parametrize("capacity", [10**9, 3000, 600])
def test_gpu_bulk_burst_vs_oracle(native, capacity):
    """Several traces of 2,000 requests at t = 0 (default bulk threshold):
    multi-trace segmented sort, the RUN feeding the FRONT for the whole trace."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params

    batch = _burst_batch(6, 2000, 40)
    p = lambda bm: make_params(get_profile("a100_qwen7b"), 16, capacity, levels=5, flags=A.SS_FLAG_DIGEST,
                               bulk_min=bm)
    gpu = native.run_host(p(0), batch)
    cpu = run_oracle(p(0), batch, threads=8)
    _compare_with_oracle(gpu, cpu, batch)
    off = native.run_host(p(-1), batch)  # bulk path disabled: same results
    assert np.array_equal(off.stats["digest"], gpu.stats["digest"])


def test_gpu_bulk_with_unservable_vs_oracle(native):
    """A bulk group containing unservable requests (prompt + 1 > capacity):
    non-identity pending list, unservable keys sorted behind the RUN."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params

    batch = _burst_batch(3, 1500, 7, levels=3)
    p = make_params(get_profile("a100_qwen7b"), 8, 100, levels=3, flags=A.SS_FLAG_DIGEST, bulk_min=0)
    gpu = native.run_host(p, batch)
    cpu = run_oracle(p, batch, threads=8)
    assert cpu.stats["unservable"].min() > 0
    _compare_with_oracle(gpu, cpu, batch)


def test_gpu_bulk_round_logs_vs_oracle(native):
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params

    batch = _burst_batch(2, 1200, 3, levels=3)
    mk = lambda fl: make_params(get_profile("a5000_qwen7b"), 16, 1800, levels=3,
                                flags=fl)
    gpu = native.run_host(mk(A.SS_FLAG_DIGEST), batch, want_log=True)
    cpu = run_oracle(mk(A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG), batch)
    for t in range(batch.n_traces):
        assert cpu.stats["status"][t] == gpu.stats["status"][t]
        if cpu.stats["status"][t] == 0:
            assert np.array_equal(gpu.logs[t], cpu.logs[t]), t


def test_gpu_pool_100k_capped_vs_oracle(native):
    """Config C's shape at 100k requests: the first 3,000 rounds (round cap)
    agree with the oracle round for round (digest + rounds)."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params

    batch = _burst_batch(1, 100_000, 1)
    p = make_params(get_profile("a100_qwen7b"), 16, 10**9, levels=5, flags=A.SS_FLAG_DIGEST, max_rounds=3000)
    gpu = native.run_host(p, batch)
    cpu = run_oracle(p, batch)
    for k in ("status", "rounds", "digest", "completed"):
        assert gpu.stats[k][0] == cpu.stats[k][0], k
    assert int(gpu.stats["status"][0]) == A.SS_TRACE_ROUND_CAP


@pytest.mark.parametrize("cap,levels,n", [(1200, 5, 800), (700, 4, 500)])
def test_gpu_tight_memory_sweep_vs_oracle(native, cap, levels, n):
    """256 traces per tight budget: thousands of lost decisions and stale heap
    entries; the kernel leaves the stale-entry path when none is left
    (queue_has_stale) and must stay exact."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.dist import shard_seeds
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    batch = generate_batch(WorkloadSpec(total_requests=n, levels=levels), shard_seeds(256, 0, seed0=17))
    p = lambda: make_params(get_profile("a100_qwen7b"), 16, cap, levels=levels, flags=A.SS_FLAG_DIGEST)
    gpu = native.run_host(p(), batch)
    cpu = run_oracle(p(), batch, threads=8)
    assert cpu.stats["anomalies"].sum() > 100
    _compare_with_oracle(gpu, cpu, batch)


# ---- edge cases ---------------------------------------------------------------

def test_gpu_edge_cases_vs_oracle(native):
    """Empty traces between others, a single-request trace, an all-unservable
    trace and a trace whose only servable request is last, in one launch."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.soa import TraceBatch, empty_batch

    base, cfg = _seeded_batch(3, 60, dict(levels=3), seed0=77)
    one = base.subset([0])
    single = TraceBatch(offsets=np.array([0, 1], np.int64), **{f: getattr(one, f)[:1].copy() for f in
                        ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie", "ids",
                         "record_pos")})
    single.tie = np.zeros(1, np.uint32)
    big = base.subset([1])
    big.prompt = np.full_like(big.prompt, 500)          # prompt + 1 > capacity: all unservable
    last = base.subset([2])
    last.prompt = last.prompt.copy()
    last.prompt[:-1] = 500                              # only the last request is servable
    e = empty_batch()
    zero = TraceBatch(offsets=np.array([0, 0], np.int64), **{f: getattr(e, f) for f in
                      ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie", "ids",
                       "record_pos")})  # one trace with no requests
    batch = TraceBatch.concat([zero, single, zero, big, last, zero])
    assert batch.n_traces == 6
    p = lambda: make_params(cfg.gpu_profile(), 4, 300, levels=3, flags=A.SS_FLAG_DIGEST)
    gpu = native.run_host(p(), batch)
    cpu = run_oracle(p(), batch)
    _compare_with_oracle(gpu, cpu, batch)
    assert gpu.stats["unservable"][3] == 60 and gpu.stats["rounds"][3] == 0
    assert gpu.stats["rounds"][0] == 0 and gpu.stats["completed"][1] == 1


def test_gpu_no_traces(native):
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.soa import empty_batch
    from paper_2506_12204_b200.costs import get_profile

    res = native.run_host(make_params(get_profile("a100_qwen7b"), 16, 1000, flags=A.SS_FLAG_DIGEST), empty_batch())
    assert len(res.stats) == 0


@pytest.mark.parametrize("b", [1, 32])
def test_gpu_extreme_batch_sizes_tight_memory(native, b):
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.results import make_params

    batch, cfg = _seeded_batch(32, 250, dict(levels=4), seed0=300 + b)
    for cap in (400, 2000):
        p = lambda: make_params(cfg.gpu_profile(), b, cap, levels=4, flags=A.SS_FLAG_DIGEST)
        _compare_with_oracle(native.run_host(p(), batch), run_oracle(p(), batch, threads=8), batch)


@pytest.mark.parametrize("capacity", [10**9, 700])
def test_gpu_pipelined_host_call_vs_oracle(native, capacity):
    """ss_run_traces_host splits >= 2,048 traces into slices on separate streams
    (uploads, kernels and downloads overlap); results, logs included, must equal
    the oracle's on every trace, across uneven slice boundaries."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    batch = generate_batch(WorkloadSpec(total_requests=40, levels=3), list(range(4099)), pinned=False)
    logs = capacity > 10**6  # tight budgets can livelock a trace (no finite log)
    p = lambda f=0: make_params(get_profile("a100_qwen7b"), 8, capacity, levels=3, flags=A.SS_FLAG_DIGEST | f)
    gpu = native.run_host(p(), batch, want_log=logs)
    cpu = run_oracle(p(A.SS_FLAG_ROUND_LOG if logs else 0), batch, threads=8)
    assert _compare_with_oracle(gpu, cpu, batch) >= batch.n_traces // 2
    if logs:
        for t in range(0, batch.n_traces, 97):
            assert np.array_equal(gpu.logs[t], cpu.logs[t]), t


@variants
def test_gpu_unservable_duplicate_pinned(native, variant):
    """The one documented divergence ("Not emulated"): seed
    2808, 40 requests, b = 8, 400 slots. A request marked unservable mid-round
    keeps a stale duplicate copy in the same batch that the reference keeps
    decoding; the oracle follows the reference into its IllegalTransitionError
    (REF_ERROR), the kernel stops the trace as LIVELOCK. Both report the same
    round count. Pinned so that a change on either side shows up."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    batch = generate_batch(WorkloadSpec(total_requests=40, levels=3), [2808], pinned=False)
    p = lambda: make_params(get_profile("a100_qwen7b"), 8, 400, levels=3, flags=A.SS_FLAG_DIGEST | VARIANTS[variant])
    gpu = native.run_host(p(), batch)
    cpu = run_oracle(p(), batch)
    assert int(cpu.stats["status"][0]) == A.SS_TRACE_REF_ERROR
    assert int(gpu.stats["status"][0]) == A.SS_TRACE_LIVELOCK
    assert int(gpu.stats["rounds"][0]) == int(cpu.stats["rounds"][0])


@pytest.mark.parametrize("b", [4, 8, 16, 32])
@variants
def test_gpu_queued_decoding_candidates_with_length_errors(native, b, variant):
    """Stretches (and chunks) that run while preempted decoding requests wait
    behind a full batch: with predictor length errors members
    decode past their predicted length, their remainder clamps at 1 and their
    f_t grows, so the last member can overtake a queued candidate mid-stretch;
    bursty arrivals (up to 12 per tick) keep preempting members. Every request
    record, round count and digest against the oracle, ample and tight budgets."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.predictors import PredictorConfig
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    spec = WorkloadSpec(total_requests=400, levels=4, concurrent=12, gap_s=0.1)
    batch = generate_batch(spec, np.arange(900 + b, 900 + b + 64),
                           PredictorConfig(length_error=0.5, urgency_error=0.1), threads=4)
    for cap in (10**9, 4000):
        p = lambda f=0: make_params(get_profile("a100_qwen7b"), b, cap, levels=4, flags=A.SS_FLAG_DIGEST | f)
        gpu = native.run_host(p(VARIANTS[variant]), batch)
        cpu = run_oracle(p(), batch, threads=8)
        assert _compare_with_oracle(gpu, cpu, batch) >= batch.n_traces // 2
