"""Comparison of a RunResult against a golden (reference-generated) case."""

from __future__ import annotations

import math

import numpy as np

from paper_2506_12204_b200 import _abi as A


def _same_float(a, b):
    if a is None or (isinstance(a, float) and math.isnan(a)):
        return b is None or (isinstance(b, float) and math.isnan(b))
    if b is None:
        return False
    return np.float64(a).tobytes() == np.float64(b).tobytes()


_STAGE = {"waiting": 0, "prefilling": 1, "decoding": 2, "evicted_offloaded": 3,
          "evicted_discarded": 4, "completed": 5}


def check_against_golden(res, case, t: int = 0, batch=None, check_log=True, check_digest=True):
    """Bit-exact comparison; raises AssertionError with the first mismatch."""
    exp = case["expected"]
    inp = case["inputs"]
    n = len(inp["ready"])
    off = int(batch.offsets[t]) if batch is not None else 0
    st = res.stats[t]
    name = case["name"]
    assert int(st["status"]) == A.SS_TRACE_OK, f"{name}: status {int(st['status'])}"
    assert int(st["rounds"]) == exp["rounds"], f"{name}: rounds {int(st['rounds'])} != {exp['rounds']}"
    assert int(st["evictions"]) == exp["eviction_count"], f"{name}: evictions"
    if check_digest:
        assert format(int(st["digest"]), "016x") == exp["digest"], f"{name}: digest"
    assert _same_float(float(st["final_clock"]), exp["final_clock"]), f"{name}: final clock"
    assert int(st["mem_used_peak"]) == exp["mem_used_peak"], f"{name}: peak"
    ids = inp["ids"]
    unserv = [ids[int(s)] for s in res.unservable[t]]
    assert unserv == exp["unservable"], f"{name}: unservable {unserv} != {exp['unservable']}"
    # records are in arrival-list order
    rec_of_slot = inp["record_pos"]
    for slot in range(n):
        rec = exp["records"][rec_of_slot[slot]]
        rid, first, fin, gen, ev, _ready = rec
        assert rid == ids[slot]
        g = off + slot
        assert _same_float(float(res.first_scheduled[g]), first), f"{name}: first_sched id {rid}"
        assert _same_float(float(res.finish_time[g]), fin), f"{name}: finish id {rid}: {res.finish_time[g]!r} vs {fin!r}"
        assert int(res.generated[g]) == gen, f"{name}: generated id {rid}"
        assert int(res.evictions[g]) == ev, f"{name}: evictions id {rid}"
        assert _same_float(float(res.f_t[g]), exp["final_f_t"][rec_of_slot[slot]]), f"{name}: final f_t id {rid}"
    if check_log and exp.get("log") is not None and res.logs is not None:
        got = res.rounds(t)
        want = exp["log"]
        assert len(got) == len(want), f"{name}: {len(got)} logged rounds != {len(want)}"
        for k, (a, b) in enumerate(zip(got, want)):
            assert a.kind == b["kind"], f"{name}: round {k} kind"
            assert list(a.granted) == b["granted"], f"{name}: round {k} granted {list(a.granted)} != {b['granted']}"
            assert list(a.completed) == b["completed"], f"{name}: round {k} completed"
            assert a.mem_used == b["mem_used"], f"{name}: round {k} mem_used"
            assert _same_float(a.time, b["time"]), f"{name}: round {k} time"
            assert len(a.decisions) == len(b["decisions"]), f"{name}: round {k} decisions"
            for x, y in zip(a.decisions, b["decisions"]):
                assert x[:5] == y[:5], f"{name}: round {k} decision {x} != {y}"
                assert _same_float(x[5], y[5]) and _same_float(x[6], y[6]), f"{name}: round {k} decision f_t"


def stats_from_golden(case):
    """Waiting-time aggregates the reference's metrics would report."""
    exp = case["expected"]
    arr = {row[0]: row[1] for row in case["arrivals"]}
    lv = {row[0]: row[4] for row in case["arrivals"]}
    waits, norms, per = [], [], {}
    for rid, first, fin, gen, ev, _ in exp["records"]:
        if fin is None:
            continue
        w = fin - arr[rid]
        waits.append(w)
        norms.append(w / gen)
        per.setdefault(lv[rid], []).append(w / gen)
    return waits, norms, per


def compare_with_oracle(gpu, cpu, batch, stats_rel: float = 0.0):
    """Statuses must agree everywhere; every other field is compared on the
    traces both finished (a reference exception ends a trace mid-round).
    ``stats_rel`` > 0 compares the floating-point waiting-time sums within that
    relative tolerance (the grid-wide end of trace), else bit for bit."""
    assert np.array_equal(gpu.stats["status"], cpu.stats["status"]), "status"
    # a reference exception ends the trace at an observable round (the raising
    # round counts on both sides); a trace the reference would never finish
    # (livelock / round cap) has no observable round count
    obs = (cpu.stats["status"] == 0) | (cpu.stats["status"] == A.SS_TRACE_REF_ERROR)
    assert np.array_equal(gpu.stats["rounds"][obs], cpu.stats["rounds"][obs]), "rounds (incl. reference errors)"
    ok = cpu.stats["status"] == 0
    for k in ("rounds", "evictions", "digest", "completed", "unservable", "mem_used_peak",
              "lost_evictions", "anomalies", "sum_pool", "sum_granted", "sum_victims",
              "sum_resident_evict"):
        assert np.array_equal(gpu.stats[k][ok], cpu.stats[k][ok]), k
    assert np.array_equal(gpu.stats["final_clock"][ok].view(np.uint64), cpu.stats["final_clock"][ok].view(np.uint64))
    for k in ("sum_wait", "sum_norm_wait", "level_norm_sum"):
        if stats_rel > 0:
            np.testing.assert_allclose(gpu.stats[k][ok], cpu.stats[k][ok], rtol=stats_rel, atol=0, err_msg=k)
        else:
            assert np.array_equal(gpu.stats[k][ok].view(np.uint64), cpu.stats[k][ok].view(np.uint64)), k
    assert np.array_equal(gpu.stats["level_count"][ok], cpu.stats["level_count"][ok])
    sizes = np.diff(batch.offsets)
    rmask = np.repeat(ok, sizes)
    for k in ("first_scheduled", "finish_time", "f_t"):
        assert np.array_equal(getattr(gpu, k)[rmask].view(np.uint64), getattr(cpu, k)[rmask].view(np.uint64)), k
    for k in ("generated", "evictions"):
        assert np.array_equal(getattr(gpu, k)[rmask], getattr(cpu, k)[rmask]), k
    for t in np.nonzero(ok)[0]:
        assert np.array_equal(gpu.unservable[t], cpu.unservable[t])
    return int(ok.sum())
