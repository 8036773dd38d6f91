"""The per-step API (batching.extract_top_b / stage_aware_schedule,
kvcache.priority_based_eviction / should_recompute) against the reference.

GPU tests replay ``golden_step.json.gz`` (made by the reference itself,
``tests/golden/make_golden_step.py``): the same state goes through this
package's device-backed functions and everything observable afterwards must
be identical — batch, decisions (f64 bit patterns), exceptions, every
request's fields and both heaps' (id, stored key) contents. CPU tests cover
the host containers, mirroring the reference's test_heaps.py."""

import random

import numpy as np
import pytest

from conftest import load_golden
from paper_2506_12204_b200 import _abi as A
from paper_2506_12204_b200.costs import GpuProfile, get_profile
from paper_2506_12204_b200.heaps import (ArrivalBuffer, DispatchQueue, DuplicateRequestError, EmptyQueueError,
                                         EvictionQueue, IndexedMinHeap, NotFoundError)
from paper_2506_12204_b200.requests import LengthBucket, Request, Stage, UrgencyLevel

STEP = load_golden("step")["cases"]
PROFILES = {"a100_qwen7b": get_profile("a100_qwen7b"), "a5000_qwen7b": get_profile("a5000_qwen7b"),
            "mixed": GpuProfile("mixed", alpha1=5e-5, alpha2=1e-4, gamma1=1e-5, gamma2=1e-3, beta_load=5e-3,
                                beta_save=5e-3)}


def _req(d) -> Request:
    rid, arr, prompt, out, fe, mid, ft, pf, dec, kvd, kvh, stage, ev = d
    r = Request(id=rid, arrival_time=arr, prompt_len=prompt, true_output_len=out, true_urgency=UrgencyLevel(fe),
                f_e=UrgencyLevel(fe), predicted_bucket=LengthBucket(0, mid), f_t=ft)
    r.prefilled_tokens, r.decoded_tokens, r.kv_device_tokens, r.kv_host_tokens = pf, dec, kvd, kvh
    r.stage, r.evictions = Stage(stage), ev
    return r


def _dump(r):
    return [r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.f_e.rank, r.predicted_bucket.representative_len,
            r.f_t, r.prefilled_tokens, r.decoded_tokens, r.kv_device_tokens, r.kv_host_tokens, r.stage.value,
            r.evictions]


def _heap_dump(q):
    return sorted([[r.id, list(k)] for r, k in zip(q._heap._items, q._heap._keys)])


def _fill(q, dump, by_id):
    for rid, key in dump:
        q._heap.insert(by_id[rid], tuple(key))


def _same(a, b):
    """Exact equality including float bit patterns (JSON floats round-trip)."""
    return json_canon(a) == json_canon(b)


def json_canon(x):
    import json

    return json.dumps(x)


# ---- GPU: replay the reference's per-step results -----------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in STEP if c["fn"] in ("extract_top_b", "stage_aware_schedule")],
                         ids=lambda c: c["name"])
def test_select_matches_reference(case):
    from paper_2506_12204_b200 import batching as B

    st = case["state"]
    reqs = [_req(d) for d in st["requests"]]
    by_id = {r.id: r for r in reqs}
    h, u = DispatchQueue(), ArrivalBuffer()
    _fill(h, st["heap"], by_id)
    for rid in st["buffer"]:
        u.append(by_id[rid])
    ongoing = [by_id[rid] for rid in st["ongoing"]]
    res = case["result"]
    if case["fn"] == "extract_top_b":
        got = B.extract_top_b(h, u, case["b"])
        assert [r.id for r in got] == res["popped"]
    else:
        batch = B.stage_aware_schedule(h, u, ongoing, case["b"])
        assert batch.kind.value == res["kind"]
        assert [r.id for r in batch.members] == res["members"]
    assert len(u) == 0
    assert _same(_heap_dump(h), res["heap_after"])
    assert _same([_dump(r) for r in reqs], res["requests_after"])
    h.check_invariants()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in STEP if c["fn"] == "priority_based_eviction"], ids=lambda c: c["name"])
def test_eviction_matches_reference(case):
    from paper_2506_12204_b200 import kvcache as K

    st = case["state"]
    reqs = [_req(d) for d in st["requests"]]
    by_id = {r.id: r for r in reqs}
    g, h = EvictionQueue(), DispatchQueue()
    _fill(g, st["g"], by_id)
    _fill(h, st["h"], by_id)
    mem = K.DeviceMemory(capacity=st["cap"], used=st["used"])
    err = None
    decisions = []
    try:
        decisions = K.priority_based_eviction(by_id[st["target"]], g, h, mem, PROFILES[st["profile"]],
                                              demand=st["demand"], protected=set(st["protected"]),
                                              dependency_rule=st["dep"])
    except K.AdmissionFailure as exc:
        err = ["AdmissionFailure", exc.rid, exc.needed, exc.free]
    res = case["result"]
    assert err == res["error"]
    assert _same([[d.victim_id, d.prefill_action, d.decode_saved, d.decode_discarded, d.freed_slots, d.f_t_before,
                   d.f_t_after] for d in decisions], res["decisions"])
    assert mem.used == res["used_after"]
    assert _same(_heap_dump(g), res["g_after"])
    assert _same(_heap_dump(h), res["h_after"])
    assert _same([_dump(r) for r in reqs], res["requests_after"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in STEP if c["fn"] == "should_recompute"], ids=lambda c: c["name"])
def test_should_recompute_matches_reference(case):
    from paper_2506_12204_b200 import kvcache as K

    st = case["state"]
    r = _req(st["requests"][0])
    d = K.should_recompute(r, PROFILES[st["profile"]], st["dep"])
    assert _same([d.victim_id, d.prefill_action, d.decode_saved, d.decode_discarded, d.freed_slots, d.f_t_before,
                  d.f_t_after], case["result"]["decision"])
    assert _same([_dump(r)], case["result"]["requests_after"])


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8191, 8193, 100_000])
def test_select_large_pool_grid_path(n):
    """Pools above 8,192 keys take the grid-wide partial top-32 pass; the
    pops must be the n smallest stored keys in order (numpy lexsort)."""
    from paper_2506_12204_b200 import step as S

    rng = np.random.default_rng(n)
    keys = np.stack([rng.integers(0, 5, n).astype(float), np.round(rng.random(n) * 20, 2),
                     rng.random(n) * 100, np.arange(n, dtype=float)], axis=1)
    cand, _, _, _ = S.select_batch(keys, None, np.zeros(n, np.uint8), np.zeros((0, 4)), np.zeros(0, np.uint8), 32,
                                   S.SS_SELECT_TOP_B)
    want = np.lexsort((keys[:, 3], keys[:, 2], keys[:, 1], keys[:, 0]))[:32]
    assert np.array_equal(cand, want)


@pytest.mark.gpu
def test_step_errors():
    from paper_2506_12204_b200 import batching as B
    from paper_2506_12204_b200 import kvcache as K

    h, u = DispatchQueue(), ArrivalBuffer()
    with pytest.raises(ValueError):
        B.extract_top_b(h, u, 0)
    assert B.stage_aware_schedule(h, u, [], 4).members == []
    r = _req([1, 0.0, 10, 5, 0, 50, 1.0, 0, 0, 0, 0, "waiting", 0])
    with pytest.raises(ValueError):
        K.should_recompute(r, PROFILES["a100_qwen7b"])  # no device-resident KV


# ---- CPU: host containers (reference tests/test_heaps.py behaviour) ------------
def _mk(rid, urgency=2, f_t=1.0, arrival=0.0):
    return Request(id=rid, arrival_time=arrival, prompt_len=10, true_output_len=5, true_urgency=UrgencyLevel(urgency),
                   f_e=UrgencyLevel(urgency), predicted_bucket=LengthBucket(0, 50), f_t=f_t)


def test_buffer_fifo_and_duplicates():
    u = ArrivalBuffer()
    for i in range(4):
        u.append(_mk(i))
    assert [r.id for r in u.items()] == [0, 1, 2, 3]
    with pytest.raises(DuplicateRequestError):
        u.append(_mk(2))


def test_drain_orders_by_priority():
    rng = random.Random(3)
    reqs = [_mk(i, rng.randrange(5), rng.random() * 10, rng.random()) for i in range(200)]
    h, u = DispatchQueue(), ArrivalBuffer()
    for r in reqs:
        u.append(r)
    assert u.drain_into(h) == 200 and len(u) == 0
    out = [h.pop_top() for _ in range(len(h))]
    assert out == sorted(reqs, key=lambda r: r.priority_key())


def test_heap_errors():
    h = IndexedMinHeap()
    with pytest.raises(EmptyQueueError):
        h.pop()
    with pytest.raises(EmptyQueueError):
        h.peek()
    with pytest.raises(NotFoundError):
        h.delete(7)
    r = _mk(1)
    h.insert(r, (1,))
    with pytest.raises(DuplicateRequestError):
        h.insert(r, (2,))


def test_eviction_root_is_dispatch_maximum():
    reqs = [_mk(i, i % 5, float(i)) for i in range(20)]
    g = EvictionQueue()
    for r in reqs:
        g.insert(r)
    assert g.peek_victim() is max(reqs, key=lambda r: r.priority_key())


def test_random_op_storm_matches_sorted_order():
    """insert / pop / delete / update storm against a sorted-list model."""
    rng = random.Random(11)
    h = IndexedMinHeap()
    model = {}
    nxt = 0
    for _ in range(4000):
        op = rng.random()
        if op < 0.45 or not model:
            r = _mk(nxt)
            key = (rng.randrange(5), rng.random(), nxt)
            h.insert(r, key)
            model[nxt] = (key, r)
            nxt += 1
        elif op < 0.65:
            got = h.pop()
            kmin = min(model.values(), key=lambda x: x[0])
            assert got is kmin[1]
            del model[got.id]
        elif op < 0.85:
            rid = rng.choice(list(model))
            assert h.delete(rid) is model.pop(rid)[1]
        else:
            rid = rng.choice(list(model))
            key = (rng.randrange(5), rng.random(), rid)
            h.update(model[rid][1], key)
            model[rid] = (key, model[rid][1])
        if rng.random() < 0.01:
            h.check_position_map()
    h.check_position_map()
    assert [h.pop().id for _ in range(len(h))] == [r.id for _, r in sorted(model.values(), key=lambda x: x[0])]


def test_pack_keys_pads_short_tuples():
    from paper_2506_12204_b200 import step as S

    k = S.pack_keys([(1, 2.5), (0, 1.0, 3.0, 7)])
    assert k.shape == (2, 4) and np.isneginf(k[0, 2:]).all() and k[1, 3] == 7.0
    with pytest.raises(ValueError):
        S.pack_keys([(1, 2, 3, 4, 5)])
