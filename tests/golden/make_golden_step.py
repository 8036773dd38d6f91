"""Golden fixtures for the per-step API, produced by the REFERENCE.

    python tests/golden/make_golden_step.py      (build container only: needs /root/reference)

Random scheduler states are built with the reference's own heaps and Request
objects and fed to its ``extract_top_b`` / ``stage_aware_schedule``
(batching.py:46-88), ``priority_based_eviction`` (kvcache.py:137-179) and
``should_recompute`` (kvcache.py:81-134). Each case records the state (every
request's fields, where it sits and the key each heap stored for it — keys go
stale when f_t changes after insertion, as in the simulator), the call's
arguments and everything observable afterwards: the batch, the decisions or
the exception, every request's fields, and the (id, stored key) contents of
both heaps. ``tests/test_step_api.py`` replays the cases through this
package's device-backed functions.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from semsched import batching as B  # noqa: E402
from semsched import kvcache as K  # noqa: E402
from semsched.costs import GpuProfile, get_profile  # noqa: E402
from semsched.heaps import ArrivalBuffer, DispatchQueue, EvictionQueue  # noqa: E402
from semsched.requests import LengthBucket, Request, Stage, UrgencyLevel  # noqa: E402

MIXED = GpuProfile("mixed", alpha1=5e-5, alpha2=1e-4, gamma1=1e-5, gamma2=1e-3, beta_load=5e-3, beta_save=5e-3)
PROFILES = {"a100_qwen7b": get_profile("a100_qwen7b"), "a5000_qwen7b": get_profile("a5000_qwen7b"), "mixed": MIXED}
FIELDS = ("id", "arrival_time", "prompt_len", "true_output_len", "f_e", "mid", "f_t", "prefilled_tokens",
          "decoded_tokens", "kv_device_tokens", "kv_host_tokens", "stage", "evictions")


def dump(r):
    return [r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.f_e.rank, r.predicted_bucket.representative_len,
            r.f_t, r.prefilled_tokens, r.decoded_tokens, r.kv_device_tokens, r.kv_host_tokens, r.stage.value,
            r.evictions]


def make(rng, rid, levels=5, stage=None):
    prompt = rng.randint(1, 256)
    out = rng.randint(1, 400)
    mid = rng.choice([50, 150, 250, 350, 450])
    r = Request(id=rid, arrival_time=round(rng.random() * 50, 6), prompt_len=prompt, true_output_len=out,
                true_urgency=UrgencyLevel(rng.randrange(levels), levels), f_e=UrgencyLevel(rng.randrange(levels), levels),
                predicted_bucket=LengthBucket(0, mid), f_t=rng.random() * 30)
    if rng.random() < 0.15:  # equal remaining times: the arrival / id tail decides
        r.f_t = 5.0
    st = stage or rng.choice([Stage.WAITING, Stage.DECODING, Stage.PREFILLING])
    r.stage = st
    if st in (Stage.DECODING, Stage.PREFILLING):
        r.prefilled_tokens = prompt if (st is Stage.DECODING or rng.random() < 0.5) else rng.randint(0, prompt)
        r.decoded_tokens = rng.randint(0, min(out - 1, 300)) if st is Stage.DECODING else 0
        r.kv_device_tokens = max(1, r.prefilled_tokens + r.decoded_tokens)
    return r


def heap_dump(q):
    return sorted([[r.id, list(k)] for r, k in zip(q._heap._items, q._heap._keys)])


def select_case(rng, name):
    n_heap = rng.choice([0, 1, 3, 17, 40, 200, 1500])
    n_buf = rng.choice([0, 0, 2, 9])
    n_ong = rng.choice([0, 1, 4, 12])
    b = rng.choice([1, 2, 4, 8, 16, 32])
    reqs = [make(rng, i) for i in range(n_heap + n_buf + n_ong)]
    for r in reqs[n_heap + n_buf:]:
        r.stage = Stage.DECODING
        r.prefilled_tokens = r.prompt_len
        r.kv_device_tokens = r.prompt_len + r.decoded_tokens
    h, u = DispatchQueue(), ArrivalBuffer()
    where = {}
    for r in reqs[:n_heap]:
        h.insert(r)
        where[r.id] = "heap"
    for r in reqs[n_heap:n_heap + n_buf]:
        u.append(r)
        where[r.id] = "buffer"
    ongoing = reqs[n_heap + n_buf:]
    for r in ongoing:
        where[r.id] = "ongoing"
    if n_heap and rng.random() < 0.5:  # stale stored keys
        for r in rng.sample(reqs[:n_heap], max(1, n_heap // 5)):
            r.f_t = rng.random() * 30
    state = {"requests": [dump(r) for r in reqs], "where": where, "heap": heap_dump(h),
             "buffer": [r.id for r in u.items()], "ongoing": [r.id for r in ongoing]}
    fn = rng.choice(["stage_aware_schedule", "stage_aware_schedule", "extract_top_b"])
    if fn == "extract_top_b":
        got = B.extract_top_b(h, u, b)
        result = {"popped": [r.id for r in got]}
    else:
        batch = B.stage_aware_schedule(h, u, ongoing, b)
        result = {"kind": batch.kind.value, "members": [r.id for r in batch.members]}
    result["heap_after"] = heap_dump(h)
    result["requests_after"] = [dump(r) for r in reqs]
    return {"name": name, "fn": fn, "b": b, "state": state, "result": result}


def evict_case(rng, name):
    n_res = rng.choice([1, 2, 5, 12, 40, 150])
    n_queued = rng.choice([0, 3, 20])
    prof = rng.choice(list(PROFILES))
    dep = rng.random() < 0.7
    residents = [make(rng, i, stage=rng.choice([Stage.DECODING, Stage.DECODING, Stage.PREFILLING]))
                 for i in range(n_res)]
    queued = [make(rng, n_res + i, stage=Stage.WAITING) for i in range(n_queued)]
    g, h = EvictionQueue(), DispatchQueue()
    for r in residents:
        g.insert(r)
    for r in queued:
        h.insert(r)
    # pushed-back residents are queued too (heap membership of a victim)
    for r in rng.sample(residents, min(len(residents), rng.choice([0, 1, 3]))):
        h.insert(r)
    if rng.random() < 0.5:  # stale eviction keys
        for r in rng.sample(residents, max(1, n_res // 4)):
            r.f_t = rng.random() * 30
    used = sum(r.kv_device_tokens for r in residents)
    cap = used + rng.choice([0, 5, 50])
    target = residents[rng.randrange(n_res)] if rng.random() < 0.5 else make(rng, 10_000)
    protected = {r.id for r in rng.sample(residents, min(n_res, rng.choice([0, 1, 4])))}
    demand = rng.choice([None, rng.randint(1, max(1, used // 2)), rng.randint(1, used + 100)])
    reqs = residents + queued + ([target] if target.id == 10_000 else [])
    state = {"requests": [dump(r) for r in reqs], "g": heap_dump(g), "h": heap_dump(h), "used": used, "cap": cap,
             "target": target.id, "protected": sorted(protected), "demand": demand, "profile": prof, "dep": dep}
    mem = K.DeviceMemory(capacity=cap, used=used)
    err = None
    decisions = []
    try:
        decisions = K.priority_based_eviction(target, g, h, mem, PROFILES[prof], demand=demand, protected=protected,
                                              dependency_rule=dep)
    except K.AdmissionFailure as exc:
        err = ["AdmissionFailure", exc.rid, exc.needed, exc.free]
    result = {"decisions": [[d.victim_id, d.prefill_action, d.decode_saved, d.decode_discarded, d.freed_slots,
                             d.f_t_before, d.f_t_after] for d in decisions],
              "error": err, "used_after": mem.used, "g_after": heap_dump(g), "h_after": heap_dump(h),
              "requests_after": [dump(r) for r in reqs]}
    return {"name": name, "fn": "priority_based_eviction", "state": state, "result": result}


def recompute_case(rng, name):
    prof = rng.choice(list(PROFILES))
    dep = rng.random() < 0.5
    r = make(rng, 0, stage=rng.choice([Stage.DECODING, Stage.PREFILLING]))
    state = {"requests": [dump(r)], "profile": prof, "dep": dep}
    d = K.should_recompute(r, PROFILES[prof], dep)
    result = {"decision": [d.victim_id, d.prefill_action, d.decode_saved, d.decode_discarded, d.freed_slots,
                           d.f_t_before, d.f_t_after], "requests_after": [dump(r)]}
    return {"name": name, "fn": "should_recompute", "state": state, "result": result}


def main():
    rng = random.Random(2506_12204)
    cases = []
    for i in range(120):
        cases.append(select_case(rng, f"select_{i}"))
    for i in range(120):
        cases.append(evict_case(rng, f"evict_{i}"))
    for i in range(60):
        cases.append(recompute_case(rng, f"recompute_{i}"))
    out = os.path.join(HERE, "golden_step.json.gz")
    with gzip.open(out, "wt", encoding="utf-8") as fh:
        json.dump({"fields": FIELDS, "cases": cases}, fh)
    kinds = {}
    for c in cases:
        k = c["fn"] + ("/error" if c["result"].get("error") else "")
        kinds[k] = kinds.get(k, 0) + 1
    print(out, kinds)


if __name__ == "__main__":
    main()
