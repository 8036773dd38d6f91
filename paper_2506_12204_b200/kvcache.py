"""Device-memory accounting and priority-based eviction — the reference's
per-step API (``/root/reference/pkg/src/semsched/kvcache.py:24-179``).

``priority_based_eviction`` and ``should_recompute`` make their decisions on
the device (``ss_evict``, ``csrc/ss_step.cu``): the victims are found by
walking the eviction heap's stored keys in order with a warp scan of the
freed slots, and every victim's offload-vs-discard choice, Eq. 6 save count
and new f_t are computed there with the same float64 expressions as the
whole-trace kernel. This module applies those results to the caller's
``Request`` objects and heaps in the reference's order, so mutations,
exceptions and heap contents match the reference step for step.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Set

from . import step as S
from .costs import GpuProfile
from .heaps import DispatchQueue, EvictionQueue
from .requests import Request, Stage


class AdmissionFailure(RuntimeError):
    """Eviction exhausted every victim and space is still insufficient
    (kvcache.py:24-31)."""

    def __init__(self, rid: int, needed: int, free: int):
        super().__init__(f"request {rid} needs {needed} slots, only {free} free")
        self.rid = rid
        self.needed = needed
        self.free = free


@dataclass
class DeviceMemory:
    """Token-slot accounting (kvcache.py:34-56)."""

    capacity: int
    used: int = 0

    def __post_init__(self) -> None:
        if self.capacity < 0:
            raise ValueError("capacity must be nonnegative")

    @property
    def free(self) -> int:
        return self.capacity - self.used

    def allocate(self, slots: int) -> None:
        if slots > self.free:
            raise AdmissionFailure(-1, slots, self.free)
        self.used += slots

    def release(self, slots: int) -> None:
        if slots > self.used:
            raise ValueError("releasing more slots than in use")
        self.used -= slots


@dataclass(frozen=True)
class EvictionDecision:
    """kvcache.py:59-67."""

    victim_id: int
    prefill_action: str  # "offload" | "discard"
    decode_saved: int
    decode_discarded: int
    freed_slots: int
    f_t_before: float
    f_t_after: float


def estimate_kv_size(r: Request) -> int:
    """Slots still needed through the predicted completion (kvcache.py:70-78)."""
    if r.stage is Stage.COMPLETED:
        raise ValueError("completed request has no KV demand")
    if r.predicted_bucket is None:
        raise ValueError(f"request {r.id} has no length prediction yet")
    return max(0, r.prompt_len + r.predicted_bucket.representative_len - r.kv_device_tokens)


def _state(reqs: List[Request]):
    for r in reqs:
        if r.predicted_bucket is None:
            raise ValueError(f"request {r.id} has no length prediction yet")
    return ([r.prompt_len for r in reqs], [r.prefilled_tokens for r in reqs], [r.decoded_tokens for r in reqs],
            [r.kv_device_tokens for r in reqs], [r.predicted_bucket.representative_len for r in reqs],
            [r.f_t for r in reqs])


def _apply(r: Request, v) -> EvictionDecision:
    """The state changes of should_recompute (kvcache.py:96-134), with the
    device-computed numbers."""
    if r.kv_device_tokens <= 0:
        raise ValueError(f"victim {r.id} has no device-resident KV")
    action = "offload" if int(v["action"]) == 0 else "discard"
    r.prefilled_tokens = int(v["prefilled"])
    saved = int(v["decode_saved"])
    r.decoded_tokens = saved
    r.kv_device_tokens = 0
    r.kv_host_tokens = int(v["kv_host"])
    r.transition(Stage.EVICTED_OFFLOADED if r.kv_host_tokens > 0 else Stage.EVICTED_DISCARDED)
    r.transition(Stage.WAITING)
    r.evictions += 1
    r.f_t = float(v["f_t_after"])
    return EvictionDecision(victim_id=r.id, prefill_action=action, decode_saved=saved,
                            decode_discarded=int(v["decode_discarded"]), freed_slots=int(v["freed_slots"]),
                            f_t_before=float(v["f_t_before"]), f_t_after=r.f_t)


def should_recompute(r_v: Request, p: GpuProfile, dependency_rule: bool = True) -> EvictionDecision:
    """Resolve one victim's device KV (kvcache.py:81-134)."""
    if r_v.kv_device_tokens <= 0:
        raise ValueError(f"victim {r_v.id} has no device-resident KV")
    pr, pf, de, kv, pl, ft = _state([r_v])
    out, _, _ = S.evict(None, pr, pf, de, kv, pl, ft, None, 0, 0, 0, p, dependency_rule, select=False)
    return _apply(r_v, out[0])


def priority_based_eviction(r: Request, g: EvictionQueue, h: DispatchQueue, mem: DeviceMemory,
                            profile: GpuProfile, demand: Optional[int] = None,
                            protected: Optional[Set[int]] = None,
                            dependency_rule: bool = True) -> List[EvictionDecision]:
    """Free device memory for ``r`` by evicting the lowest-priority residents
    (kvcache.py:137-179). Raises AdmissionFailure when the unprotected
    residents cannot cover ``demand``; evictions already made stand."""
    if demand is None:
        demand = estimate_kv_size(r)
    protected = set(protected or ()) | {r.id}
    reqs = g._heap.items()
    decisions: List[EvictionDecision] = []
    if demand + mem.used <= mem.capacity or not reqs:
        if demand + mem.used > mem.capacity:
            raise AdmissionFailure(r.id, demand, mem.free)
        return decisions
    keys = S.pack_keys(g._heap.keys())
    prot = [1 if x.id in protected else 0 for x in reqs]
    pr, pf, de, kv, pl, ft = _state(reqs)
    victims, skipped, failed = S.evict(keys, pr, pf, de, kv, pl, ft, prot, demand, mem.used, mem.capacity,
                                       profile, dependency_rule, select=True)
    # replay the reference's pop sequence: protected entries are popped (and
    # set aside) as the eviction order reaches them, victims are processed
    skip = [(keys_i, reqs[int(i)]) for i, keys_i in ((i, g._heap.key_of(reqs[int(i)].id)) for i in skipped)]
    popped: List[Request] = []

    def pop_skipped_before(key) -> None:
        while skip and (key is None or skip[0][0] < key):
            x = skip.pop(0)[1]
            g.delete_by_id(x.id)
            popped.append(x)

    try:
        for v in victims:
            victim = reqs[int(v["index"])]
            pop_skipped_before(g._heap.key_of(victim.id))
            g.delete_by_id(victim.id)
            if victim.id in h:
                h.delete_by_id(victim.id)
            mem.release(victim.kv_device_tokens)
            decisions.append(_apply(victim, v))
            h.insert(victim)
        if failed:
            pop_skipped_before(None)
            raise AdmissionFailure(r.id, demand, mem.free)
    finally:
        for x in popped:
            g.insert(x)
    return decisions
