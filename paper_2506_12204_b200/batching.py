"""Batch types and the per-step selection API
(``/root/reference/pkg/src/semsched/batching.py:19-88``).

Inside whole-trace runs the stage-aware selection is part of the scheduler
kernel (``csrc/ss_kernel.cu``, "stage-aware composition"). For callers that
drive their own loop, ``extract_top_b`` and ``stage_aware_schedule`` keep the
reference's signatures and heap side effects; the selection runs on the
device (``ss_select_batch``, ``csrc/ss_step.cu``): a grid-wide top-b of the
dispatch heap's stored keys, then one warp applies the p*-stage rule and
ranks the merge."""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List

from . import step as S
from .requests import Request, Stage


class BatchKind(enum.Enum):
    PREFILL = "prefill"
    DECODE = "decode"


def _needs_prefill_work(r: Request) -> bool:
    return r.stage is not Stage.DECODING


@dataclass
class Batch:
    kind: BatchKind
    members: List[Request] = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.members)

    def prefill_members(self) -> List[Request]:
        return [r for r in self.members if _needs_prefill_work(r)]

    def decode_members(self) -> List[Request]:
        return [r for r in self.members if not _needs_prefill_work(r)]


def _pop_candidates(h, u, want: int) -> List[Request]:
    """Drain the buffer, then pop the ``want`` smallest stored keys (device
    selection over the whole heap)."""
    u.drain_into(h)
    if want <= 0 or len(h) == 0:
        return []
    items = h._heap.items()
    cand, _, _, _ = S.select_batch(S.pack_keys(h._heap.keys()), None, [0] * len(items),
                                   S.pack_keys([]), [], min(want, 32), S.SS_SELECT_TOP_B)
    out = [items[int(i)] for i in cand]
    for r in out:
        h.delete_by_id(r.id)
    return out


def extract_top_b(h, u, b: int) -> List[Request]:
    """Drain the buffer, then pop up to b best candidates (batching.py:46-54)."""
    if b < 1:
        raise ValueError("batch size must be >= 1")
    if b > 32:
        raise ValueError("batch size above 32 (SS_MAX_BATCH) is not supported")
    return _pop_candidates(h, u, b)


def _compose(h, candidates: List[Request], ongoing: List[Request], b: int, mode: int) -> Batch:
    """Device merge of the popped candidates with the ongoing requests on
    current keys; pushes back what the reference pushes back."""
    key = h.key_fn
    cur = S.pack_keys([key(r) for r in candidates])
    cand, merged, nsel, kind = S.select_batch(cur, None, [0 if _needs_prefill_work(r) else 1 for r in candidates],
                                              S.pack_keys([key(r) for r in ongoing]),
                                              [0 if _needs_prefill_work(r) else 1 for r in ongoing],
                                              b, mode)
    # merge entries j < len(cand) name the device's j-th candidate
    pool = [candidates[int(i)] for i in cand] + list(ongoing)
    members = [pool[int(j)] for j in merged]
    if mode == S.SS_SELECT_STAGE_AWARE and kind == 0:
        # decode batch: prefill candidates go back first (batching.py:78-79)
        in_merge = {id(r) for r in members}
        h.push_back([r for r in candidates if id(r) not in in_merge])
    if mode != S.SS_SELECT_FCFS:
        h.push_back(members[nsel:])
    return Batch(BatchKind.DECODE if kind == 0 else BatchKind.PREFILL, members[:nsel])


def stage_aware_schedule(h, u, ongoing: List[Request], b: int) -> Batch:
    """Select the next batch, merging candidates with ongoing requests
    (batching.py:57-88); everything considered but not selected is pushed
    back into the dispatch heap."""
    candidates = extract_top_b(h, u, b)
    if not candidates and not ongoing:
        return Batch(BatchKind.DECODE, [])
    if len(ongoing) > 32:
        raise ValueError("more than 32 ongoing requests (SS_MAX_BATCH) is not supported")
    return _compose(h, candidates, list(ongoing), b, S.SS_SELECT_STAGE_AWARE)
