"""Batch container types (``/root/reference/pkg/src/semsched/batching.py:19-43``).

The stage-aware selection itself (batching.py:46-88) runs on the device:
candidates are the first b keys of the sorted queue front, merged with the
ongoing members (held one per lane) by rank counting in shared memory, with
the p*-stage rule deciding which candidates are eligible
(``csrc/ss_kernel.cu``, "stage-aware composition")."""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List

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
