"""Named workloads of BASELINE.json / SURVEY.md §8(d) (configs A-E).

Each builder returns plain ``Request`` lists (ground truth only), so the same
arrivals can be fed to this package's ``run`` and to the reference's
``run(cfg, arrivals)``.

A  medical: 1,000 requests, 3 uniform levels, Poisson arrivals (rate 15/s,
   ``random.Random(seed).expovariate``), prompt U[16,128], output U[1,500],
   a100_qwen7b, fixed KV budget of 4,096 slots.
B  4,096 traces x ``generate(WorkloadSpec(total_requests=1000, seed=s))``,
   s = 0..4095, ample memory (10**9 slots), a100_qwen7b, b = 16.
C  one trace of N requests all at t = 0 (``concurrent=N, concurrent_mode="fixed"``).
D  memory-constrained: a config A/B trace with capacity = ample peak // 4
   under a100_qwen7b (offload), a5000_qwen7b (discard) and ``MIXED_PROFILE``.
E  65,536 traces x 2,000 requests (``WorkloadSpec(total_requests=2000, seed=s)``).
"""

from __future__ import annotations

import random
from typing import List

from .costs import GpuProfile
from .requests import Request, UrgencyLevel
from .workload import WorkloadSpec

MIXED_PROFILE = GpuProfile("mixed", alpha1=5e-5, alpha2=1e-4, gamma1=1e-5, gamma2=1e-3,
                           beta_load=5e-3, beta_save=5e-3)


def medical_arrivals(seed: int = 0, n: int = 1000, rate: float = 15.0, levels: int = 3,
                     prompt_len_range=(16, 128), output_len_range=(1, 500)) -> List[Request]:
    """Config A arrivals: Poisson process, uniform urgency."""
    rng = random.Random(seed)
    t = 0.0
    out = []
    for i in range(n):
        t += rng.expovariate(rate)
        u = rng.randrange(levels)
        p = rng.randint(*prompt_len_range)
        o = rng.randint(*output_len_range)
        out.append(Request(id=i, arrival_time=t, prompt_len=p, true_output_len=o,
                           true_urgency=UrgencyLevel(u, levels)))
    return out


def workload_b(seed: int, total_requests: int = 1000) -> WorkloadSpec:
    return WorkloadSpec(total_requests=total_requests, seed=seed)


def workload_c(n: int, seed: int = 1) -> WorkloadSpec:
    return WorkloadSpec(total_requests=n, concurrent=n, concurrent_mode="fixed", seed=seed)


def workload_e(seed: int) -> WorkloadSpec:
    return WorkloadSpec(total_requests=2000, seed=seed)
