"""Trace sharding across ranks and the one collective.

Traces are independent. Weak scaling (configs B, D): T traces per rank, rank
r takes seeds ``[r*T, (r+1)*T)``. Strong scaling (config E): one fixed job of
T traces split into contiguous seed blocks (``job_seeds``). Either way no
communication happens until the end, when the fixed-size per-trace
statistics records are all-gathered. The same
functions run over NCCL (``bench.py``) and gloo (``tests/test_dist.py``).
"""

from __future__ import annotations

import numpy as np

from . import _abi as A


def shard_seeds(traces_per_rank: int, rank: int, seed0: int = 0) -> np.ndarray:
    return np.arange(seed0 + rank * traces_per_rank, seed0 + (rank + 1) * traces_per_rank, dtype=np.int64)


def stats_to_tensor(stats: np.ndarray, device="cpu"):
    import torch

    raw = np.ascontiguousarray(stats).view(np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


def all_gather_stats(local, world: int, out=None):
    """The one collective: all-gather the per-trace ss_trace_stats records
    (a uint8 tensor on the rank's device; NCCL over NVLink on GPUs, gloo on
    CPU) into ``out`` (allocated when None), rank-major. Stays on the device
    and is stream-ordered, so bench.py issues it inside the timed step."""
    import torch
    import torch.distributed as dist

    if out is None:
        out = torch.empty(world * local.numel(), dtype=torch.uint8, device=local.device)
    if world > 1:
        dist.all_gather_into_tensor(out, local)
    else:
        out.copy_(local)
    return out


def stats_of(gathered) -> np.ndarray:
    """Structured per-trace records of a gathered uint8 tensor."""
    return gathered.cpu().numpy().view(A.stats_dtype())


def gather_stats(local, world: int):
    """all-gather per-trace ss_trace_stats records (uint8 tensor) from every rank;
    returns the concatenated structured array in rank order."""
    return stats_of(all_gather_stats(local, world))


def job_seeds(total_traces: int, world: int, rank: int, seed0: int = 0) -> np.ndarray:
    """Strong scaling: ONE job of ``total_traces`` traces (seeds
    seed0..seed0+total-1) block-partitioned over ``world`` ranks; the blocks
    are equal when world divides the total, else the first ranks take one more."""
    base, extra = divmod(total_traces, world)
    lo = seed0 + rank * base + min(rank, extra)
    return np.arange(lo, lo + base + (rank < extra), dtype=np.int64)


def job_summary(stats: np.ndarray) -> dict:
    """Whole-job aggregates from gathered per-trace records."""
    done = stats["completed"].astype(np.int64)
    return {
        "traces": int(len(stats)),
        "decisions": int(stats["rounds"].sum()),
        "evictions": int(stats["evictions"].sum()),
        "completed": int(done.sum()),
        "failed_traces": int((stats["status"] != A.SS_TRACE_OK).sum()),
        "mean_wait_s": float(stats["sum_wait"].sum() / max(done.sum(), 1)),
        "mean_norm_wait_s_per_tok": float(stats["sum_norm_wait"].sum() / max(done.sum(), 1)),
    }
