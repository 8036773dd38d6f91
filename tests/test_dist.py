"""Multi-rank host logic on CPU (gloo, world size 2): trace sharding and the
all-gather of per-trace statistics reproduce a single-process job exactly.
The per-shard results come from the oracle here (no GPU); on GPUs the same
functions carry the CUDA results over NCCL (bench.py)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, traces, out_path):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist

    from oracle_binding import run_oracle
    from paper_2506_12204_b200 import _abi as A
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.dist import gather_stats, job_summary, shard_seeds, stats_to_tensor
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = shard_seeds(traces, rank)
    batch = generate_batch(WorkloadSpec(total_requests=150, levels=3), seeds, threads=2)
    res = run_oracle(make_params(get_profile("a100_qwen7b"), 16, 800, levels=3, flags=A.SS_FLAG_DIGEST), batch)
    allst = gather_stats(stats_to_tensor(res.stats), world)
    if rank == 0:
        np.save(out_path, allst)
        summ = job_summary(allst)
        assert summ["traces"] == world * traces
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_matches_single_process(tmp_path):
    from oracle_binding import run_oracle
    from paper_2506_12204_b200 import _abi as A
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    world, traces = 2, 12
    out = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(world, _free_port(), traces, out), nprocs=world, start_method="spawn")
    gathered = np.load(out)
    batch = generate_batch(WorkloadSpec(total_requests=150, levels=3), np.arange(world * traces), threads=2)
    ref = run_oracle(make_params(get_profile("a100_qwen7b"), 16, 800, levels=3, flags=A.SS_FLAG_DIGEST), batch)
    for k in ("digest", "rounds", "evictions", "completed", "status"):
        assert np.array_equal(gathered[k], ref.stats[k]), k
    assert np.array_equal(gathered["sum_wait"].view(np.uint64), ref.stats["sum_wait"].view(np.uint64))


def test_shard_seeds_partition():
    from paper_2506_12204_b200.dist import shard_seeds

    parts = [shard_seeds(4096, r) for r in range(8)]
    allv = np.concatenate(parts)
    assert np.array_equal(allv, np.arange(8 * 4096))


def _bench_dry(nproc, traces):
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(repo, "bench.py"), "--dry", "--workload", "E", "--traces", str(traces),
           "--gpus", str(nproc)]
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}"] + cmd[1:]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=repo)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_config_e_sharding_gathers_one_job():
    """bench.py --workload E under torchrun (2 ranks, gloo): one fixed job
    split in seed blocks, every trace's record gathered once, in seed order,
    identical to a single-process run."""
    two = _bench_dry(2, 512)
    one = _bench_dry(1, 512)
    assert two["gathered_traces"] == one["gathered_traces"] == two["traces_total"] == 512
    assert two["seeds_in_order"] and one["seeds_in_order"]
    assert two["checksum"] == one["checksum"]


def test_job_seeds_blocks():
    from paper_2506_12204_b200.dist import job_seeds

    for total, world in ((65536, 8), (65536, 2), (10, 3), (5, 8)):
        parts = [job_seeds(total, world, r) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), np.arange(total))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
