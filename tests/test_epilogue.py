"""Grid-wide end of trace (csrc/ss_epilogue.cu) for long traces.

A trace of >= ss_params.epilogue_min requests (default 16,384; config C's
one-million-request pool) leaves its per-request read-out and its waiting-time
sums (metrics.py:35-56) to two grid-wide kernels instead of its scheduler
warp. Per-request outputs and every schedule field stay bit-exact; the float
sums are exact double-double tile sums, compared with CPython's sequential
sum (oracle) at 1e-12 relative (north_star's contract: 1e-6)."""

import numpy as np
import pytest

from conftest import case_batch, case_params, golden_cases
from parity_helpers import check_against_golden, compare_with_oracle

from paper_2506_12204_b200 import _abi as A

pytestmark = pytest.mark.gpu

REL = 1e-12
LARGE = golden_cases("large")


@pytest.fixture(scope="module")
def native():
    from paper_2506_12204_b200 import native as nat

    nat.device_info()
    return nat


def _stats_close(a, b, rel=REL):
    for k in ("sum_wait", "sum_norm_wait", "level_norm_sum"):
        np.testing.assert_allclose(a[k], b[k], rtol=rel, atol=0, err_msg=k)
    for k in ("completed", "level_count"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("case", LARGE, ids=[c["name"] for c in LARGE])
def test_epilogue_forced_matches_reference(native, case):
    """epilogue_min = 1: every golden trace ends through the grid-wide kernels."""
    batch = case_batch(case)
    p = case_params(case, A.SS_FLAG_DIGEST)
    p.epilogue_min = 1
    res = native.run_host(p, batch)
    check_against_golden(res, case, batch=batch)
    warp = native.run_host(case_params(case, A.SS_FLAG_DIGEST), batch)  # sequential CPython sum in the warp
    _stats_close(res.stats, warp.stats)
    assert np.array_equal(res.state, warp.state) and np.array_equal(res.generated, warp.generated)


@pytest.mark.parametrize("capacity", [10**9, 900])
def test_epilogue_mixed_lengths_vs_oracle(native, capacity):
    """Short and long traces in one launch (threshold 500): long ones end on the
    grid, short ones in their warp; tiles of a trace straddle CTA boundaries."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.soa import TraceBatch
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    parts = [generate_batch(WorkloadSpec(total_requests=n, levels=4), [s], pinned=False)
             for s, n in enumerate((300, 9000, 40, 4096, 4097, 700, 12000))]
    batch = TraceBatch.concat(parts)
    p = lambda e: make_params(get_profile("a100_qwen7b"), 16, capacity, levels=4, flags=A.SS_FLAG_DIGEST,
                              epilogue_min=e)
    gpu = native.run_host(p(500), batch)
    cpu = run_oracle(p(0), batch, threads=8)
    compare_with_oracle(gpu, cpu, batch, stats_rel=REL)
    assert np.array_equal(gpu.state, cpu.state)
    sizes = np.diff(batch.offsets)
    short = sizes < 500
    for k in ("sum_wait", "sum_norm_wait"):  # warp-finished traces stay bit-exact
        assert np.array_equal(gpu.stats[k][short].view(np.uint64), cpu.stats[k][short].view(np.uint64))


@pytest.mark.slow
def test_config_c_pool_to_completion_vs_oracle(native):
    """Config C (BASELINE.json configs[2]): one pool of 1,000,000 requests at
    t = 0, run to completion (~16M rounds) and compared with the oracle: status,
    rounds, digest, every request's first_scheduled / finish bits, generated
    tokens and final f_t, and the fused statistics."""
    from oracle_binding import run_oracle
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    n = 1_000_000
    batch = generate_batch(WorkloadSpec(total_requests=n, concurrent=n, concurrent_mode="fixed", seed=1), [1])
    p = lambda: make_params(get_profile("a100_qwen7b"), 16, 10**9, levels=5, flags=A.SS_FLAG_DIGEST)
    gpu = native.run_host(p(), batch)
    assert int(gpu.stats["status"][0]) == A.SS_TRACE_OK
    assert int(gpu.stats["completed"][0]) == n
    cpu = run_oracle(p(), batch)
    compare_with_oracle(gpu, cpu, batch, stats_rel=REL)
    assert np.array_equal(gpu.state, cpu.state)
