"""Small workloads that reach every kernel, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck --error-exitcode 9 \\
        python tools/sanitize_cases.py

Covers the three scheduler variants (no-eviction chunked, chunked, one round
per step) under both batch-duration modes, the baseline policies, the bulk
admission sort (all requests at t = 0), the grid-wide end of trace, the round
log, the device trace generator and the Eq. 2 audit (the per-step API through
tests/test_step_api.py, tools/sanitize.sh). Results are checked against the oracle so a
sanitizer-clean run is also a correct one.
"""

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from oracle_binding import run_oracle  # noqa: E402
from paper_2506_12204_b200 import _abi as A  # noqa: E402
from paper_2506_12204_b200 import native  # noqa: E402
from paper_2506_12204_b200.costs import get_profile  # noqa: E402
from paper_2506_12204_b200.results import make_params  # noqa: E402
from paper_2506_12204_b200.tracegen import generate_batch, generate_batch_device  # noqa: E402
from paper_2506_12204_b200.workload import WorkloadSpec  # noqa: E402


def check(name, params, batch, log=True):
    gpu = native.run_host(params, batch, want_log=log)
    cpu = run_oracle(params, batch, threads=4)
    ok = cpu.stats["status"] == 0
    assert np.array_equal(gpu.stats["status"], cpu.stats["status"]), name
    assert np.array_equal(gpu.stats["digest"][ok], cpu.stats["digest"][ok]), name
    print(f"{name}: {batch.n_traces} traces, {int(gpu.stats['rounds'].sum())} rounds ok", flush=True)


def main():
    prof = get_profile("a100_qwen7b")
    small = generate_batch(WorkloadSpec(total_requests=120, levels=3), list(range(6)))
    burst = generate_batch(WorkloadSpec(total_requests=1500, concurrent=1500, concurrent_mode="fixed", levels=3),
                           [3])
    for cost in ("max", "sum"):
        for tag, cap, flag in (("noevict", 10**9, 0), ("chunked", 700, A.SS_FLAG_FORCE_CHUNKED),
                               ("perround", 700, A.SS_FLAG_FORCE_PERROUND)):
            p = make_params(prof, 16, cap, levels=3, decode_batch_cost=cost, flags=A.SS_FLAG_DIGEST | flag)
            check(f"{tag}/{cost}", p, small)
    for pol in ("fcfs", "sjf", "hpjf"):
        check(pol, make_params(prof, 5, 700, policy=pol, levels=3, flags=A.SS_FLAG_DIGEST), small)
    # bulk admission (radix sort of the t = 0 group) + grid-wide end of trace
    check("bulk+epilogue", make_params(prof, 16, 10**9, levels=3, flags=A.SS_FLAG_DIGEST, epilogue_min=1000),
          burst, log=False)
    check("bulk+evict", make_params(prof, 16, 3000, levels=3, flags=A.SS_FLAG_DIGEST), burst, log=False)
    # device trace generator
    import torch

    db = generate_batch_device(WorkloadSpec(total_requests=120, levels=3), list(range(6)), device="cuda")
    assert torch.equal(db.t["ready"][: small.n_requests].cpu(), torch.from_numpy(small.ready))
    print("tracegen_device ok", flush=True)
    # the Eq. 2 audit (the per-step API runs under the sanitizer through
    # tests/test_step_api.py, see tools/sanitize.sh)
    from paper_2506_12204_b200.metrics import audit_batch

    gpu = native.run_host(make_params(prof, 16, 10**9, levels=3), small)
    viol, comp = audit_batch(small, gpu.finish_time)
    print(f"audit ok: {int(viol.sum())} violations", flush=True)


if __name__ == "__main__":
    main()
