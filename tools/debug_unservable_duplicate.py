"""Dev tool: the unservable-duplicate trace (seed 2808, 40 requests, b = 8, 400 slots) where
the kernel reports LIVELOCK and the reference / oracle an IllegalTransitionError."""
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from oracle_binding import run_oracle
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
from paper_2506_12204_b200.tracegen import generate_batch
from paper_2506_12204_b200.workload import WorkloadSpec
batch = generate_batch(WorkloadSpec(total_requests=40, levels=3), [2808], pinned=False)
p = lambda g=0: make_params(get_profile("a100_qwen7b"), 8, 400, levels=3, flags=A.SS_FLAG_DIGEST | g)
gpu = native.run_host(p(), batch, want_log=True)
cpu = run_oracle(p(A.SS_FLAG_ROUND_LOG), batch)
g, c = gpu.rounds(0), cpu.rounds(0)
print(len(g), len(c), gpu.stats["status"], cpu.stats["status"], gpu.stats["anomalies"], cpu.stats["anomalies"], gpu.stats["lost_evictions"], cpu.stats["lost_evictions"])
for k in range(min(len(g), len(c))):
    a, w = g[k], c[k]
    if (a.kind != w.kind or list(a.granted) != list(w.granted) or a.mem_used != w.mem_used or
            list(a.completed) != list(w.completed) or a.time != w.time or [d[:5] for d in a.decisions] != [d[:5] for d in w.decisions]):
        print("first divergent", k)
        break
for j in range(k - 6, k + 2):
    if j < len(g): print("gpu", j, g[j].kind, list(g[j].granted), list(g[j].completed), g[j].mem_used, g[j].decisions)
    if j < len(c): print("cpu", j, c[j].kind, list(c[j].granted), list(c[j].completed), c[j].mem_used, c[j].decisions)
print("prompt", list(batch.prompt), "out", list(batch.true_out), "mid", list(batch.pred_len))
