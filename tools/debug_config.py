"""Dev tool: per-trace GPU-vs-oracle comparison on a bench workload sample,
with the first divergent round of each mismatching trace.

    python tools/debug_config.py D 64 [bulk_min]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np

import bench
from oracle_binding import run_oracle
from paper_2506_12204_b200 import _abi as A
from paper_2506_12204_b200 import native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params

wname, ntr = sys.argv[1], int(sys.argv[2])
wl = bench.WORKLOADS[wname]
batch, T = bench.build_batch(wl, 0, ntr, pinned=False)
prof = get_profile(wl["profile"])
mk = lambda fl: make_params(prof, 16, wl["capacity"], levels=wl["levels"], flags=fl)
gpu = native.run_host(mk(A.SS_FLAG_DIGEST), batch)
cpu = run_oracle(mk(A.SS_FLAG_DIGEST), batch, threads=os.cpu_count())
keys = ("status", "rounds", "digest", "evictions", "lost_evictions", "anomalies", "completed")
bad = [t for t in range(T) if any(gpu.stats[k][t] != cpu.stats[k][t] for k in keys)]
print(f"{len(bad)} / {T} traces differ: {bad[:20]}")
for t in bad[:4]:
    print(f" trace {t}: " + ", ".join(f"{k} gpu {gpu.stats[k][t]} cpu {cpu.stats[k][t]}" for k in keys))
    sub = batch.subset([t])
    g = native.run_host(mk(A.SS_FLAG_DIGEST), sub, want_log=True)
    c = run_oracle(mk(A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG), sub)
    gr, cr = g.rounds(0), c.rounds(0)
    for k in range(min(len(gr), len(cr))):
        a, w = gr[k], cr[k]
        if (a.kind != w.kind or list(a.granted) != list(w.granted) or a.mem_used != w.mem_used or
                list(a.completed) != list(w.completed) or a.time != w.time or
                [d[:5] for d in a.decisions] != [d[:5] for d in w.decisions]):
            print(f"  first divergent logged round {k} of {len(gr)}/{len(cr)}")
            for j in range(max(0, k - 3), min(k + 2, len(gr), len(cr))):
                print("    gpu", j, gr[j].kind, list(gr[j].granted), list(gr[j].completed), gr[j].mem_used, gr[j].time,
                      gr[j].decisions)
                print("    cpu", j, cr[j].kind, list(cr[j].granted), list(cr[j].completed), cr[j].mem_used, cr[j].time,
                      cr[j].decisions)
            break
    else:
        print(f"  logs equal over {min(len(gr), len(cr))} rounds")
