"""Dev tool: first divergent logged round, GPU vs oracle, for one golden case.
    python tools/debug_golden.py <group> <case-name>"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from conftest import case_batch, case_params, golden_cases
from oracle_binding import run_oracle
from paper_2506_12204_b200 import _abi as A, native

group, name = sys.argv[1], sys.argv[2]
case = [c for c in golden_cases(group) if c["name"] == name][0]
batch = case_batch(case)
g = native.run_host(case_params(case, A.SS_FLAG_DIGEST), batch, want_log=True)
c = run_oracle(case_params(case, A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG), batch)
print("status", g.stats["status"][0], c.stats["status"][0], "rounds", g.stats["rounds"][0], c.stats["rounds"][0],
      "anomalies", g.stats["anomalies"][0], c.stats["anomalies"][0])
gr, cr = g.rounds(0), c.rounds(0)
for k in range(min(len(gr), len(cr))):
    a, w = gr[k], cr[k]
    if (a.kind != w.kind or list(a.granted) != list(w.granted) or a.mem_used != w.mem_used or
            list(a.completed) != list(w.completed) or a.time != w.time or
            [d[:5] for d in a.decisions] != [d[:5] for d in w.decisions]):
        print(f"first divergent logged round {k} of {len(gr)}/{len(cr)}")
        for j in range(max(0, k - 4), min(k + 3, len(gr), len(cr))):
            print("  gpu", j, gr[j].kind, list(gr[j].granted), list(gr[j].completed), gr[j].mem_used, gr[j].time, [d[:5] for d in gr[j].decisions])
            print("  cpu", j, cr[j].kind, list(cr[j].granted), list(cr[j].completed), cr[j].mem_used, cr[j].time, [d[:5] for d in cr[j].decisions])
        break
else:
    print("logs equal", len(gr), len(cr))
