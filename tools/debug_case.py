"""Dev tool: first divergent logged round, GPU vs oracle, for one seeded case.
    python tools/debug_case.py <b> <capacity> <profile> <levels> <seed0> <ntraces> <total> [outlen_hi]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from test_gpu_parity import _seeded_batch
from oracle_binding import run_oracle
from paper_2506_12204_b200.results import make_params
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200 import _abi as A, native

b, cap, prof, levels, seed0, nt, total = sys.argv[1:8]
b, cap, levels, seed0, nt, total = int(b), int(cap), int(levels), int(seed0), int(nt), int(total)
kw = dict(levels=levels)
if len(sys.argv) > 8:
    kw["output_len_range"] = (1, int(sys.argv[8]))
batch, cfg = _seeded_batch(nt, total, kw, seed0=seed0)
pr = get_profile(prof)
for dep, cost in ((True, "max"), (False, "sum")):
    mk = lambda fl: make_params(pr, b, cap, levels=levels, dependency_rule=dep, decode_batch_cost=cost, flags=fl)
    g = native.run_host(mk(A.SS_FLAG_DIGEST), batch, want_log=True)
    c = run_oracle(mk(A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG), batch)
    bad = [t for t in range(nt) if g.stats["digest"][t] != c.stats["digest"][t] or g.stats["status"][t] != c.stats["status"][t]]
    print(f"dep={dep} cost={cost}: {len(bad)} traces differ {bad[:10]}")
    for t in bad[:2]:
        gr, cr = g.rounds(t), c.rounds(t)
        for k in range(min(len(gr), len(cr))):
            a, w = gr[k], cr[k]
            if (a.kind != w.kind or list(a.granted) != list(w.granted) or a.mem_used != w.mem_used or
                    list(a.completed) != list(w.completed) or a.time != w.time or
                    [d[:5] for d in a.decisions] != [d[:5] for d in w.decisions]):
                print(f"  trace {t}: first divergent logged round {k} of {len(gr)}/{len(cr)}")
                for j in range(max(0, k - 3), min(k + 2, len(gr), len(cr))):
                    print("    gpu", j, gr[j].kind, list(gr[j].granted), list(gr[j].completed), gr[j].mem_used, gr[j].time, gr[j].decisions)
                    print("    cpu", j, cr[j].kind, list(cr[j].granted), list(cr[j].completed), cr[j].mem_used, cr[j].time, cr[j].decisions)
                break
        else:
            print(f"  trace {t}: logs equal over {min(len(gr), len(cr))} (gpu {len(gr)} cpu {len(cr)} rounds; "
                  f"status gpu {g.stats['status'][t]} cpu {c.stats['status'][t]}; rounds {g.stats['rounds'][t]} "
                  f"{c.stats['rounds'][t]}; anomalies {g.stats['anomalies'][t]} {c.stats['anomalies'][t]})")
            if len(gr) > len(cr):
                for j in range(len(cr), min(len(gr), len(cr) + 2)):
                    print("    gpu extra", j, gr[j].kind, list(gr[j].granted), gr[j].mem_used, gr[j].decisions)
            for j in range(max(0, min(len(gr), len(cr)) - 3), min(len(gr), len(cr))):
                print("    last", j, gr[j].kind, list(gr[j].granted), list(gr[j].completed), gr[j].mem_used, gr[j].decisions)
