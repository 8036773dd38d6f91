"""Dev tool: first round whose digest differs (GPU vs oracle) by bisecting
max_rounds, then the per-request state differences after that round.
    python tools/dbg_bisect.py b cap levels seed0 ntraces total trace_index"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
from test_gpu_parity import _seeded_batch
from oracle_binding import run_oracle
from paper_2506_12204_b200.results import make_params
from paper_2506_12204_b200 import _abi as A, native

b, cap, levels, seed0, nt, total, ti = map(int, sys.argv[1:8])
batch, cfg = _seeded_batch(nt, total, dict(levels=levels), seed0=seed0)
sub = batch.subset([ti])
mk = lambda r, fl=A.SS_FLAG_DIGEST: make_params(cfg.gpu_profile(), b, cap, levels=levels, flags=fl, max_rounds=r)
def both(r):
    return native.run_host(mk(r), sub), run_oracle(mk(r), sub)
g, c = both(0)
print("full:", g.stats["rounds"][0], c.stats["rounds"][0], g.stats["status"][0], c.stats["status"][0])
lo, hi = 1, int(min(g.stats["rounds"][0], c.stats["rounds"][0]))
while lo < hi:
    mid = (lo + hi) // 2
    g, c = both(mid)
    if g.stats["digest"][0] == c.stats["digest"][0] and g.stats["rounds"][0] == c.stats["rounds"][0]:
        lo = mid + 1
    else:
        hi = mid
print("first differing round cap", lo)
for r in (lo - 1, lo):
    g, c = both(r)
    print(f"-- after {r} rounds: status {g.stats['status'][0]} {c.stats['status'][0]} evictions {g.stats['evictions'][0]} {c.stats['evictions'][0]} lost {g.stats['lost_evictions'][0]} {c.stats['lost_evictions'][0]} anomalies {g.stats['anomalies'][0]} {c.stats['anomalies'][0]} clock {g.stats['final_clock'][0]} {c.stats['final_clock'][0]}")
    for k in ("f_t", "state", "generated", "evictions", "first_scheduled", "finish_time"):
        a, w = getattr(g, k), getattr(c, k)
        d = np.nonzero(~((a == w) | (np.isnan(a.astype(float)) & np.isnan(w.astype(float)))))[0]
        if len(d):
            print("  ", k, "slots", d[:10], "gpu", a[d[:10]], "cpu", w[d[:10]])
gl = native.run_host(mk(lo), sub, want_log=True)
cl = run_oracle(mk(lo, A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG), sub)
for j in range(max(0, len(gl.rounds(0)) - 3), len(gl.rounds(0))):
    x = gl.rounds(0)[j]; print("  gpu log", j, x.kind, list(x.granted), list(x.completed), x.mem_used, [d[:5] for d in x.decisions])
for j in range(max(0, len(cl.rounds(0)) - 3), len(cl.rounds(0))):
    x = cl.rounds(0)[j]; print("  cpu log", j, x.kind, list(x.granted), list(x.completed), x.mem_used, [d[:5] for d in x.decisions])
