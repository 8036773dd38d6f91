"""Dev tool: first divergent round between the CUDA path and the oracle."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from test_gpu_parity import _seeded_batch
from oracle_binding import run_oracle
from paper_2506_12204_b200.results import make_params
from paper_2506_12204_b200 import _abi as A, native

policy, cap = sys.argv[1], int(sys.argv[2])
bs = [int(x) for x in sys.argv[3].split(",")]
batch, cfg = _seeded_batch(48, 250, dict(levels=3), seed0=500)
for b in bs:
    gpu = native.run_host(make_params(cfg.gpu_profile(), b, cap, policy=policy, levels=3, flags=A.SS_FLAG_DIGEST), batch, want_log=True)
    cpu = run_oracle(make_params(cfg.gpu_profile(), b, cap, policy=policy, levels=3, flags=A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG), batch)
    bad = np.nonzero(gpu.stats["status"] != cpu.stats["status"])[0]
    print(f"b={b} mismatching traces {list(bad)} gpu {list(gpu.stats['status'][bad])} cpu {list(cpu.stats['status'][bad])}")
    for t in bad[:3]:
        g, c = gpu.rounds(t), cpu.rounds(t)
        for k in range(min(len(g), len(c))):
            a, w = g[k], c[k]
            if (a.kind != w.kind or list(a.granted) != list(w.granted) or a.mem_used != w.mem_used or
                    list(a.completed) != list(w.completed) or a.time != w.time or
                    [d[:5] for d in a.decisions] != [d[:5] for d in w.decisions]):
                print(f"  trace {t}: first divergent logged round {k} of {len(g)}/{len(c)}")
                for j in range(max(0, k - 2), min(k + 2, len(g), len(c))):
                    print("    gpu", j, g[j].kind, list(g[j].granted), list(g[j].completed), g[j].mem_used, g[j].time, g[j].decisions)
                    print("    cpu", j, c[j].kind, list(c[j].granted), list(c[j].completed), c[j].mem_used, c[j].time, c[j].decisions)
                break
        else:
            print(f"  trace {t}: logs equal over {min(len(g), len(c))} rounds (gpu {len(g)}, cpu {len(c)}); "
                  f"anomalies gpu {gpu.stats['anomalies'][t]} cpu {cpu.stats['anomalies'][t]} lost {gpu.stats['lost_evictions'][t]}/{cpu.stats['lost_evictions'][t]}")

# save GPU round logs of the mismatching traces for offline analysis
if len(sys.argv) > 4:
    out = {}
    for b in bs:
        gpu = native.run_host(make_params(cfg.gpu_profile(), b, cap, policy=policy, levels=3, flags=A.SS_FLAG_DIGEST), batch, want_log=True)
        cpu = run_oracle(make_params(cfg.gpu_profile(), b, cap, policy=policy, levels=3, flags=A.SS_FLAG_DIGEST | A.SS_FLAG_ROUND_LOG), batch)
        for t in np.nonzero(gpu.stats["status"] != cpu.stats["status"])[0]:
            out[f"b{b}_t{t}"] = gpu.logs[t]
    np.savez_compressed(sys.argv[4], **out)
