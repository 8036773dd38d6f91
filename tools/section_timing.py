"""Dev tool: warp-cycles per scheduler-kernel section (libss_dbgtime.so, built with
-DSS_DEBUG_TIMING) on a bench workload. Usage: section_timing.py <workload> [traces]"""
import ctypes as C, os, sys
os.environ["SS_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2506_12204_b200", "_lib", os.environ.get("SS_DBG_LIB", "libss_dbgtime.so"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import bench
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
W = sys.argv[1]
wl = bench.WORKLOADS[W]
T = int(sys.argv[2]) if len(sys.argv) > 2 else wl["traces"]
batch, T = bench.build_batch(wl, 0, T, pinned=False)
prm = make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST)
lib = native.lib()
buf = (C.c_ulonglong * 16)()
native.run_host(prm, batch)  # warm-up
lib.ss_debug_cycles(buf)
res = native.run_host(prm, batch)
lib.ss_debug_cycles(buf)
v = list(buf)
tot = sum(v[:8]) or 1
names = ["init/admission/top", "fast per-round body", "chunk", "general round", "outputs", "stretch entry", "stretch vote", "stretch order"]
rounds = int(res.stats["rounds"].sum())
print(f"{W}: {T} traces, {rounds} rounds, kernel {res.kernel_ms:.2f} ms")
for i, n in enumerate(names):
    print(f"  {n:20s} {100 * v[i] / tot:5.1f}%  {v[i] / max(rounds, 1):8.1f} warp-cycles/round")
print(f"  chunks {v[8]}, chunk rounds {v[9]} ({v[9] / max(v[8], 1):.1f}/chunk), per-round fast {v[10]}, general {v[11]}")
if v[8]: print(f"  cycles/chunk {v[2] / v[8]:.0f}, per chunk round {v[2] / max(v[9], 1):.0f}")
if v[10]: print(f"  cycles per per-round fast round {v[1] / v[10]:.0f} (incl. stretch setup/exit)")
if v[11]: print(f"  cycles per general round {v[3] / v[11]:.0f}")
